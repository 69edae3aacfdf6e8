"""Time the fused config-5 (edge mix) kernels of several builds of libvndf.

python tools/edge_variants.py lib1.so [lib2.so ...]
"""
import ctypes, os, sys, json, torch
dev = torch.device("cuda:0"); n = 1 << 26
outs = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(4)]
P = [ctypes.c_void_p(t.data_ptr()) for t in outs]
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for p in sys.argv[1:]:
    L = ctypes.CDLL(os.path.abspath(p)); res = {"lib": os.path.basename(p)}
    for fn in ("vndf_sample_cap_philox_edge", "vndf_sample_heitz2018_philox_edge"):
        f = getattr(L, fn); f.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64] + [ctypes.c_void_p] * 5
        for _ in range(3): f(4, 0, n, *P, s)
        torch.cuda.synchronize(); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): f(4, 0, n, *P, s)
        b.record(); torch.cuda.synchronize(); res[fn] = round(n / (a.elapsed_time(b) / 20) / 1e6, 2)
    print(json.dumps(res), flush=True)
