"""A/B of the default streamed launch shape of two or more builds: device time per
call (CUDA-graph replay of 20 calls) of cap+pdf and Heitz at 2^16..2^26 samples
(config-2 inputs), twice.

python tools/stream_ab.py libA.so libB.so
"""
import ctypes, json, os, sys, torch
sys.path.insert(0, '/root/repo')
import synth
dev = torch.device('cuda:0')
libs = sys.argv[1:]
N = 1 << 26
x = synth.fill(2, 1, N, device=dev)
out = [torch.empty(N, device=dev) for _ in range(4)]
def fns(path):
    L = ctypes.CDLL(os.path.abspath(path))
    for fn in ("vndf_sample_cap_pdf", "vndf_sample_heitz2018"):
        getattr(L, fn).argtypes = [ctypes.c_void_p] * 11 + [ctypes.c_int64, ctypes.c_void_p]
    return L
Ls = {p: fns(p) for p in libs}
def ptrs(n):
    return [ctypes.c_void_p(x[k][:n].data_ptr()) for k in synth.PLANES] + [ctypes.c_void_p(t[:n].data_ptr()) for t in out]
def graph_us(f, n):
    P = ptrs(n); s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert f(*P, n, s) == 0; torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        for _ in range(20): f(*P, n, s)
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): g.replay()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / 200
for rep in range(2):
    for lg in range(16, 27):
        n = 1 << lg
        row = {"log2n": lg}
        for p, L in Ls.items():
            nm = os.path.basename(p).replace('.so', '')
            c = graph_us(L.vndf_sample_cap_pdf, n); h = graph_us(L.vndf_sample_heitz2018, n)
            row[nm + "_cap_us"] = round(c, 3); row[nm + "_heitz_us"] = round(h, 3)
        print(json.dumps(row), flush=True)
