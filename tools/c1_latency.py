"""Device time per launch of the streamed kernels at small n (config-1 size,
L2-resident, latency-bound): 50 launches captured in a CUDA graph and replayed.

python tools/c1_latency.py lib1.so [lib2.so ...]
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402

dev = torch.device("cuda:0")
for path in sys.argv[1:]:
    L = ctypes.CDLL(os.path.abspath(path))
    for fn in ("vndf_sample_cap_pdf", "vndf_sample_heitz2018"):
        getattr(L, fn).argtypes = [ctypes.c_void_p] * 11 + [ctypes.c_int64, ctypes.c_void_p]
    res = {"lib": os.path.basename(path)}
    for n in (1 << 14, 1 << 16, 1 << 18, 1 << 20):
        x = synth.fill(1, 0, n, device=dev)
        out = [torch.empty(n, device=dev) for _ in range(4)]
        P = [ctypes.c_void_p(x[k].data_ptr()) for k in synth.PLANES] + [ctypes.c_void_p(t.data_ptr()) for t in out]
        for name in ("vndf_sample_cap_pdf", "vndf_sample_heitz2018"):
            f = getattr(L, name)
            f(*P, n, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
                for _ in range(50):
                    f(*P, n, s)
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            res[f"{name.split('_')[-1]}_2^{n.bit_length() - 1}_us"] = round(a.elapsed_time(b) * 1e3 / 500, 3)
    print(json.dumps(res), flush=True)
