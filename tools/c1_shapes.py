"""Config-1 latency (2^16 samples, L2-resident) of the cap and Heitz streamed
kernels against the launch shape (vector width x block size), for one or more
builds of libvndf: device time per launch, 50 launches in a CUDA graph replayed
10 times (tools/c1_latency.py's method).

python tools/c1_shapes.py [--log2n 16,18,20] lib1.so [lib2.so ...]
(sizes above 2^16 use config-2 inputs)
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
args = sys.argv[1:]
sizes = [16]
if args and args[0] == "--log2n":
    sizes = [int(v) for v in args[1].split(",")]
    args = args[2:]
n = P = None


def inputs(lg):
    global n, P
    n = 1 << lg
    x = synth.fill(1 if lg <= 16 else 2, 0, n, device=dev)
    out = [torch.empty(n, device=dev) for _ in range(4)]
    P = [ctypes.c_void_p(x[k].data_ptr()) for k in synth.PLANES] + [ctypes.c_void_p(t.data_ptr()) for t in out]
    return x, out


def per_launch_us(f):
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert f(*P, n, s) == 0
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
    return round(a.elapsed_time(b) * 1e3 / 500, 3)


for lg in sizes:
    keep = inputs(lg)
    for path in args:
        L = ctypes.CDLL(os.path.abspath(path))
        for fn in ("vndf_sample_cap_pdf", "vndf_sample_heitz2018"):
            getattr(L, fn).argtypes = [ctypes.c_void_p] * 11 + [ctypes.c_int64, ctypes.c_void_p]
        L.vndf_set_launch_config.argtypes = [ctypes.c_int] * 3
        for vw in (0, 8, 4, 1):
            for blk in ((0,) if vw == 0 else (64, 128, 256)):
                assert L.vndf_set_launch_config(vw, blk, 0) == 0
                cap = per_launch_us(L.vndf_sample_cap_pdf)
                hz = per_launch_us(L.vndf_sample_heitz2018)
                print(json.dumps({"lib": os.path.basename(path), "log2n": lg, "vector_width": vw or "default",
                                  "block": blk or "default", "cap_us": cap, "heitz_us": hz,
                                  "t_heitz_over_t_cap": round(hz / cap, 4)}), flush=True)
        L.vndf_set_launch_config(0, 0, 0)
