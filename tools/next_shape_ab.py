"""Interleaved A/B of explicit launch shapes for the streamed NEXT kernels
(vndf_sample_cap_reflect, vndf_pdf) at given sizes (config-2 inputs; the pdf
is evaluated at the inputs' own wi as h): device time per call by graph replay
of 20 calls, median of R rounds.

python tools/next_shape_ab.py 16,18,20,22,24,26 8x128,4x128,1x256,1x64 [R]
"""
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402

sizes = [int(v) for v in sys.argv[1].split(",")]
shapes = [tuple(int(t) for t in s.split("x")) for s in sys.argv[2].split(",")]
R = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dev = torch.device("cuda:0")
N = 1 << max(sizes)
x = synth.fill(2, 1, N, device=dev)
out = [torch.empty(N, device=dev) for _ in range(5)]
L = ctypes.CDLL(os.path.join(ROOT, "paper_2306_05044_b200", "libvndf.so"))
L.vndf_sample_cap_reflect.argtypes = [ctypes.c_void_p] * 12 + [ctypes.c_int64, ctypes.c_void_p]
L.vndf_pdf.argtypes = [ctypes.c_void_p] * 9 + [ctypes.c_int64, ctypes.c_void_p]
L.vndf_set_launch_config.argtypes = [ctypes.c_int] * 3


def ptrs(n, which):
    p = lambda t: ctypes.c_void_p(t[:n].data_ptr())  # noqa: E731
    ins = [p(x[k]) for k in synth.PLANES]
    if which == "reflect":
        return ins + [p(t) for t in out]
    return [ins[0], ins[1], ins[2], ins[0], ins[1], ins[2], ins[3], ins[4], p(out[0])]


def graph_us(f, P, n):
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert f(*P, n, s) == 0
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        for _ in range(20):
            f(*P, n, s)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / 100


for lg in sizes:
    n = 1 << lg
    res = {(w, sh): [] for w in ("reflect", "pdf") for sh in shapes}
    for _ in range(R):
        for w, f in (("reflect", L.vndf_sample_cap_reflect), ("pdf", L.vndf_pdf)):
            P = ptrs(n, w)
            for sh in shapes:
                L.vndf_set_launch_config(sh[0], sh[1], 0)
                res[(w, sh)].append(graph_us(f, P, n))
    L.vndf_set_launch_config(0, 0, 0)
    row = {"log2n": lg}
    for (w, sh), v in res.items():
        row[f"{w}_{sh[0]}x{sh[1]}"] = round(statistics.median(v), 3)
    print(json.dumps(row), flush=True)
