"""Interleaved A/B of explicit streamed launch shapes at given call sizes (cap+pdf
and Heitz, config-2 inputs): device time per call by CUDA-graph replay of 20
calls, shapes measured round-robin R times so drift hits all of them alike;
prints the median per shape.

python tools/shape_ab.py 21,22,23,24 8x128,8x64,4x64,4x128 [R] [graph|stream]
(stream: 20 calls launched back to back on the current stream, no graph)
VNDF_AB_SEPARATE=1: inputs and outputs allocated at exactly n per size (as the
bench's per-config buffers) instead of slices of one 2^max allocation.
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
MODE = sys.argv[4] if len(sys.argv) > 4 else "graph"
dev = torch.device("cuda:0")
SEPARATE = os.environ.get("VNDF_AB_SEPARATE") == "1"
N = 1 << max(sizes)
x = out = None
if not SEPARATE:
    x = synth.fill(2, 1, N, device=dev)
    out = [torch.empty(N, device=dev) for _ in range(4)]
L = ctypes.CDLL(os.path.join(ROOT, "paper_2306_05044_b200", "libvndf.so"))
for fn in ("vndf_sample_cap_pdf", "vndf_sample_heitz2018"):
    getattr(L, fn).argtypes = [ctypes.c_void_p] * 11 + [ctypes.c_int64, ctypes.c_void_p]
L.vndf_set_launch_config.argtypes = [ctypes.c_int] * 3


def graph_us(f, n):
    P = [ctypes.c_void_p(x[k][:n].data_ptr()) for k in synth.PLANES] + [ctypes.c_void_p(t[:n].data_ptr()) for t in out]
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert f(*P, n, s) == 0
    torch.cuda.synchronize()
    if MODE == "stream":
        for _ in range(3):
            f(*P, n, s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            f(*P, n, s)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e3 / 20
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
    if SEPARATE:
        x = out = None
        torch.cuda.empty_cache()
        x = synth.fill(2, 1, n, device=dev)
        out = [torch.empty(n, device=dev) for _ in range(4)]
    res = {sh: {"cap": [], "heitz": []} for sh in shapes}
    for _ in range(R):
        for sh in shapes:
            L.vndf_set_launch_config(sh[0], sh[1], 0)
            res[sh]["cap"].append(graph_us(L.vndf_sample_cap_pdf, n))
            res[sh]["heitz"].append(graph_us(L.vndf_sample_heitz2018, n))
    L.vndf_set_launch_config(0, 0, 0)
    row = {"log2n": lg, "mode": MODE, "separate": SEPARATE}
    for sh in shapes:
        row[f"{sh[0]}x{sh[1]}"] = [round(statistics.median(res[sh]["cap"]), 3), round(statistics.median(res[sh]["heitz"]), 3)]
    print(json.dumps(row), flush=True)
