"""Per-launch overhead of the streamed cap+pdf kernel: back-to-back launches on
config-2-recipe inputs of several sizes; a least-squares fit t = a + n b gives
the fixed cost per launch (a: ramp, drain, grid boundary) and the asymptotic
bandwidth (44 B / b).

python tools/size_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_05044_b200 as vndf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
sizes = [1 << k for k in range(20, 28)]
x = synth.fill(2, 1, sizes[-1], device=dev)
out = vndf.empty_outputs(sizes[-1], dev)
rows = []
for n in sizes:
    ins = [x[k][:n] for k in synth.PLANES]
    o = [t[:n] for t in out]
    reps = max(20, min(400, (1 << 30) // n))
    for _ in range(5):
        vndf.vndf_sample_cap_pdf(*ins, *o)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            vndf.vndf_sample_cap_pdf(*ins, *o)
        b.record(st)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    rows.append((n, best))
    print(f"n=2^{n.bit_length() - 1:2d}  {best * 1e3:9.2f} us/launch  {44 * n / best / 1e6:7.0f} GB/s", flush=True)
big = [(n, t) for n, t in rows if n >= 1 << 23]
A = np.array([[1.0, n] for n, _ in big])
y = np.array([t for _, t in big])
(a, b), *_ = np.linalg.lstsq(A, y, rcond=None)
print(f"fit over n >= 2^23: fixed {a * 1e3:.2f} us/launch, asymptotic {44 / b / 1e6:.0f} GB/s")
