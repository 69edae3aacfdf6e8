"""Host-path throughput probe: torch pinned copies vs vndf_sample_cap_pdf_host."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_05044_b200 as vndf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
n = 1 << 24
x = synth.fill(2, 1, n, device=dev)
hin = [x[k].cpu().pin_memory() for k in synth.PLANES]
hout = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(4)]
d = [torch.empty(n, device=dev) for _ in range(7)]
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    for k in range(7):
        d[k].copy_(hin[k], non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for k in range(4):
        hout[k].copy_(d[k], non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    t3 = time.perf_counter()
    with torch.cuda.stream(s1):
        for k in range(7):
            d[k].copy_(hin[k], non_blocking=True)
    with torch.cuda.stream(s2):
        for k in range(4):
            hout[k].copy_(d[k], non_blocking=True)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"h2d {28 * n / (t1 - t0) / 1e9:.1f} GB/s  d2h {16 * n / (t2 - t1) / 1e9:.1f} GB/s  "
          f"duplex {44 * n / (t4 - t3) / 1e9:.1f} GB/s ({(t4 - t3) * 1e3:.2f} ms)")
for rep in range(5):
    t0 = time.perf_counter()
    vndf.vndf_sample_cap_pdf_host(*hin, *hout)
    t1 = time.perf_counter()
    print(f"host api {(t1 - t0) * 1e3:.2f} ms  {n / (t1 - t0) / 1e9:.3f} Gsamples/s")
