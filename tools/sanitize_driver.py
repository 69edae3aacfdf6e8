"""Small driver exercising every libvndf entry point (ragged sizes, all vector
paths, fix-up paths) for `compute-sanitizer --tool memcheck` (one tool per run)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_05044_b200 as vndf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
for n in (1, 7, 9, 4099, 70001):
    for off in (0, 4, 1):
        x = synth.fill(5, 4, n, device=dev)
        ins = []
        for k in synth.PLANES:
            b = torch.zeros(n + 8, device=dev)
            b[off:off + n] = x[k]
            ins.append(b[off:off + n])
        outs = [torch.zeros(n + 8, device=dev)[off:off + n] for _ in range(5)]
        vndf.vndf_sample_cap_pdf(*ins, *outs[:4])
        vndf.vndf_sample_cap(*ins, *outs[:3])
        vndf.vndf_sample_heitz2018(*ins, *outs[:4])
        vndf.vndf_sample_heitz2018(*ins, *outs[:3], None)
        vndf.vndf_sample_cap_reflect(*ins, *outs)
        vndf.vndf_pdf(*outs[:3], *ins[:5], outs[3])
        c = torch.zeros(1, dtype=torch.int64, device=dev)
        vndf.vndf_count_fixups(*ins, c)
        o = [torch.zeros(n + 8, device=dev)[off:off + n] for _ in range(4)]
        vndf.vndf_sample_cap_philox(3, 2**32 - 5, n, *o)
        vndf.vndf_sample_heitz2018_philox(3, 7, n, *o[:3], None)
        vndf.vndf_count_fixups_philox(3, 0, n, c)
        vndf.vndf_sample_cap_philox_edge(4, 3, n, *o)
        vndf.vndf_sample_heitz2018_philox_edge(4, 0, n, *o[:3], None)
        vndf.vndf_sample_cap_pdf_native(*ins, *outs[:4])
        r = [torch.zeros(n + 8, device=dev)[off:off + n] for _ in range(5)]
        vndf.vndf_sample_cap_reflect_philox(3, 1, n, *r)
        w = torch.zeros(4 * n, dtype=torch.int32, device=dev)
        vndf.vndf_philox4x32_10(3, 0, n, 1, w)
    hin = [x[k].cpu().pin_memory() for k in synth.PLANES]
    hout = [torch.zeros(n).pin_memory() for _ in range(4)]
    vndf.vndf_sample_cap_pdf_host(*hin, *hout)
    vndf.vndf_sample_cap_pdf_host(*hin, *hout[:3], None)
    vndf.vndf_sample_cap_philox_host(3, 5, n, *hout)
s = torch.zeros(2, dtype=torch.float64, device=dev)
vndf.vndf_furnace(0, (0.3, 0.2, 0.9327379), (0.05, 0.3), 1, 100003, s)
vndf.vndf_furnace(1, (0.3, 0.2, 0.9327379), (0.05, 0.3), 1, 100003, s)
ck = torch.zeros(1000, device=dev)
for m in (0, 1, 2):
    vndf.vndf_microbench(m, 1, 1000, 64, ck)
torch.cuda.synchronize()
print("sanitize driver ok")
