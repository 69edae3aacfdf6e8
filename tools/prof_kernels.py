"""Small driver for ncu captures: a few launches of each hot kernel.

python tools/prof_kernels.py [which]   which in {all, c2, c3, c4, c4full, c5, c5fused, reflect_philox, next}
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2306_05044_b200 as vndf  # noqa: E402
import synth  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
dev = torch.device("cuda:0")
for cid in (2, 3, 5):
    if which not in ("all", f"c{cid}"):
        continue
    cfg = synth.CONFIGS[cid]
    x = synth.fill(cfg.recipe, cfg.seed, cfg.n, device=dev)
    ins = [x[k] for k in synth.PLANES]
    out = vndf.empty_outputs(cfg.n, dev, pdf=cfg.pdf)
    for _ in range(2):
        if cfg.pdf:
            vndf.vndf_sample_cap_pdf(*ins, *out)
            vndf.vndf_sample_heitz2018(*ins, *out)
        else:
            vndf.vndf_sample_cap(*ins, *out)
            vndf.vndf_sample_heitz2018(*ins, *out, None)
    torch.cuda.synchronize()
    del x, ins, out
if which in ("all", "c4"):
    n = 1 << 26
    o = vndf.empty_outputs(n, dev)
    for _ in range(2):
        vndf.vndf_sample_cap_philox(3, 0, n, *o)
        vndf.vndf_sample_heitz2018_philox(3, 0, n, *o)
    torch.cuda.synchronize()
if which == "c4full":  # the bench step's launch shape: 2^30 samples, one call each
    n = 1 << 30
    o = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_philox(3, 0, n, *o)
    vndf.vndf_sample_heitz2018_philox(3, 0, n, *o)
    torch.cuda.synchronize()
if which in ("all", "c5fused"):
    n = 1 << 26
    o = vndf.empty_outputs(n, dev)
    for _ in range(2):
        vndf.vndf_sample_cap_philox_edge(4, 0, n, *o)
        vndf.vndf_sample_heitz2018_philox_edge(4, 0, n, *o)
    torch.cuda.synchronize()
if which in ("all", "reflect_philox"):
    n = 1 << 26
    o = [torch.empty(n, device=dev) for _ in range(5)]
    for _ in range(2):
        vndf.vndf_sample_cap_reflect_philox(3, 0, n, *o)
        vndf.vndf_sample_heitz2018_reflect_philox(3, 0, n, *o)
    torch.cuda.synchronize()
print("ok")

if which in ("all", "next"):
    cfg = synth.CONFIGS[2]
    x = synth.fill(cfg.recipe, cfg.seed, cfg.n, device=dev)
    ins = [x[k] for k in synth.PLANES]
    ro = [torch.empty(cfg.n, device=dev) for _ in range(5)]
    for _ in range(2):
        vndf.vndf_sample_cap_reflect(*ins, *ro)
        vndf.vndf_pdf(*ro[:3], *ins[:5], ro[3])
    ck = torch.empty(148 * 2048 * 16, device=dev)
    for m in (0, 1, 2):
        vndf.vndf_microbench(m, 5, ck.numel(), 64, ck)
    s = torch.zeros(2, dtype=torch.float64, device=dev)
    for m in (0, 1):
        vndf.vndf_furnace(m, (0.5, 0.2, 0.8426149773176359), (0.3, 0.1), 17, 1 << 26, s)
    torch.cuda.synchronize()
    print("next ok")
