"""HBM layout A/B for the streamed kernels: the planes of a batch as separate
allocations (one torch tensor per plane) vs carved from one slab (consecutive
planes of one allocation), config 3 (h only, 2^28) and config 2 (h + pdf,
2^24), cap and Heitz, measured interleaved (back-to-back calls, median of R).

python tools/slab_ab.py [R]
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

R = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dev = torch.device("cuda:0")
L = ctypes.CDLL(os.path.join(ROOT, "paper_2306_05044_b200", "libvndf.so"))
L.vndf_sample_cap.argtypes = [ctypes.c_void_p] * 10 + [ctypes.c_int64, ctypes.c_void_p]
for fn in ("vndf_sample_cap_pdf", "vndf_sample_heitz2018"):
    getattr(L, fn).argtypes = [ctypes.c_void_p] * 11 + [ctypes.c_int64, ctypes.c_void_p]


def layouts(cid):
    cfg = synth.CONFIGS[cid]
    n, nout = cfg.n, 4 if cfg.pdf else 3
    sep_in = synth.fill(cfg.recipe, cfg.seed, n, device=dev)
    sep_out = [torch.empty(n, device=dev) for _ in range(nout)]
    slab = torch.empty((7 + nout) * n, device=dev)
    views = {k: slab[j * n:(j + 1) * n] for j, k in enumerate(synth.PLANES)}
    synth.fill(cfg.recipe, cfg.seed, n, out=views)
    slab_out = [slab[(7 + j) * n:(8 + j) * n] for j in range(nout)]
    return cfg, {"separate": ([sep_in[k] for k in synth.PLANES], sep_out),
                 "slab": ([views[k] for k in synth.PLANES], slab_out)}


def t_us(f, args, n, reps):
    for _ in range(3):
        f(*args, n, None)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f(*args, n, None)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


for cid in (3, 2):
    cfg, lay = layouts(cid)
    nb = (44 if cfg.pdf else 40) * cfg.n
    res = {}
    for _ in range(R):
        for name, (ins, outs) in lay.items():
            P = [ctypes.c_void_p(t.data_ptr()) for t in ins] + [ctypes.c_void_p(t.data_ptr()) for t in outs]
            cap = L.vndf_sample_cap_pdf if cfg.pdf else L.vndf_sample_cap
            hz = P + ([] if cfg.pdf else [None])
            reps = 10 if cid == 3 else 50
            res.setdefault((name, "cap"), []).append(t_us(cap, P, cfg.n, reps))
            res.setdefault((name, "heitz"), []).append(t_us(L.vndf_sample_heitz2018, hz, cfg.n, reps))
            # outputs identical across layouts
    row = {"config": cid}
    for (name, m), v in res.items():
        us = statistics.median(v)
        row[f"{name}_{m}_gbs"] = round(nb / us / 1e3, 1)
    print(json.dumps(row), flush=True)
    del lay
    torch.cuda.empty_cache()
