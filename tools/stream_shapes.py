"""Streamed-kernel launch shapes (vndf_set_launch_config: vector width x block
size) at configs 2, 3 and 5, cap and Heitz, GB/s (CUDA events, 20 launches).

python tools/stream_shapes.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2306_05044_b200 as vndf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")


def gbs(fn, nbytes, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return round(nbytes * reps / (a.elapsed_time(b) * 1e-3) / 1e9, 1)


for cid in (2, 3, 5):
    cfg = synth.CONFIGS[cid]
    x = synth.fill(cfg.recipe, cfg.seed, cfg.n, device=dev)
    ins = [x[k] for k in synth.PLANES]
    out = vndf.empty_outputs(cfg.n, dev, pdf=cfg.pdf)
    nb = (44 if cfg.pdf else 40) * cfg.n
    for vw, blk in ((8, 64), (8, 128), (8, 256), (4, 128), (4, 256)):
        vndf.vndf_set_launch_config(vw, blk, 0)
        if cfg.pdf:
            cap = gbs(lambda: vndf.vndf_sample_cap_pdf(*ins, *out), nb)
            hz = gbs(lambda: vndf.vndf_sample_heitz2018(*ins, *out), nb)
        else:
            cap = gbs(lambda: vndf.vndf_sample_cap(*ins, *out), nb)
            hz = gbs(lambda: vndf.vndf_sample_heitz2018(*ins, *out, None), nb)
        print(json.dumps({"config": cid, "vector_width": vw, "block": blk, "cap_gbs": cap, "heitz_gbs": hz}),
              flush=True)
    vndf.vndf_set_launch_config(0, 0, 0)
    del x, ins, out
    torch.cuda.empty_cache()
