"""Launch-configuration sweep and host-path diagnostics (GPU box only).

python tools/tune.py  -> one JSON line per measurement on stdout.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2306_05044_b200 as vndf  # noqa: E402
import synth  # noqa: E402


def timed(fn, reps=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def emit(**kw):
    print(json.dumps(kw), flush=True)


dev = torch.device("cuda:0")
# reference copy bandwidth (same method as MEASURED_PEAKS: b.copy_(a), read+write bytes)
a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
b = torch.empty_like(a)
ms = timed(lambda: b.copy_(a), reps=10, warm=3)
emit(what="copy_1Gi_bf16", gb_s=2 * a.numel() * 2 / ms / 1e6)
a2 = torch.empty(1 << 28, dtype=torch.float32, device=dev)
b2 = torch.empty_like(a2)
ms = timed(lambda: b2.copy_(a2), reps=10, warm=3)
emit(what="copy_2^28_f32", gb_s=2 * a2.numel() * 4 / ms / 1e6)
del a, b, a2, b2

for cid in (2, 3):
    cfg = synth.CONFIGS[cid]
    x = synth.fill(cfg.recipe, cfg.seed, cfg.n, device=dev)
    ins = [x[k] for k in synth.PLANES]
    out = vndf.empty_outputs(cfg.n, dev, pdf=cfg.pdf)
    bps = 44 if cfg.pdf else 40
    for vw in (8, 4):
        for bs in (256, 128):
            for bpsm in (0, 2, 3, 4, -1):
                try:
                    vndf.vndf_set_launch_config(vw, bs, bpsm)
                except Exception as e:  # noqa: BLE001
                    continue
                if cfg.pdf:
                    f = lambda: vndf.vndf_sample_cap_pdf(*ins, *out)  # noqa: E731
                else:
                    f = lambda: vndf.vndf_sample_cap(*ins, *out)  # noqa: E731
                ms = timed(f)
                emit(what=f"c{cid}", vw=vw, block=bs, bpsm=bpsm, ms=ms, gb_s=bps * cfg.n / ms / 1e6)
    vndf.vndf_set_launch_config(0, 0, 0)
    del x, ins, out
    torch.cuda.empty_cache()

# fused Philox
for bs in (256, 128):
    for bpsm in (0, -1):
        vndf.vndf_set_launch_config(0, bs, bpsm)
        n = 1 << 28
        o = vndf.empty_outputs(n, dev)
        ms = timed(lambda: vndf.vndf_sample_cap_philox(3, 0, n, *o), reps=5, warm=2)
        ms2 = timed(lambda: vndf.vndf_sample_heitz2018_philox(3, 0, n, *o), reps=5, warm=2)
        emit(what="c4_2^28", block=bs, bpsm=bpsm, cap_gs=n / ms / 1e6, heitz_gs=n / ms2 / 1e6)
vndf.vndf_set_launch_config(0, 0, 0)

# host path pieces
cfg = synth.CONFIGS[2]
n = cfg.n
x = synth.fill(cfg.recipe, cfg.seed, n, device=dev)
hin = [x[k].cpu().pin_memory() for k in synth.PLANES]
hout = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(4)]
d = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(7)]
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(7):
    d[k].copy_(hin[k], non_blocking=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
emit(what="torch_h2d_pinned_7planes", gb_s=28 * n / (t1 - t0) / 1e9, s=t1 - t0)
t0 = time.perf_counter()
for k in range(4):
    hout[k].copy_(d[k], non_blocking=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
emit(what="torch_d2h_pinned_4planes", gb_s=16 * n / (t1 - t0) / 1e9, s=t1 - t0)
for rep in range(4):
    t0 = time.perf_counter()
    vndf.vndf_sample_cap_pdf_host(*hin, *hout)
    t1 = time.perf_counter()
    emit(what="host_api", rep=rep, s=t1 - t0, gsamples_s=n / (t1 - t0) / 1e9)
