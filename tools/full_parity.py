"""Exhaustive parity run: EVERY sample of every BASELINE config (C1-C5, the
fused C4 at its full 2^30, and C5 in the native frame) against the float64
oracle, in chunks of 2^24 so host memory stays bounded.  The pytest suite
compares full ranges up to 2^24 and sampled indices beyond; this one-off run
(a few minutes on the GPU box) closes the gap.

python tools/full_parity.py > profiles/r2/full_parity_r2.txt
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2306_05044_b200 as vndf  # noqa: E402
import synth  # noqa: E402

TOL_H, TOL_PDF = 2e-5, 1e-4
CHUNK = 1 << 24
dev = torch.device("cuda:0")


def report(label, n, eh, ep, bad, t0):
    pdf = f"{ep:.2e}" if ep is not None else "  (h only)"
    print(f"{label:34s} n={n:>11d}  max|dh| {eh:.2e}  max pdf rel {pdf}  "
          f"over tolerance {bad}  ({time.time() - t0:.0f} s)", flush=True)


def streamed(cid, native=False, fused_edge=False):
    """fused_edge: config 5 through vndf_sample_cap_philox_edge (inputs generated
    in-kernel), checked against the oracle on the recipe's planes."""
    cfg = synth.CONFIGS[cid]
    n = cfg.n if not native else CHUNK  # the native oracle runs binary128, single-threaded: a 2^24 prefix
    t0 = time.time()
    x = synth.fill(cfg.recipe, cfg.seed, n, device=dev)
    out = vndf.empty_outputs(n, dev, pdf=cfg.pdf or native)
    ins = [x[k] for k in synth.PLANES]
    if fused_edge:
        vndf.vndf_sample_cap_philox_edge(cfg.seed, 0, n, *out)
    elif native:
        vndf.vndf_sample_cap_pdf_native(*ins, *out)
    elif cfg.pdf:
        vndf.vndf_sample_cap_pdf(*ins, *out)
    else:
        vndf.vndf_sample_cap(*ins, *out)
    # (a full-size launch, checked chunk by chunk)
    torch.cuda.synchronize()
    eh = ep = 0.0
    bad = 0
    for lo in range(0, n, CHUNK):
        hi = min(n, lo + CHUNK)
        host = [x[k][lo:hi].cpu().numpy() for k in synth.PLANES]
        if native:
            h_ref, p_ref = oracle.batch_sample_native(oracle.CAP, *host)
        else:
            h_ref, p_ref, _ = oracle.batch_sample(oracle.CAP, *host, pdf=cfg.pdf)
        h = np.stack([o[lo:hi].cpu().numpy() for o in out[:3]]).astype(np.float64)
        e = np.abs(h - h_ref).max(axis=0)
        over = e > TOL_H
        eh = max(eh, float(e.max()))
        if p_ref is not None:
            p = out[3][lo:hi].cpu().numpy().astype(np.float64)
            r = np.abs(p - p_ref) / p_ref
            ep = max(ep, float(r.max()))
            over |= r > TOL_PDF
        bad += int(over.sum())
    report(f"config {cid}{' native (2^24 prefix)' if native else ''}{' fused edge' if fused_edge else ''}", n, eh,
           ep if (cfg.pdf or native) else None, bad, t0)
    del x, out


def fused():
    cfg = synth.CONFIGS[4]
    t0 = time.time()
    out = vndf.empty_outputs(cfg.n, dev)
    vndf.vndf_sample_cap_philox(cfg.seed, 0, cfg.n, *out)
    torch.cuda.synchronize()
    eh = ep = 0.0
    bad = 0
    for lo in range(0, cfg.n, CHUNK):
        hi = min(cfg.n, lo + CHUNK)
        h_ref, p_ref, _ = oracle.batch_sample_philox(oracle.CAP, cfg.seed, np.arange(lo, hi, dtype=np.uint64))
        h = np.stack([o[lo:hi].cpu().numpy() for o in out[:3]]).astype(np.float64)
        p = out[3][lo:hi].cpu().numpy().astype(np.float64)
        e = np.abs(h - h_ref).max(axis=0)
        r = np.abs(p - p_ref) / p_ref
        eh, ep = max(eh, float(e.max())), max(ep, float(r.max()))
        bad += int(((e > TOL_H) | (r > TOL_PDF)).sum())
    report("config 4 (fused Philox)", cfg.n, eh, ep, bad, t0)


TOL_WO, TOL_W = 6e-5, 1e-4  # reflection (DESIGN.md s.6.5)


def reflect(cid):
    cfg = synth.CONFIGS[cid]
    t0 = time.time()
    x = synth.fill(cfg.recipe, cfg.seed, cfg.n, device=dev)
    out = [torch.empty(cfg.n, device=dev) for _ in range(5)]
    vndf.vndf_sample_cap_reflect(*[x[k] for k in synth.PLANES], *out)
    torch.cuda.synchronize()
    _reflect_check(f"reflect, config {cid}", cfg.n, out,
                   lambda lo, hi: oracle.batch_sample_reflect(oracle.CAP, *[x[k][lo:hi].cpu().numpy() for k in synth.PLANES]), t0)
    del x, out


def reflect_fused(n=1 << 28):
    t0 = time.time()
    out = [torch.empty(n, device=dev) for _ in range(5)]
    vndf.vndf_sample_cap_reflect_philox(3, 0, n, *out)
    torch.cuda.synchronize()
    _reflect_check("reflect, fused Philox (2^28)", n, out,
                   lambda lo, hi: oracle.batch_sample_reflect_philox(oracle.CAP, 3, np.arange(lo, hi, dtype=np.uint64)), t0)
    del out


def _reflect_check(label, n, out, ref_fn, t0):
    ewo = epd = ewt = 0.0
    bad = 0
    for lo in range(0, n, CHUNK):
        hi = min(n, lo + CHUNK)
        ref = ref_fn(lo, hi)
        got = np.stack([o[lo:hi].cpu().numpy() for o in out]).astype(np.float64)
        a = np.abs(got[:3] - ref[:3]).max(axis=0)
        b = np.abs(got[3] - ref[3]) / ref[3]
        c = np.abs(got[4] - ref[4])
        ewo, epd, ewt = max(ewo, float(a.max())), max(epd, float(b.max())), max(ewt, float(c.max()))
        bad += int(((a > TOL_WO) | (b > TOL_PDF) | (c > TOL_W)).sum())
    print(f"{label:34s} n={n:>11d}  max|dwo| {ewo:.2e}  max pdf rel {epd:.2e}  max|dweight| {ewt:.2e}  "
          f"over tolerance {bad}  ({time.time() - t0:.0f} s)", flush=True)


print(f"# every sample against the float64 oracle; tolerances |dh| <= {TOL_H}, pdf rel <= {TOL_PDF}"
      f" (reflection: |dwo| <= {TOL_WO}, pdf rel <= {TOL_PDF}, |dweight| <= {TOL_W})")
for cid in (1, 2, 3, 5):
    streamed(cid)
streamed(5, native=True)
streamed(5, fused_edge=True)
fused()
reflect(2)
reflect(5)
reflect_fused()
