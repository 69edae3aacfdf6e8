"""Time the streamed cap/Heitz kernels (configs 2, 3, 5) for several builds of libvndf.

python tools/stream_variants.py lib1.so lib2.so ...
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402

dev = torch.device("cuda:0")
data = {}
for cid in (2, 3, 5):
    cfg = synth.CONFIGS[cid]
    x = synth.fill(cfg.recipe, cfg.seed, cfg.n, device=dev)
    out = [torch.empty(cfg.n, device=dev) for _ in range(4)]
    data[cid] = (cfg, [x[k] for k in synth.PLANES], out)
for path in sys.argv[1:]:
    L = ctypes.CDLL(os.path.abspath(path))
    for fn in ("vndf_sample_cap_pdf", "vndf_sample_heitz2018"):
        getattr(L, fn).argtypes = [ctypes.c_void_p] * 11 + [ctypes.c_int64, ctypes.c_void_p]
    L.vndf_sample_cap.argtypes = [ctypes.c_void_p] * 10 + [ctypes.c_int64, ctypes.c_void_p]
    res = {"lib": os.path.basename(path)}
    for cid, (cfg, ins, out) in data.items():
        P = [ctypes.c_void_p(t.data_ptr()) for t in ins]
        Q = [ctypes.c_void_p(t.data_ptr()) for t in out]
        for name, f, args in (("cap", L.vndf_sample_cap_pdf if cfg.pdf else L.vndf_sample_cap,
                               P + (Q if cfg.pdf else Q[:3])),
                              ("heitz", L.vndf_sample_heitz2018, P + Q[:3] + [Q[3] if cfg.pdf else None])):
            reps = 50 if cid != 3 else 10
            for _ in range(5):
                f(*args, cfg.n, None)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                f(*args, cfg.n, None)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            res[f"c{cid}_{name}_gbs"] = round((44 if cfg.pdf else 40) * cfg.n / ms / 1e6, 1)
    print(json.dumps(res), flush=True)
