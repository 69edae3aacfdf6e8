"""Fraction of samples the conditioning test flags (float64 recomputation),
per config, for one or more builds of libvndf (vndf_count_fixups on the
config planes synth/ generates, vndf_count_fixups_philox for config 4).

python tools/flag_rates.py paper_2306_05044_b200/libvndf.so [var_*.so ...]
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
planes = {c: synth.fill(c, synth.CONFIGS[c].seed, synth.CONFIGS[c].n, device=dev) for c in (1, 2, 3, 5)}
for path in sys.argv[1:]:
    L = ctypes.CDLL(os.path.abspath(path))
    L.vndf_count_fixups.argtypes = [ctypes.c_void_p] * 7 + [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    L.vndf_count_fixups_philox.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p,
                                           ctypes.c_void_p]
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    res = {"lib": os.path.basename(path)}
    for c, x in planes.items():
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        n = synth.CONFIGS[c].n
        assert L.vndf_count_fixups(*[ctypes.c_void_p(x[k].data_ptr()) for k in synth.PLANES], n,
                                   ctypes.c_void_p(cnt.data_ptr()), s) == 0
        torch.cuda.synchronize()
        res[f"c{c}"] = round(int(cnt.item()) / n, 6)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    n = 1 << 28
    assert L.vndf_count_fixups_philox(3, 0, n, ctypes.c_void_p(cnt.data_ptr()), s) == 0
    torch.cuda.synchronize()
    res["c4_2^28"] = round(int(cnt.item()) / n, 6)
    print(json.dumps(res), flush=True)
