"""Time the fused Philox kernels of several compiled variants of libvndf.

python tools/variants.py paper_2306_05044_b200/var_*.so
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

dev = torch.device("cuda:0")
n = 1 << 28
outs = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(4)]
ref = None
for path in sys.argv[1:]:
    L = ctypes.CDLL(os.path.abspath(path))
    for fn in ("vndf_sample_cap_philox", "vndf_sample_heitz2018_philox"):
        getattr(L, fn).argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64] + [ctypes.c_void_p] * 5
    P = [ctypes.c_void_p(t.data_ptr()) for t in outs]
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    res = {"lib": os.path.basename(path)}
    for fn in ("vndf_sample_cap_philox", "vndf_sample_heitz2018_philox"):
        f = getattr(L, fn)
        for _ in range(3):
            assert f(3, 0, n, *P, s) == 0
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            f(3, 0, n, *P, s)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        res[fn] = round(n / ms / 1e6, 2)
        if fn == "vndf_sample_cap_philox":
            chk = torch.stack([t[:: 1 << 10].clone() for t in outs])
            if ref is None:
                ref = chk
            res["same_as_first"] = bool(torch.equal(chk, ref))
    print(json.dumps(res), flush=True)
