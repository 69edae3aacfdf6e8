"""Host cost of one Python-binding call (argument checks + ctypes + launch):
wall time per call of 2000 back-to-back tiny launches (n = 1024), against the
same launches made through ctypes directly with pre-built arguments.

python tools/binding_overhead.py
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_05044_b200 as vndf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
n = 1024
x = synth.fill(2, 1, n, device=dev)
ins = [x[k] for k in synth.PLANES]
out = vndf.empty_outputs(n, dev)
K = 2000


def per_call(f):
    for _ in range(50):
        f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(K):
            f()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) / K)
    return best * 1e6


L = vndf.lib()
P = [ctypes.c_void_p(t.data_ptr()) for t in ins + list(out)]
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
raw = per_call(lambda: L.vndf_sample_cap_pdf(*P, n, s))
py = per_call(lambda: vndf.vndf_sample_cap_pdf(*ins, *out))
print(f"ctypes direct: {raw:.2f} us/call; binding: {py:.2f} us/call; binding overhead {py - raw:.2f} us")
