"""End-to-end host paths on one B200: the zero-copy kernel (outputs written by
the SMs into mapped pinned host planes) against the staged path (device staging
+ cudaMemcpyAsync DMA over three streams; forced with VNDF_HOST_ZERO_COPY=0),
for config 4 (vndf_sample_cap_philox_host, 16 B per sample device -> host) and
config 2 (vndf_sample_cap_pdf_host, 28 B in, 16 B out), next to plain pinned
copies in each direction.

python tools/e2e_c4_probe.py
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r"""
import json, sys, time, torch
sys.path.insert(0, ROOT)
import paper_2306_05044_b200 as vndf, synth
dev = torch.device("cuda:0")
res = {}
n4 = 1 << 28
h4 = [torch.empty(n4, dtype=torch.float32, pin_memory=True) for _ in range(4)]
vndf.vndf_sample_cap_philox_host(3, 0, n4, *h4)
t = time.perf_counter()
for _ in range(3):
    vndf.vndf_sample_cap_philox_host(3, 0, n4, *h4)
res["c4_gsamples_s"] = round(3 * n4 / (time.perf_counter() - t) / 1e9, 4)
del h4
n2 = 1 << 24
x = {k: v.cpu().pin_memory() for k, v in synth.fill(2, 1, n2, device=dev).items()}
h2 = [torch.empty(n2, dtype=torch.float32, pin_memory=True) for _ in range(4)]
ins = [x[k] for k in synth.PLANES]
vndf.vndf_sample_cap_pdf_host(*ins, *h2)
t = time.perf_counter()
for _ in range(5):
    vndf.vndf_sample_cap_pdf_host(*ins, *h2)
res["c2_gsamples_s"] = round(5 * n2 / (time.perf_counter() - t) / 1e9, 4)
if MEASURE_COPIES:
    d = torch.empty(1 << 28, dtype=torch.float32, device=dev)
    h = torch.empty(1 << 28, dtype=torch.float32, pin_memory=True)
    for name, fn in (("d2h_copy_gb_s", lambda: h.copy_(d)), ("h2d_copy_gb_s", lambda: d.copy_(h))):
        fn(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        res[name] = round(3 * (1 << 30) / (time.perf_counter() - t) / 1e9, 2)
print(json.dumps(res))
"""


def run(zero_copy: bool, copies: bool):
    env = dict(os.environ)
    env["VNDF_HOST_ZERO_COPY"] = "1" if zero_copy else "0"
    code = CODE.replace("ROOT", repr(ROOT)).replace("MEASURE_COPIES", repr(copies))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    if r.returncode != 0:
        sys.exit(r.stderr[-3000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


out = {"zero_copy": run(True, True), "staged_dma": run(False, False)}
print(json.dumps(out))
