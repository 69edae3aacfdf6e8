"""Time per call of the config-2 cap kernel over ~4 s of back-to-back calls,
in batches of 20, with the SM and memory clocks (NVML) beside each batch:
shows the device settling from a slower to a faster state.

python tools/state_probe.py
"""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import pynvml  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
dev = torch.device("cuda:0")
cfg = synth.CONFIGS[2]
x = synth.fill(cfg.recipe, cfg.seed, cfg.n, device=dev)
out = [torch.empty(cfg.n, device=dev) for _ in range(4)]
L = ctypes.CDLL(os.path.join(ROOT, "paper_2306_05044_b200", "libvndf.so"))
L.vndf_sample_cap_pdf.argtypes = [ctypes.c_void_p] * 11 + [ctypes.c_int64, ctypes.c_void_p]
P = [ctypes.c_void_p(x[k].data_ptr()) for k in synth.PLANES] + [ctypes.c_void_p(t.data_ptr()) for t in out]
t0 = time.perf_counter()
batch = 0
while time.perf_counter() - t0 < 4.0:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        L.vndf_sample_cap_pdf(*P, cfg.n, None)
    b.record()
    torch.cuda.synchronize()
    if batch % 10 == 0:
        print(json.dumps({"t_s": round(time.perf_counter() - t0, 3), "us_per_call": round(a.elapsed_time(b) * 50, 2),
                          "sm_mhz": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                          "mem_mhz": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                          "power_w": round(pynvml.nvmlDeviceGetPowerUsage(h) / 1000, 1),
                          "temp_c": pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU)}), flush=True)
    batch += 1
