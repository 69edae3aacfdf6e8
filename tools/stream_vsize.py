"""Streamed cap+pdf GB/s against the call size for 8- and 4-sample chunks (config-2 inputs).

python tools/stream_vsize.py
"""
import json, sys, torch
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_05044_b200 as vndf, synth
dev = torch.device("cuda:0")
x = synth.fill(2, 1, 1 << 28, device=dev)
out = vndf.empty_outputs(1 << 28, dev)
def gbs(fn, nb, reps):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return round(nb * reps / (a.elapsed_time(b) * 1e-3) / 1e9, 1)
for lg in (20, 22, 23, 24, 25, 26, 27, 28):
    n = 1 << lg
    ins = [x[k][:n] for k in synth.PLANES]; o = [t[:n] for t in out]
    res = {"log2n": lg}
    for vw, blk in ((8, 128), (4, 128), (4, 256), (8, 256)):
        vndf.vndf_set_launch_config(vw, blk, 0)
        res[f"v{vw}b{blk}"] = gbs(lambda: vndf.vndf_sample_cap_pdf(*ins, *o), 44 * n, max(5, (1 << 28) // n * 2))
    vndf.vndf_set_launch_config(0, 0, 0)
    print(json.dumps(res), flush=True)
