"""PDL probe: config-2 launches back to back, with and without per-step events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_05044_b200 as vndf  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
cfg = synth.CONFIGS[2]
x = synth.fill(cfg.recipe, cfg.seed, cfg.n, device=dev)
ins = [x[k] for k in synth.PLANES]
out = vndf.empty_outputs(cfg.n, dev)
st = torch.cuda.current_stream()


def run(K, per_step):
    for _ in range(10):
        vndf.vndf_sample_cap_pdf(*ins, *out)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    ev[0].record(st)
    for k in range(K):
        vndf.vndf_sample_cap_pdf(*ins, *out)
        if per_step:
            ev[k + 1].record(st)
    if not per_step:
        ev[K].record(st)
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[K]) / K


for per_step in (True, False):
    ms = min(run(200, per_step) for _ in range(3))
    print(f"PDL={os.environ.get('VNDF_NO_PDL', '0') != '1'} per_step_events={per_step}: "
          f"{ms * 1e3:.2f} us/step  {44 * cfg.n / ms / 1e6:.0f} GB/s")
