"""Both host paths of each end-to-end entry point (vndf.cu zero_copy_allowed):
by default vndf_sample_cap_pdf_host runs zero-copy on mapped pinned buffers and
vndf_sample_cap_philox_host stages 2 Mi-sample chunks through device memory with
DMA copies (measured faster for each, tools/e2e_c4_probe.py); the test hook
VNDF_HOST_ZERO_COPY=0 / =1 forces the other path.  Every path must be
bit-identical to the device entry points."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_RUN = r"""
import sys, numpy as np, torch
sys.path.insert(0, ROOT)
import paper_2306_05044_b200 as vndf, synth
dev = torch.device("cuda:0")
n = (1 << 22) + 2 ** 21 + 13
x = synth.fill(5, 4, n, device=dev)
hx = {k: v.cpu().pin_memory() for k, v in x.items()}
h = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(4)]
vndf.vndf_sample_cap_pdf_host(*[hx[k] for k in synth.PLANES], *h)
p = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(4)]
vndf.vndf_sample_cap_philox_host(3, 2**32 - 1000, n, *p)
np.savez(OUT, *[t.numpy() for t in h + p])
"""


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2306_05044_b200 as vndf
    import synth
    return vndf, synth, torch.device("cuda:0")


def _run(tmp_path, mode):
    out = str(tmp_path / f"host_{mode}.npz")
    e = dict(os.environ)
    e.pop("VNDF_HOST_ZERO_COPY", None)
    if mode is not None:
        e["VNDF_HOST_ZERO_COPY"] = mode
    r = subprocess.run([sys.executable, "-c", _RUN.replace("ROOT", repr(ROOT)).replace("OUT", repr(out))],
                       env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    z = np.load(out)
    return [z[f"arr_{k}"] for k in range(8)]


def test_every_host_path_bit_identical_to_device(env, tmp_path):
    vndf, synth, dev = env
    n = (1 << 22) + 2 ** 21 + 13
    x = synth.fill(5, 4, n, device=dev)
    d = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_pdf(*[x[k] for k in synth.PLANES], *d)
    q = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_philox(3, 2**32 - 1000, n, *q)
    ref = [t.cpu().numpy() for t in list(d) + list(q)]
    for mode in (None, "0", "1"):
        got = _run(tmp_path, mode)
        for k, (a, b) in enumerate(zip(ref, got)):
            np.testing.assert_array_equal(a, b, err_msg=f"mode {mode} output {k}")
