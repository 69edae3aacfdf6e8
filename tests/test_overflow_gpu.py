"""Fix-up queue overflow paths of the fused kernels (vndf.cu test hooks
VNDF_DEBUG_FIXUP_CAP and VNDF_DEBUG_BLOCK_QUEUE): with the global queue shrunk
to one entry the fix-up kernel rescans every flag; with only the shared-memory
block queues shrunk, the overflowing samples go to the global queue directly.
Results must be bit-identical to the normal path (which the parity tests hold
against the oracle).  The streamed kernels (fix-ups in the flagged thread, no
queue) are run too, as a control."""
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
n = (1 << 20) + 3
x = synth.fill(5, 4, n, device=dev)
o = vndf.empty_outputs(n, dev)
vndf.vndf_sample_cap_pdf(*[x[k] for k in synth.PLANES], *o)
p = vndf.empty_outputs(n, dev)
vndf.vndf_sample_cap_philox(3, 5, n, *p)
r = [torch.empty(n, device=dev) for _ in range(5)]
vndf.vndf_sample_cap_reflect_philox(3, 5, n, *r)
e = vndf.empty_outputs(n, dev)
vndf.vndf_sample_cap_philox_edge(4, 5, n, *e)
torch.cuda.synchronize()
np.savez(OUT, *[t.cpu().numpy() for t in list(o) + list(p) + r + list(e)])
"""


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    return True


def _run(tmp_path, cap, block_cap=0):
    out = str(tmp_path / f"out_{cap}_{block_cap}.npz")
    env = dict(os.environ)
    env.pop("VNDF_DEBUG_FIXUP_CAP", None)
    env.pop("VNDF_DEBUG_BLOCK_QUEUE", None)
    if cap:
        env["VNDF_DEBUG_FIXUP_CAP"] = str(cap)
    if block_cap:
        env["VNDF_DEBUG_BLOCK_QUEUE"] = str(block_cap)
    code = _RUN.replace("ROOT", repr(ROOT)).replace("OUT", repr(out))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    z = np.load(out)
    return [z[f"arr_{k}"] for k in range(len(z.files))]


def test_overflow_paths_bit_identical(env, tmp_path):
    normal = _run(tmp_path, 0)
    tiny = _run(tmp_path, 1)
    assert len(normal) == len(tiny) == 17
    for k, (a, b) in enumerate(zip(normal, tiny)):
        np.testing.assert_array_equal(a, b, err_msg=f"output {k}")


def test_block_queue_overflow_bit_identical(env, tmp_path):
    normal = _run(tmp_path, 0)
    small = _run(tmp_path, 0, block_cap=1)
    for k, (a, b) in enumerate(zip(normal, small)):
        np.testing.assert_array_equal(a, b, err_msg=f"output {k}")
