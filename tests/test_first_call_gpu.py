"""vndf.h: every device call only enqueues stream-ordered work -- including the
FIRST call of a process, which builds the library's per-device state (cached
attributes, the fix-up queue's memory pool).  Each case runs in a fresh
interpreter so that it really is the first call."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PRELUDE = f"""
import sys, time
sys.path.insert(0, {ROOT!r})
import torch
import paper_2306_05044_b200 as vndf
torch.cuda.init()
dev = torch.device("cuda:0")
"""


def _run(code: str):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    r = subprocess.run([sys.executable, "-c", PRELUDE + code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    return r.stdout


def test_first_fused_call_is_graph_capturable():
    out = _run("""
n = (1 << 20) + 5
outs = [vndf.empty_outputs(n, dev) for _ in range(2)]
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):                      # the process's first libvndf call
    vndf.vndf_sample_cap_philox(3, 7, n, *outs[0])
    vndf.vndf_sample_heitz2018_philox(3, 7, n, *outs[1])
g.replay()
torch.cuda.synchronize()
ref = [vndf.empty_outputs(n, dev) for _ in range(2)]
vndf.vndf_sample_cap_philox(3, 7, n, *ref[0])
vndf.vndf_sample_heitz2018_philox(3, 7, n, *ref[1])
torch.cuda.synchronize()
assert all(torch.equal(a, b) for o, r in zip(outs, ref) for a, b in zip(o, r))
print("ok")
""")
    assert "ok" in out


def test_first_fused_call_does_not_synchronise():
    """After vndf_init (the CUDA runtime's start-up inside the library, which
    waits for queued device work), the first fused call -- which in round 1
    uploaded a table synchronously -- creates the queue pool and launches
    without waiting."""
    out = _run("""
n = 1 << 24
o = vndf.empty_outputs(n, dev)
s = torch.cuda.Stream(dev)
vndf.vndf_init()
with torch.cuda.stream(s):
    torch.cuda._sleep(2_000_000_000)          # ~1 s of GPU time ahead of the call
t0 = time.perf_counter()
vndf.vndf_sample_cap_philox(3, 0, n, *o, stream=s)   # first call: builds device state
dt = time.perf_counter() - t0
pending = not s.query()
s.synchronize()
print("first call host time", dt)
assert pending, "the first call waited for the stream"
assert dt < 0.5, dt
print("ok")
""")
    assert "ok" in out


def test_calls_follow_the_stream_device():
    """A call runs on the device of its stream even when another device is
    current: tensors on cuda:1 while cuda:0 is current."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two CUDA devices")
    out = _run("""
d1 = torch.device("cuda:1")
torch.cuda.set_device(0)
n = (1 << 20) + 3
a = vndf.empty_outputs(n, d1)
vndf.vndf_sample_cap_philox(3, 0, n, *a)
torch.cuda.set_device(1)
b = vndf.empty_outputs(n, d1)
vndf.vndf_sample_cap_philox(3, 0, n, *b)
torch.cuda.synchronize(d1)
assert all(torch.equal(x, y) for x, y in zip(a, b))
print("ok")
""")
    assert "ok" in out
