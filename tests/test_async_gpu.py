"""vndf.h behaviour contract on the GPU: calls only enqueue (no implicit
synchronisation), honour the caller's stream, and are thread-safe."""
import threading
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2306_05044_b200 as vndf
    import synth
    return vndf, synth, torch.device("cuda:0")


def test_calls_do_not_synchronise(env):
    vndf, synth, dev = env
    n = 1 << 30
    out = vndf.empty_outputs(n, dev)
    s = torch.cuda.Stream(dev)
    vndf.vndf_sample_cap_philox(3, 0, n, *out, stream=s)         # warm: table, pool growth, attributes
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    vndf.vndf_sample_cap_philox(3, 0, n, *out, stream=s)         # ~6 ms of GPU work
    dt = time.perf_counter() - t0
    pending = not s.query()
    s.synchronize()
    assert pending, "the call returned after the work had finished: it synchronised"
    assert dt < 2e-3, dt
    del out


def test_stream_ordering(env):
    """Inputs produced on a side stream and consumed there: results match the
    default-stream run (the library launches on the stream it is given)."""
    vndf, synth, dev = env
    n = (1 << 22) + 3
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        x = synth.fill(2, 1, n, device=dev, stream=s)
        a = vndf.empty_outputs(n, dev)
        vndf.vndf_sample_cap_pdf(*[x[k] for k in synth.PLANES], *a, stream=s)
    s.synchronize()
    y = synth.fill(2, 1, n, device=dev)
    b = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_pdf(*[y[k] for k in synth.PLANES], *b)
    torch.cuda.synchronize()
    for u, v in zip(a, b):
        assert torch.equal(u, v)


def test_thread_safety(env):
    """Eight host threads, each with its own stream, call the streamed, fused and
    host entry points concurrently; every result equals the single-thread one."""
    vndf, synth, dev = env
    n = (1 << 20) + 11
    x = synth.fill(5, 4, n, device=dev)
    ins = [x[k] for k in synth.PLANES]
    ref = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_pdf(*ins, *ref)
    refp = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_philox(9, 5, n, *refp)
    hin = [t.cpu().pin_memory() for t in ins]
    torch.cuda.synchronize()
    errors = []

    def work(k):
        try:
            torch.cuda.set_device(dev)
            s = torch.cuda.Stream(dev)
            with torch.cuda.stream(s):
                for _ in range(3):
                    o = vndf.empty_outputs(n, dev)
                    vndf.vndf_sample_cap_pdf(*ins, *o, stream=s)
                    p = vndf.empty_outputs(n, dev)
                    vndf.vndf_sample_cap_philox(9, 5, n, *p, stream=s)
                    s.synchronize()
                    for u, v in zip(o, ref):
                        assert torch.equal(u, v)
                    for u, v in zip(p, refp):
                        assert torch.equal(u, v)
                    if k % 2 == 0:
                        hout = [torch.empty(n) for _ in range(4)]
                        vndf.vndf_sample_cap_pdf_host(*hin, *hout, stream=s)
                        for u, v in zip(hout, ref):
                            assert torch.equal(u, v.cpu())
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    th = [threading.Thread(target=work, args=(k,)) for k in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors[:3]
