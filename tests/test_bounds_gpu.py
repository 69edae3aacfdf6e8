"""Out-of-bounds write check for every entry point (compute-sanitizer is not
available on this pool): outputs live inside NaN-pattern guard bands of 64
floats on both sides; after the call the guards must be bit-identical and the
outputs fully written.  Ragged sizes and all three vector paths."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

G = 64
SENT = float(np.frombuffer(np.uint32(0x7FC0DEAD).tobytes(), dtype=np.float32)[0])


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2306_05044_b200 as vndf
    import synth
    return vndf, synth, torch.device("cuda:0")


def guarded(n, off, dev, k):
    bufs = [torch.full((n + 2 * G + 8,), SENT, dtype=torch.float32, device=dev) for _ in range(k)]
    return bufs, [b[G + off:G + off + n] for b in bufs]


def check(bufs, n, off):
    for b in bufs:
        h = b.cpu().numpy().view(np.uint32)
        assert np.all(h[:G + off] == 0x7FC0DEAD), "write before the output"
        assert np.all(h[G + off + n:] == 0x7FC0DEAD), "write after the output"
        assert not np.any(h[G + off:G + off + n] == 0x7FC0DEAD), "output element not written"


@pytest.mark.parametrize("n", [1, 9, 4099, 65541, (1 << 20) + 3])
@pytest.mark.parametrize("off", [0, 4, 1])
def test_guard_bands(env, n, off):
    vndf, synth, dev = env
    x = synth.fill(5, 4, n, device=dev)
    ins = []
    for k in synth.PLANES:
        b = torch.zeros(n + 16, device=dev)
        b[off:off + n] = x[k]
        ins.append(b[off:off + n])
    calls = [
        (4, lambda o: vndf.vndf_sample_cap_pdf(*ins, *o)),
        (3, lambda o: vndf.vndf_sample_cap(*ins, *o)),
        (4, lambda o: vndf.vndf_sample_heitz2018(*ins, *o)),
        (5, lambda o: vndf.vndf_sample_cap_reflect(*ins, *o)),
        (4, lambda o: vndf.vndf_sample_cap_philox(3, 2**32 - 3, n, *o)),
        (4, lambda o: vndf.vndf_sample_heitz2018_philox(3, 11, n, *o)),
        (1, lambda o: vndf.vndf_pdf(*ins[:3], *ins[:3], ins[3], ins[4], o[0])),
        (4, lambda o: vndf.vndf_sample_cap_pdf_native(*ins, *o)),
        (4, lambda o: vndf.vndf_sample_cap_philox_edge(4, 5, n, *o)),
        (4, lambda o: vndf.vndf_sample_heitz2018_philox_edge(4, 0, n, *o)),
        (5, lambda o: vndf.vndf_sample_cap_reflect_philox(3, 2, n, *o)),
    ]
    for k, fn in calls:
        bufs, outs = guarded(n, off, dev, k)
        fn(outs)
        torch.cuda.synchronize()
        check(bufs, n, off)
