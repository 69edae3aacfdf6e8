"""CUDA-graph capture of the C-ABI calls (vndf.h: every device entry point only
enqueues stream-ordered work): the streamed, fused and reflection calls
captured into one torch.cuda.CUDAGraph and replayed give the eager results
bit for bit, and a replay after the inputs change recomputes."""
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


def test_capture_and_replay(env):
    vndf, synth, dev = env
    n = (1 << 20) + 5
    x = synth.fill(5, 4, n, device=dev)
    ins = [x[k] for k in synth.PLANES]
    # eager references (also the warm-up: device caches are filled outside capture)
    ref_s = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_pdf(*ins, *ref_s)
    ref_p = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_philox(3, 7, n, *ref_p)
    ref_r = [torch.empty(n, device=dev) for _ in range(5)]
    vndf.vndf_sample_cap_reflect_philox(3, 7, n, *ref_r)
    torch.cuda.synchronize()

    out_s = vndf.empty_outputs(n, dev)
    out_p = vndf.empty_outputs(n, dev)
    out_r = [torch.empty(n, device=dev) for _ in range(5)]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        vndf.vndf_sample_cap_pdf(*ins, *out_s)
        vndf.vndf_sample_cap_philox(3, 7, n, *out_p)
        vndf.vndf_sample_cap_reflect_philox(3, 7, n, *out_r)
    for t in out_s + out_p + tuple(out_r):
        t.zero_()
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(out_s + out_p + tuple(out_r), ref_s + ref_p + tuple(ref_r)):
        assert torch.equal(a, b)
    # new inputs in the captured buffers -> the replay recomputes
    y = synth.fill(2, 1, n, device=dev)
    for k in synth.PLANES:
        x[k].copy_(y[k])
    g.replay()
    ref2 = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_pdf(*[y[k] for k in synth.PLANES], *ref2)
    torch.cuda.synchronize()
    for a, b in zip(out_s, ref2):
        assert torch.equal(a, b)
