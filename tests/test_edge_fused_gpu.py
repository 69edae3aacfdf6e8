"""Fused config-5 kernels (vndf_sample_cap_philox_edge / _heitz2018_philox_edge):
the edge-mix inputs (grazing, below-horizon and upper incidence, u = 0 and rim
injections; BASELINE config 5, DESIGN.md s.5) generated in-kernel from the
sample's Philox words.  They must be, bit for bit, the fp32 inputs of the
config-5 recipe, so the fused outputs equal the streamed kernels' outputs on
the planes synth/ generates for the same seed and indices (whose parity with
the float64 oracle test_parity_gpu.py holds); and the full 2^26-sample
configuration is checked against the oracle at sampled indices."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_H, TOL_PDF = 2e-5, 1e-4


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import oracle
    import paper_2306_05044_b200 as vndf
    import synth
    oracle.build()
    return oracle, vndf, synth, torch.device("cuda:0")


@pytest.mark.parametrize("first,n", [(0, (1 << 20) + 5), (12345, (1 << 18) + 77), ((1 << 32) - 4096, 8192 + 3)])
def test_edge_fused_equals_streamed_on_recipe_planes(env, first, n):
    _, vndf, synth, dev = env
    x = synth.fill(5, 4, n, first=first, device=dev)
    ins = [x[k] for k in synth.PLANES]
    for fused, streamed in ((vndf.vndf_sample_cap_philox_edge, vndf.vndf_sample_cap_pdf),
                            (vndf.vndf_sample_heitz2018_philox_edge, vndf.vndf_sample_heitz2018)):
        a = vndf.empty_outputs(n, dev)
        b = vndf.empty_outputs(n, dev)
        fused(4, first, n, *a)
        streamed(*ins, *b)
        torch.cuda.synchronize()
        for k, (p, q) in enumerate(zip(a, b)):
            assert torch.equal(p, q), (fused.__name__, k, int((p != q).sum()))


def test_edge_fused_h_only_matches(env):
    _, vndf, synth, dev = env
    n = (1 << 16) + 9
    a = vndf.empty_outputs(n, dev)
    b = vndf.empty_outputs(n, dev, pdf=False)
    vndf.vndf_sample_cap_philox_edge(4, 0, n, *a)
    vndf.vndf_sample_cap_philox_edge(4, 0, n, *b)
    torch.cuda.synchronize()
    for p, q in zip(a[:3], b):
        assert torch.equal(p, q)


def test_edge_fused_full_size_sampled(env):
    """Config 5 at its full 2^26 samples, the fused kernel, 2^18 sampled indices
    (plus both ends) against the float64 oracle on the recipe's fp32 inputs."""
    oracle, vndf, synth, dev = env
    n = synth.CONFIGS[5].n
    out = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_philox_edge(4, 0, n, *out)
    rng = np.random.default_rng(55)
    idx = np.unique(np.concatenate([rng.integers(0, n, 1 << 18), np.arange(2048), np.arange(n - 2048, n)]))
    # the recipe's inputs at those indices: contiguous windows of the generator
    ti = torch.from_numpy(idx).to(dev)
    x = synth.fill(5, 4, n, device=dev)
    host = [x[k][ti].cpu().numpy() for k in synth.PLANES]
    del x
    h_ref, p_ref, _ = oracle.batch_sample(oracle.CAP, *host, pdf=True)
    hg = np.stack([o[ti].cpu().numpy() for o in out[:3]]).astype(np.float64)
    pg = out[3][ti].cpu().numpy().astype(np.float64)
    eh = np.abs(hg - h_ref).max(axis=0)
    ep = np.abs(pg - p_ref) / p_ref
    assert eh.max() <= TOL_H, float(eh.max())
    assert ep.max() <= TOL_PDF, float(ep.max())
    # the recipe really is the edge mix: grazing, back-side and upper incidence present
    wz = host[2]
    assert (wz < 0).mean() > 0.15 and ((wz > 0) & (wz <= 0.05)).mean() > 0.3
