"""Degenerate and extreme inputs (SURVEY 8(b) domain; vndf.h), against the
float64 oracle, and sizes beyond 2^31 samples (64-bit indexing)."""
import itertools

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
    return oracle, vndf, synth, torch.device("cuda:0")


def _grid():
    dirs = [(0, 0, 1), (0, 0, -1), (1, 0, 0), (0, 1, 0), (1, 0, -0.0), (0.6, 0.8, 0.0),
            (0.6, 0.8, -0.0), (1e-7, 0, 1), (0.3, -0.4, 1e-6), (0.3, -0.4, -1e-6),
            (0.5, 0.5, 0.7071068), (-0.5, 0.5, -0.7071068), (2.0, 0.0, 0.5), (0.01, 0.02, -0.03)]
    alphas = [(1, 1), (1e-3, 1e-3), (1e-4, 1e-4), (1e-3, 1), (1, 1e-3), (0.5, 0.5), (0.05, 0.3)]
    us = [(0.0, 0.0), (0.0, 0.5), (0.5, 0.0), (0.25, 1 - 2**-24), (1 - 2**-24, 1 - 2**-24),
          (0.123, 0.456), (2**-24, 2**-24), (0.75, 0.999)]
    rows = [(*d, *a, *u) for d, a, u in itertools.product(dirs, alphas, us)]
    return np.array(rows, dtype=np.float32).T


def test_degenerate_grid(env):
    """Pole / horizon (+0 and -0) / straight-below incidence, non-unit wi,
    alpha from 1e-4 (below the 1e-3 floor of vndf.h) to 1 in both axes, u at 0,
    the 2^-24 grid and the rim 1 - 2^-24.  Within the vndf.h domain every sample
    meets the contract; outside it (alpha = 1e-4) outputs are finite unit
    vectors."""
    oracle, vndf, synth, dev = env
    g = _grid()
    n = g.shape[1]
    t = [torch.from_numpy(np.ascontiguousarray(r)).to(dev) for r in g]
    out = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_pdf(*t, *out)
    torch.cuda.synchronize()
    h_ref, p_ref, _ = oracle.batch_sample(oracle.CAP, *g)
    h = np.stack([o.cpu().numpy() for o in out[:3]]).astype(np.float64)
    p = out[3].cpu().numpy().astype(np.float64)
    assert np.all(np.isfinite(h)) and np.all(np.isfinite(p)) and np.all(p > 0)
    assert np.abs(np.linalg.norm(h, axis=0) - 1).max() < 2e-6
    in_domain = np.minimum(g[3], g[4]) >= 1e-3
    eh = np.abs(h - h_ref).max(axis=0)
    ep = np.abs(p - p_ref) / p_ref
    assert eh[in_domain].max() <= TOL_H, float(eh[in_domain].max())
    assert ep[in_domain].max() <= TOL_PDF, float(ep[in_domain].max())
    # identity warp (alpha = 1) and the pole: closed forms hold on the GPU too
    pole = (g[0] == 0) & (g[1] == 0) & (g[2] == 1) & (g[3] == 1) & (g[4] == 1)
    u1, u2 = g[5][pole].astype(np.float64), g[6][pole].astype(np.float64)
    want = np.stack([np.sqrt(u2) * np.cos(2 * np.pi * u1), np.sqrt(u2) * np.sin(2 * np.pi * u1), np.sqrt(1 - u2)])
    np.testing.assert_allclose(h[:, pole], want, atol=TOL_H)


def test_beyond_2e31_samples(env):
    """n = 2^31 + 7: the fused kernel indexes past 32 bits; the last samples
    are compared with the oracle, and the streamed kernel over the same range
    (7 x 8.6 GB inputs) agrees at sampled indices."""
    oracle, vndf, synth, dev = env
    n = (1 << 31) + 7
    out = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(3)]
    vndf.vndf_sample_cap_philox(3, 0, n, *out)
    torch.cuda.synchronize()
    idx = np.concatenate([np.arange(n - 2048, n), np.array([0, (1 << 31) - 1, 1 << 31])]).astype(np.int64)
    ti = torch.from_numpy(idx).to(dev)
    h_ref, _, _ = oracle.batch_sample_philox(oracle.CAP, 3, idx.astype(np.uint64))
    h = np.stack([o[ti].cpu().numpy() for o in out]).astype(np.float64)
    assert np.abs(h - h_ref).max() <= TOL_H
    del out
    torch.cuda.empty_cache()
    x = synth.fill(3, 2, n, device=dev)
    o2 = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(3)]
    vndf.vndf_sample_cap(*[x[k] for k in synth.PLANES], *o2)
    torch.cuda.synchronize()
    rng = np.random.default_rng(31)
    idx = np.unique(np.concatenate([rng.integers(0, n, 1 << 16), np.arange(n - 1024, n)])).astype(np.int64)
    ti = torch.from_numpy(idx).to(dev)
    host = [x[k][ti].cpu().numpy() for k in synth.PLANES]
    h_ref, _, _ = oracle.batch_sample(oracle.CAP, *host, pdf=False)
    h = np.stack([o[ti].cpu().numpy() for o in o2]).astype(np.float64)
    assert np.abs(h - h_ref).max() <= TOL_H
    del x, o2
    torch.cuda.empty_cache()


def test_garbage_inputs_never_trap(env):
    """Outside the per-sample domain the result is unspecified but never traps
    (vndf.h): random bit patterns (NaN, inf, subnormals, negatives) through every
    streamed entry point; the CUDA context stays healthy afterwards."""
    oracle, vndf, synth, dev = env
    n = (1 << 18) + 5
    g = torch.Generator(device="cpu").manual_seed(123)
    bits = torch.randint(-2**31, 2**31 - 1, (7, n), generator=g, dtype=torch.int64).to(torch.int32)
    ins = [bits[k].view(torch.float32).to(dev) for k in range(7)]
    out = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(5)]
    vndf.vndf_sample_cap_pdf(*ins, *out[:4])
    vndf.vndf_sample_cap(*ins, *out[:3])
    vndf.vndf_sample_heitz2018(*ins, *out[:4])
    vndf.vndf_sample_cap_pdf_native(*ins, *out[:4])
    vndf.vndf_sample_cap_reflect(*ins, *out)
    vndf.vndf_pdf(*ins[:3], *ins[:3], ins[3], ins[4], out[0])
    c = torch.zeros(1, dtype=torch.int64, device=dev)
    vndf.vndf_count_fixups(*ins, c)
    torch.cuda.synchronize()
    # the context is still usable and correct
    x = synth.fill(1, 0, 4096, device=dev)
    o = vndf.empty_outputs(4096, dev)
    vndf.vndf_sample_cap_pdf(*[x[k] for k in synth.PLANES], *o)
    torch.cuda.synchronize()
    h_ref, p_ref, _ = oracle.batch_sample(oracle.CAP, *[x[k].cpu().numpy() for k in synth.PLANES])
    h = np.stack([t.cpu().numpy() for t in o[:3]]).astype(np.float64)
    assert np.abs(h - h_ref).max() <= TOL_H


@pytest.mark.parametrize("seed", [0, 1])
def test_whole_domain_random(env, seed):
    """vndf.h's whole per-sample domain at once: wi uniform over the sphere
    (both hemispheres, grazing included) with |wi| log-uniform in [0.5, 2],
    alpha_x, alpha_y independently log-uniform in [1e-3, 1], u1, u2 uniform on
    the fp32 grid of [0, 1); 2^22 samples, every one against the oracle."""
    oracle, vndf, synth, dev = env
    n = 1 << 22
    g = torch.Generator(device="cpu").manual_seed(1234 + seed)
    d = torch.randn(3, n, generator=g, dtype=torch.float64)
    d /= d.norm(dim=0, keepdim=True)
    mag = torch.exp(torch.empty(n, dtype=torch.float64).uniform_(np.log(0.5), np.log(2.0), generator=g))
    w = (d * mag).float()
    a = torch.exp(torch.empty(2, n, dtype=torch.float64).uniform_(np.log(1e-3), 0.0, generator=g)).float()
    u = (torch.randint(0, 1 << 24, (2, n), generator=g).double() * 2.0**-24).float()
    planes = [w[0], w[1], w[2], a[0], a[1], u[0], u[1]]
    t = [p.contiguous().to(dev) for p in planes]
    out = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_pdf(*t, *out)
    torch.cuda.synchronize()
    h_ref, p_ref, _ = oracle.batch_sample(oracle.CAP, *[p.numpy() for p in planes])
    h = np.stack([o.cpu().numpy() for o in out[:3]]).astype(np.float64)
    p = out[3].cpu().numpy().astype(np.float64)
    eh = np.abs(h - h_ref).max()
    ep = (np.abs(p - p_ref) / p_ref).max()
    print(f"whole domain seed {seed}: max |dh| {eh:.2e}, pdf rel {ep:.2e}")
    assert eh <= TOL_H and ep <= TOL_PDF
    # the paper's native below-horizon handling (NEXT-3) on the same inputs
    vndf.vndf_sample_cap_pdf_native(*t, *out)
    torch.cuda.synchronize()
    m = 1 << 19  # the native oracle runs binary128 (reading R17): a 2^19 prefix
    h_ref, p_ref = oracle.batch_sample_native(oracle.CAP, *[p[:m].numpy() for p in planes])
    h = np.stack([o[:m].cpu().numpy() for o in out[:3]]).astype(np.float64)
    p = out[3][:m].cpu().numpy().astype(np.float64)
    eh, ep = np.abs(h - h_ref).max(), (np.abs(p - p_ref) / p_ref).max()
    print(f"  native: max |dh| {eh:.2e}, pdf rel {ep:.2e}")
    assert eh <= TOL_H and ep <= TOL_PDF
    # reflection (NEXT-2; tolerances of DESIGN.md s.6.5)
    ro = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(5)]
    vndf.vndf_sample_cap_reflect(*t, *ro)
    torch.cuda.synchronize()
    ref = oracle.batch_sample_reflect(oracle.CAP, *[p.numpy() for p in planes])
    got = np.stack([o.cpu().numpy() for o in ro]).astype(np.float64)
    ewo = np.abs(got[:3] - ref[:3]).max()
    epd = (np.abs(got[3] - ref[3]) / ref[3]).max()
    ewt = np.abs(got[4] - ref[4]).max()
    print(f"  reflect: max |dwo| {ewo:.2e}, pdf rel {epd:.2e}, |dweight| {ewt:.2e}")
    assert ewo <= 6e-5 and epd <= 1e-4 and ewt <= 1e-4
