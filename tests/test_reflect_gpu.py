"""NEXT-2 on the GPU: reflection sampling (appendix steps (1)-(2))
with the Eq. 20 pdf and the G2/G1 weight, and the Eq. 19 white-furnace
estimator, against the float64 oracle.

Tolerances (DESIGN.md s.6.5): wo <= 6e-5 per component (wo = 2(w.h)h - w moves
by at most ~3x the h error), pdf relative 1e-4, weight absolute 1e-4."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_WO, TOL_PDF, TOL_W = 6e-5, 1e-4, 1e-4


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


@pytest.mark.parametrize("cid,n", [(1, 1 << 16), (2, 1 << 22), (3, 1 << 21), (5, 1 << 22), (5, 4099)])
def test_reflect_parity(env, cid, n):
    oracle, vndf, synth, dev = env
    cfg = synth.CONFIGS[cid]
    x = synth.fill(cfg.recipe, cfg.seed, n, device=dev)
    out = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(5)]
    vndf.vndf_sample_cap_reflect(*[x[k] for k in synth.PLANES], *out)
    torch.cuda.synchronize()
    ref = oracle.batch_sample_reflect(oracle.CAP, *[x[k].cpu().numpy() for k in synth.PLANES])
    got = np.stack([o.cpu().numpy() for o in out]).astype(np.float64)
    ewo = np.abs(got[:3] - ref[:3]).max(axis=0)
    epdf = np.abs(got[3] - ref[3]) / ref[3]
    ew = np.abs(got[4] - ref[4])
    print(f"config {cid}: max |dwo| {ewo.max():.2e}, pdf rel {epdf.max():.2e}, |dweight| {ew.max():.2e}")
    assert ewo.max() <= TOL_WO, float(ewo.max())
    assert epdf.max() <= TOL_PDF, float(epdf.max())
    assert ew.max() <= TOL_W, float(ew.max())
    # invariants: unit wo, mirror symmetry about h is implicit in the oracle; weights in [0, 1]
    assert np.abs(np.linalg.norm(got[:3], axis=0) - 1).max() < 1e-5
    assert got[4].min() >= 0.0 and got[4].max() <= 1.0 + 1e-6


@pytest.mark.parametrize("method", [0, 1], ids=["cap", "heitz"])
@pytest.mark.parametrize("theta,alpha", [(0, (0.1, 0.1)), (45, (0.5, 0.5)), (75, (0.3, 0.05)),
                                         (85, (0.2, 0.2)), (85, (0.02, 0.02))])
def test_furnace_gpu(env, method, theta, alpha):
    """GPU Eq. 19 estimate equals the oracle's estimate on the same Philox
    samples, and the quadrature albedo within 5 standard errors."""
    oracle, vndf, synth, dev = env
    t = np.radians(theta)
    wa = np.array([np.sin(t) * np.cos(0.35), np.sin(t) * np.sin(0.35), np.cos(t)], dtype=np.float32)
    n = 1 << 22
    sums = torch.zeros(2, dtype=torch.float64, device=dev)
    vndf.vndf_furnace(method, wa, alpha, 99, n, sums)
    torch.cuda.synchronize()
    s1, s2 = sums.cpu().numpy()
    mean = s1 / n
    var = s2 / n - mean * mean
    m = 1 << 18
    o1, _ = oracle.furnace(method, wa.astype(np.float64), *alpha, seed=99, n=m)
    sums_m = torch.zeros(2, dtype=torch.float64, device=dev)
    vndf.vndf_furnace(method, wa, alpha, 99, m, sums_m)
    torch.cuda.synchronize()
    assert abs(float(sums_m[0]) - o1) / m <= 1e-4  # per-sample weight tolerance
    if alpha == (0.02, 0.02):
        # at grazing incidence the reflected lobe is ~2 alpha cos(theta) = 3e-3 rad wide
        # in azimuth: beyond the product quadrature; the oracle-equality check above holds
        return
    dirs, w = oracle.sphere_quadrature(nz=1024, nphi=1024, upper_only=True)
    albedo = float((oracle.batch_brdf_cos(wa.astype(np.float64), *alpha, dirs) * w).sum())
    se = np.sqrt(max(var, 0) / n)
    assert abs(mean - albedo) <= 5 * se + 1e-5, (mean, albedo, se)


@pytest.mark.parametrize("theta,alpha", [(30, (0.4, 0.4)), (70, (0.3, 0.6)), (85, (0.2, 0.2))])
def test_reflect_gpu_distribution_eq20(env, theta, alpha):
    """GPU reflected directions (2^21 per seed, 3 seeds) against the Eq. 20 masses
    over the whole sphere (32 x 64 bins in (cos theta, phi))."""
    oracle, vndf, synth, dev = env
    from oracle import stats
    t = np.radians(theta)
    wa = np.array([np.sin(t) * np.cos(0.7), np.sin(t) * np.sin(0.7), np.cos(t)], dtype=np.float32)
    masses = stats.sphere_bin_masses(lambda d: oracle.batch_pdf_reflect(wa.astype(np.float64), *alpha, d))
    passes = []
    for seed in (3000, 3001, 3002):
        n = 1 << 21
        x = synth.fill(0, seed, n, device=dev, fixed=[wa[0], wa[1], wa[2], alpha[0], alpha[1]])
        out = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(5)]
        vndf.vndf_sample_cap_reflect(*[x[k] for k in synth.PLANES], *out)
        torch.cuda.synchronize()
        wo = np.stack([o.cpu().numpy() for o in out[:3]]).astype(np.float64)
        passes.append(stats.pearson(stats.sphere_histogram(wo), masses)[2] > 1e-3)
    assert sum(passes) >= 2, passes


def _reflect_errors(got, ref):
    ewo = np.abs(got[:3] - ref[:3]).max(axis=0)
    epdf = np.abs(got[3] - ref[3]) / ref[3]
    ew = np.abs(got[4] - ref[4])
    return ewo, epdf, ew


@pytest.mark.parametrize("first,n", [(0, (1 << 20) + 3), ((1 << 32) - 4097, 8192 + 5)])
def test_reflect_philox_parity(env, first, n):
    """Fused Philox reflection (config-4 inputs generated in-kernel): every
    sample against the oracle's orc_sample_reflect on orc_c4_inputs, across
    aligned / unaligned first_index and the 32-bit counter carry."""
    oracle, vndf, synth, dev = env
    out = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(5)]
    vndf.vndf_sample_cap_reflect_philox(3, first, n, *out)
    torch.cuda.synchronize()
    ref = oracle.batch_sample_reflect_philox(oracle.CAP, 3, np.arange(first, first + n, dtype=np.uint64))
    got = np.stack([o.cpu().numpy() for o in out]).astype(np.float64)
    ewo, epdf, ew = _reflect_errors(got, ref)
    print(f"philox reflect first={first}: max |dwo| {ewo.max():.2e}, pdf rel {epdf.max():.2e}, "
          f"|dweight| {ew.max():.2e}")
    assert ewo.max() <= TOL_WO and epdf.max() <= TOL_PDF and ew.max() <= TOL_W
    assert np.abs(np.linalg.norm(got[:3], axis=0) - 1).max() < 1e-5


def test_reflect_philox_full_size_sampled(env):
    """2^28 samples in one call (the bench size), 2^20 sampled indices plus the
    ends compared one by one; and the fused outputs equal the streamed kernel's
    on the same (fp32-rounded) inputs within the contract."""
    oracle, vndf, synth, dev = env
    n = 1 << 28
    out = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(5)]
    vndf.vndf_sample_cap_reflect_philox(3, 0, n, *out)
    torch.cuda.synchronize()
    rng = np.random.default_rng(28)
    idx = np.unique(np.concatenate([rng.integers(0, n, 1 << 20), np.arange(2048), np.arange(n - 2048, n)]))
    ti = torch.from_numpy(idx).to(dev)
    ref = oracle.batch_sample_reflect_philox(oracle.CAP, 3, idx.astype(np.uint64))
    got = np.stack([o[ti].cpu().numpy() for o in out]).astype(np.float64)
    ewo, epdf, ew = _reflect_errors(got, ref)
    assert ewo.max() <= TOL_WO and epdf.max() <= TOL_PDF and ew.max() <= TOL_W
    assert bool(torch.isfinite(out[3]).all()) and float(out[3].min()) > 0
    assert float(out[4].min()) >= 0.0 and float(out[4].max()) <= 1.0 + 1e-6
    del out
    torch.cuda.empty_cache()


def test_reflect_philox_offsets_and_heitz(env):
    """first_index offsets are bit-identical to slices of a first_index = 0
    call (cap and Heitz); the Heitz baseline (literal fp32, no fix-up) meets
    the contract on >= 98% of samples and keeps unit directions."""
    oracle, vndf, synth, dev = env
    n = (1 << 16) + 3
    for fn in (vndf.vndf_sample_cap_reflect_philox, vndf.vndf_sample_heitz2018_reflect_philox):
        ref = [torch.empty(n + 8, dtype=torch.float32, device=dev) for _ in range(5)]
        fn(11, 0, n + 8, *ref)
        for f in (1, 3, 4, 6):
            out = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(5)]
            fn(11, f, n, *out)
            torch.cuda.synchronize()
            for u, v in zip(out, ref):
                assert torch.equal(u, v[f:f + n]), (fn.__name__, f)
    out = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(5)]
    vndf.vndf_sample_heitz2018_reflect_philox(11, 0, n, *out)
    torch.cuda.synchronize()
    ref = oracle.batch_sample_reflect_philox(oracle.HEITZ, 11, np.arange(n, dtype=np.uint64))
    got = np.stack([o.cpu().numpy() for o in out]).astype(np.float64)
    ewo, epdf, ew = _reflect_errors(got, ref)
    ok = (ewo <= TOL_WO) & (epdf <= TOL_PDF) & (ew <= TOL_W)
    print(f"heitz philox reflect: within contract on {ok.mean():.5f} of samples")
    assert ok.mean() >= 0.98
    assert np.abs(np.linalg.norm(got[:3], axis=0) - 1).max() < 1e-4
