"""GPU parity: libvndf (through its C ABI) against the float64 oracle.

Tolerances (BASELINE.json north_star), written here once:
  spherical-cap kernels: max |dh| <= 2e-5 per component, |dpdf|/pdf <= 1e-4,
  on EVERY compared sample; Philox words bit-exact.
Inputs come from synth/ (seeded, counter-based; DESIGN.md s.5) and are copied
back to the host so both sides see identical fp32 values.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL_H = 2e-5
TOL_PDF = 1e-4


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


def _host(x, keys):
    return [x[k].cpu().numpy() for k in keys]


def _errors(h_gpu, p_gpu, h_ref, p_ref):
    h = np.stack(h_gpu).astype(np.float64)
    eh = np.abs(h - h_ref).max(axis=0)
    ep = None
    if p_gpu is not None:
        ep = np.abs(p_gpu.astype(np.float64) - p_ref) / p_ref
    return eh, ep


def _stream_run(vndf, x, keys, pdf=True, kernel="cap", stream=None):
    n = x["wi_x"].numel()
    dev = x["wi_x"].device
    out = vndf.empty_outputs(n, dev, pdf=pdf)
    ins = [x[k] for k in keys]
    if kernel == "cap":
        if pdf:
            vndf.vndf_sample_cap_pdf(*ins, *out, stream=stream)
        else:
            vndf.vndf_sample_cap(*ins, *out, stream=stream)
    else:
        vndf.vndf_sample_heitz2018(*ins, *out[:3], out[3] if pdf else None, stream=stream)
    torch.cuda.synchronize()
    return out


def _check_full(env, cid, n=None):
    oracle, vndf, synth, dev = env
    cfg = synth.CONFIGS[cid]
    n = n or cfg.n
    x = synth.fill(cfg.recipe, cfg.seed, n, device=dev)
    out = _stream_run(vndf, x, synth.PLANES, pdf=cfg.pdf)
    host = _host(x, synth.PLANES)
    h_ref, p_ref, _ = oracle.batch_sample(oracle.CAP, *host, pdf=cfg.pdf)
    hg = [o.cpu().numpy() for o in out[:3]]
    pg = out[3].cpu().numpy() if cfg.pdf else None
    eh, ep = _errors(hg, pg, h_ref, p_ref)
    bad = np.flatnonzero(eh > TOL_H)
    assert bad.size == 0, (cid, bad.size, float(eh.max()), [float(host[k][bad[0]]) for k in range(7)])
    if cfg.pdf:
        badp = np.flatnonzero(ep > TOL_PDF)
        assert badp.size == 0, (cid, badp.size, float(ep.max()), [float(host[k][badp[0]]) for k in range(7)])
    return float(eh.max()), (float(ep.max()) if ep is not None else None)


def test_config1_full(env):
    _check_full(env, 1)


def test_config2_full(env):
    _check_full(env, 2)


def test_config5_full_range_subset(env):
    # 2^22 of config 5's inputs, every sample compared (the full 2^26 is sampled below)
    _check_full(env, 5, n=1 << 22)


def test_config3_range_subset_h_only(env):
    _check_full(env, 3, n=1 << 22)


@pytest.mark.parametrize("cid", [3, 5])
def test_full_size_sampled(env, cid):
    """BASELINE full sizes, the launch configuration bench.py times; 2^20 sampled
    indices (plus the first and last 4096) compared one by one."""
    oracle, vndf, synth, dev = env
    cfg = synth.CONFIGS[cid]
    n = cfg.n
    x = synth.fill(cfg.recipe, cfg.seed, n, device=dev)
    out = _stream_run(vndf, x, synth.PLANES, pdf=cfg.pdf)
    rng = np.random.default_rng(cid)
    idx = np.unique(np.concatenate([rng.integers(0, n, 1 << 20), np.arange(4096), np.arange(n - 4096, n)]))
    ti = torch.from_numpy(idx).to(dev)
    host = [x[k][ti].cpu().numpy() for k in synth.PLANES]
    h_ref, p_ref, _ = oracle.batch_sample(oracle.CAP, *host, pdf=cfg.pdf)
    hg = [o[ti].cpu().numpy() for o in out[:3]]
    pg = out[3][ti].cpu().numpy() if cfg.pdf else None
    eh, ep = _errors(hg, pg, h_ref, p_ref)
    assert eh.max() <= TOL_H
    if cfg.pdf:
        assert ep.max() <= TOL_PDF
    # invariants on EVERY sample, evaluated on the device (properties at any size)
    s = torch.where(x["wi_z"] < 0, -1.0, 1.0)
    norm = torch.sqrt(out[0].double() ** 2 + out[1].double() ** 2 + out[2].double() ** 2)
    assert float((norm - 1).abs().max()) < 2e-6
    dot = x["wi_x"] * out[0] + x["wi_y"] * out[1] + x["wi_z"] * out[2]
    assert float(dot.min()) >= -1e-6
    assert float((s * out[2]).min()) >= 0.0
    assert bool(torch.isfinite(out[0]).all() and torch.isfinite(out[2]).all())
    if cfg.pdf:
        assert bool(torch.isfinite(out[3]).all()) and float(out[3].min()) > 0


def test_config4_philox_sampled(env):
    """Config 4 at its full size (2^30, 17 GB of outputs), sampled indices."""
    oracle, vndf, synth, dev = env
    cfg = synth.CONFIGS[4]
    n = cfg.n
    out = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_philox(cfg.seed, 0, n, *out)
    torch.cuda.synchronize()
    rng = np.random.default_rng(4)
    idx = np.unique(np.concatenate([rng.integers(0, n, 1 << 20), np.arange(4096), np.arange(n - 4096, n)]))
    ti = torch.from_numpy(idx).to(dev)
    h_ref, p_ref, _ = oracle.batch_sample_philox(oracle.CAP, cfg.seed, idx)
    hg = [o[ti].cpu().numpy() for o in out[:3]]
    eh, ep = _errors(hg, out[3][ti].cpu().numpy(), h_ref, p_ref)
    assert eh.max() <= TOL_H and ep.max() <= TOL_PDF, (float(eh.max()), float(ep.max()))
    assert bool(torch.isfinite(out[3]).all()) and float(out[3].min()) > 0
    # properties at any size, on EVERY sample: unit h on the upper hemisphere
    # (config-4 incidence is upper-hemisphere, so h.z >= 0 without a flip)
    nrm = out[0].double().square_() + out[1].double().square_() + out[2].double().square_()
    assert float((nrm - 1.0).abs().max()) < 1e-6
    del nrm
    assert float(out[2].min()) >= 0.0
    del out
    torch.cuda.empty_cache()


def test_philox_full_range_small(env):
    """Every sample of a 2^20 Philox range, across the 32-bit carry of the counter."""
    oracle, vndf, synth, dev = env
    # first % 4 != 0 selects the kernel without the shared-high-word counters
    for first, n in ((0, 1 << 20), ((1 << 32) - 4096, 8192 + 3), ((1 << 32) - 4097, 8192 + 5), (3, 65539)):
        out = vndf.empty_outputs(n, dev)
        vndf.vndf_sample_cap_philox(3, first, n, *out)
        torch.cuda.synchronize()
        h_ref, p_ref, _ = oracle.batch_sample_philox(oracle.CAP, 3, np.arange(first, first + n, dtype=np.uint64))
        eh, ep = _errors([o.cpu().numpy() for o in out[:3]], out[3].cpu().numpy(), h_ref, p_ref)
        assert eh.max() <= TOL_H and ep.max() <= TOL_PDF, (first, float(eh.max()), float(ep.max()))


def test_philox_counter_wraps_and_extreme_seeds(env):
    """Counters are first_index + k modulo 2^64 (vndf.h): ranges across the
    wrap, aligned (first = 0 mod 8) and not, and the extreme seeds 0 and
    2^64 - 1, every sample against the oracle on the wrapped indices, and the
    samples past the wrap bit-identical to a call that starts at index 0."""
    oracle, vndf, synth, dev = env
    M = 1 << 64
    for seed, first, n in ((3, M - 64, 8 * 20 + 3), (3, M - 13, 8 * 16 + 5),
                           (0, M - 4096, 8192), ((1 << 64) - 1, 12345, 4099)):
        out = vndf.empty_outputs(n, dev)
        vndf.vndf_sample_cap_philox(seed, first, n, *out)
        torch.cuda.synchronize()
        idx = (np.arange(n, dtype=np.uint64) + np.uint64(first))  # wraps modulo 2^64
        h_ref, p_ref, _ = oracle.batch_sample_philox(oracle.CAP, seed, idx)
        eh, ep = _errors([o.cpu().numpy() for o in out[:3]], out[3].cpu().numpy(), h_ref, p_ref)
        assert eh.max() <= TOL_H and ep.max() <= TOL_PDF, (seed, first, float(eh.max()), float(ep.max()))
        # the same samples from a call that starts at the wrapped index 0
        k0 = int((M - first) % M)
        if 0 < k0 < n:
            tail = vndf.empty_outputs(n - k0, dev)
            vndf.vndf_sample_cap_philox(seed, 0, n - k0, *tail)
            torch.cuda.synchronize()
            for a, b in zip(out, tail):
                assert torch.equal(a[k0:], b)


def test_philox_first_index_offsets_bit_identical(env):
    """Sample k of a call with first_index f is sample f + k of a call with
    first_index 0, for every residue of f mod 4 (aligned and unaligned chunk
    counters) and for unaligned output pointers."""
    oracle, vndf, synth, dev = env
    n = (1 << 16) + 3
    ref = vndf.empty_outputs(n + 8, dev)
    vndf.vndf_sample_cap_philox(7, 0, n + 8, *ref)
    for f in (1, 2, 3, 4, 5, 7):
        out = vndf.empty_outputs(n, dev)
        vndf.vndf_sample_cap_philox(7, f, n, *out)
        torch.cuda.synchronize()
        for u, v in zip(out, ref):
            assert torch.equal(u, v[f:f + n]), f
    out = [torch.empty(n + 1, dtype=torch.float32, device=dev)[1:] for _ in range(4)]  # 4 B aligned
    vndf.vndf_sample_cap_philox(7, 2, n, *out)
    torch.cuda.synchronize()
    for u, v in zip(out, ref):
        assert torch.equal(u, v[2:2 + n])
    href = vndf.empty_outputs(n + 8, dev)
    vndf.vndf_sample_heitz2018_philox(7, 0, n + 8, *href)
    hout = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_heitz2018_philox(7, 3, n, *hout)
    torch.cuda.synchronize()
    for u, v in zip(hout, href):
        assert torch.equal(u, v[3:3 + n])


def test_philox_words_bit_exact(env):
    oracle, vndf, synth, dev = env
    rng = np.random.default_rng(9)
    ranges = [(0, 1 << 20), ((1 << 32) - 1024, 2048)] + [(int(s), 1024) for s in rng.integers(0, 1 << 40, 64)]
    for seed in (3, 0xDEADBEEFCAFEF00D):
        for first, n in ranges:
            for block in (0, 1):
                w = torch.empty(4 * n, dtype=torch.int32, device=dev)
                vndf.vndf_philox4x32_10(seed, first, n, block, w)
                got = w.cpu().numpy().view(np.uint32).reshape(n, 4)
                want = oracle.philox_words(seed, np.arange(first, first + n, dtype=np.uint64), block)
                np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("n", [1, 2, 7, 8, 9, 31, 33, 4099, 65537])
def test_ragged_sizes_and_vector_paths(env, n):
    """Tails (n mod 8 != 0) and the three vector paths (32 B, 16 B, 4 B aligned
    planes) give bit-identical results, all within tolerance."""
    oracle, vndf, synth, dev = env
    x = synth.fill(5, 4, n, device=dev)
    results = []
    for off in (0, 4, 1):  # 32 B, 16 B and 4 B aligned planes
        ins = []
        for k in synth.PLANES:
            b = torch.zeros(n + 8, dtype=torch.float32, device=dev)
            b[off:off + n] = x[k]
            ins.append(b[off:off + n])
        outs = [torch.zeros(n + 8, dtype=torch.float32, device=dev)[off:off + n] for _ in range(4)]
        vndf.vndf_sample_cap_pdf(*ins, *outs)
        torch.cuda.synchronize()
        results.append([t.cpu().numpy().copy() for t in outs])
    for r in results[1:]:
        for a, b in zip(results[0], r):
            np.testing.assert_array_equal(a, b)
    h_ref, p_ref, _ = oracle.batch_sample(oracle.CAP, *_host(x, synth.PLANES))
    eh, ep = _errors(results[0][:3], results[0][3], h_ref, p_ref)
    assert eh.max() <= TOL_H and ep.max() <= TOL_PDF


def test_determinism_and_chunking(env):
    """Outputs are a pure function of the inputs: repeated calls, split calls
    and different streams are bit-identical (vndf.h)."""
    oracle, vndf, synth, dev = env
    n = (1 << 20) + 5
    x = synth.fill(2, 1, n, device=dev)
    a = _stream_run(vndf, x, synth.PLANES)
    s = torch.cuda.Stream(dev)
    b = _stream_run(vndf, x, synth.PLANES, stream=s)
    k = 333331
    c = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_pdf(*[x[p][:k] for p in synth.PLANES], *[t[:k] for t in c], n=k)
    vndf.vndf_sample_cap_pdf(*[x[p][k:] for p in synth.PLANES], *[t[k:] for t in c], n=n - k)
    torch.cuda.synchronize()
    for u, v, w in zip(a, b, c):
        assert torch.equal(u, v) and torch.equal(u, w)
    # Philox chunking by first_index
    m = 100003
    p1 = vndf.empty_outputs(m, dev)
    vndf.vndf_sample_cap_philox(3, 5000, m, *p1)
    p2 = vndf.empty_outputs(m, dev)
    vndf.vndf_sample_cap_philox(3, 5000, 40000, *[t[:40000] for t in p2])
    vndf.vndf_sample_cap_philox(3, 45000, m - 40000, *[t[40000:] for t in p2])
    torch.cuda.synchronize()
    for u, v in zip(p1, p2):
        assert torch.equal(u, v)


def test_h_only_matches_h_pdf(env):
    oracle, vndf, synth, dev = env
    x = synth.fill(3, 2, 1 << 20, device=dev)
    a = _stream_run(vndf, x, synth.PLANES, pdf=False)
    b = _stream_run(vndf, x, synth.PLANES, pdf=True)
    for u, v in zip(a, b[:3]):
        assert torch.equal(u, v)


@pytest.mark.parametrize("cid", [1, 2, 5])
def test_heitz_baseline_conditioned_parity(env, cid):
    """The literal fp32 Listing 2 baseline (reading R8) carries no
    accuracy contract: its reprojection ti = sqrt(1 - t1^2 - t2^2) and
    sqrt(1 - t1^2) cancel, and its hs.z error is absolute, so the
    unstretch amplifies it by 1/|m|.  Model: |dh| <~ 1e-6 (1/ti + 1/sqrt(1 - t1^2)) / |m|.
    Where the model predicts <= 2e-5 the kernel must meet the 2e-5 / 1e-4
    contract; overall it must stay within tolerance on >= 98% of samples."""
    oracle, vndf, synth, dev = env
    cfg = synth.CONFIGS[cid]
    n = min(cfg.n, 1 << 22)
    x = synth.fill(cfg.recipe, cfg.seed, n, device=dev)
    out = _stream_run(vndf, x, synth.PLANES, pdf=True, kernel="heitz")
    host = _host(x, synth.PLANES)
    h_ref, p_ref, ti = oracle.batch_sample(oracle.HEITZ, *host)
    eh, ep = _errors([o.cpu().numpy() for o in out[:3]], out[3].cpu().numpy(), h_ref, p_ref)
    ax, ay = host[3].astype(np.float64), host[4].astype(np.float64)
    s = np.where(host[2] < 0, -1.0, 1.0)
    N = 1.0 / np.sqrt((s * h_ref[0] / ax) ** 2 + (s * h_ref[1] / ay) ** 2 + h_ref[2] ** 2)
    rim = 1.0 - host[6].astype(np.float64) * np.cos(2 * np.pi * host[5].astype(np.float64)) ** 2
    with np.errstate(divide="ignore"):
        est = 1e-6 * (1.0 / ti + 1.0 / np.sqrt(np.maximum(rim, 0))) / N
    good = est <= TOL_H
    within = (eh <= TOL_H) & (ep <= TOL_PDF)
    print(f"config {cid}: Heitz fp32 within tolerance on {within.mean():.5f} of samples; "
          f"model-conditioned subset {good.mean():.4f}, max|dh| there {eh[good].max():.2e}, "
          f"outside {eh[~good].max() if (~good).any() else 0:.2e}")
    assert good.mean() > 0.5
    assert eh[good].max() <= TOL_H, float(eh[good].max())
    assert ep[good].max() <= TOL_PDF, float(ep[good].max())
    assert within.mean() >= 0.98
    assert bool(torch.isfinite(out[0]).all())


def test_host_entry_point_matches_device(env):
    oracle, vndf, synth, dev = env
    n = (1 << 23) + 17  # three pipeline chunks, ragged
    x = synth.fill(5, 4, n, device=dev)
    d = _stream_run(vndf, x, synth.PLANES)
    # page-locked, mapped buffers: the zero-copy path
    hin = [x[k].cpu().pin_memory() for k in synth.PLANES]
    hout = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(4)]
    vndf.vndf_sample_cap_pdf_host(*hin, *hout)
    for a, b in zip(d, hout):
        assert torch.equal(a.cpu(), b)
    # pageable numpy buffers: the staged, pipelined path (several 2 Mi chunks, ragged)
    nin = [t.numpy().copy() for t in hin]
    nout = [np.empty(n, dtype=np.float32) for _ in range(4)]
    vndf.vndf_sample_cap_pdf_host(*nin, *nout)
    for a, b in zip(d, nout):
        np.testing.assert_array_equal(a.cpu().numpy(), b)
    # mixed: pinned inputs, pageable outputs -> staged path as well
    mout = [np.empty(n, dtype=np.float32) for _ in range(4)]
    vndf.vndf_sample_cap_pdf_host(*hin, *mout)
    for a, b in zip(d, mout):
        np.testing.assert_array_equal(a.cpu().numpy(), b)
    # h only (pdf = NULL: config 3's end-to-end form), zero-copy and staged
    h3 = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(3)]
    vndf.vndf_sample_cap_pdf_host(*hin, *h3, None)
    n3 = [np.empty(n, dtype=np.float32) for _ in range(3)]
    vndf.vndf_sample_cap_pdf_host(*nin, *n3, None)
    for a, b, c in zip(d[:3], h3, n3):
        assert torch.equal(a.cpu(), b)
        np.testing.assert_array_equal(a.cpu().numpy(), c)


def test_philox_host_entry_point_matches_device(env):
    """vndf_sample_cap_philox_host (config-4 end to end, host outputs) is bit
    identical to vndf_sample_cap_philox: pinned and pageable outputs (staged
    chunks, ragged), and without pdf (the forced zero-copy path:
    test_host_paths_gpu.py)."""
    oracle, vndf, synth, dev = env
    n = (1 << 22) + 2 ** 21 + 13     # three staging chunks, ragged
    first = 2**32 - 1000             # the 32-bit counter carry inside the call
    d = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_philox(3, first, n, *d)
    ref = [t.cpu() for t in d]
    hp = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(4)]
    vndf.vndf_sample_cap_philox_host(3, first, n, *hp)
    for a, b in zip(ref, hp):
        assert torch.equal(a, b)
    nu = [np.empty(n, dtype=np.float32) for _ in range(4)]
    vndf.vndf_sample_cap_philox_host(3, first, n, *nu)
    for a, b in zip(ref, nu):
        np.testing.assert_array_equal(a.numpy(), b)
    h3 = [np.empty(n, dtype=np.float32) for _ in range(3)]
    vndf.vndf_sample_cap_philox_host(3, first, n, *h3)
    for a, b in zip(ref[:3], h3):
        np.testing.assert_array_equal(a.numpy(), b)


def test_fixup_rates(env):
    """The float64 fix-up stays rare (it is the accuracy safety net, DESIGN.md s.6)."""
    oracle, vndf, synth, dev = env
    for cid in (1, 2, 3, 5):
        cfg = synth.CONFIGS[cid]
        n = min(cfg.n, 1 << 24)
        x = synth.fill(cfg.recipe, cfg.seed, n, device=dev)
        c = torch.zeros(1, dtype=torch.int64, device=dev)
        vndf.vndf_count_fixups(*[x[k] for k in synth.PLANES], c)
        rate = int(c.item()) / n
        print(f"config {cid}: fix-up rate {rate:.3e}")
        assert rate < 0.02
    c = torch.zeros(1, dtype=torch.int64, device=dev)
    vndf.vndf_count_fixups_philox(3, 0, 1 << 24, c)
    assert int(c.item()) / (1 << 24) < 0.02


def test_error_codes(env):
    oracle, vndf, synth, dev = env
    L = vndf.lib()
    import ctypes
    x = synth.fill(1, 0, 64, device=dev)
    o = vndf.empty_outputs(64, dev)
    P = [ctypes.c_void_p(x[k].data_ptr()) for k in synth.PLANES]
    Q = [ctypes.c_void_p(t.data_ptr()) for t in o]
    assert L.vndf_sample_cap_pdf(*P, *Q, -1, None) == vndf.VNDF_ERR_INVALID_ARGUMENT
    assert L.vndf_sample_cap_pdf(*P, *Q, 0, None) == vndf.VNDF_OK
    assert L.vndf_sample_cap_pdf(*P[:6], None, *Q, 64, None) == vndf.VNDF_ERR_INVALID_ARGUMENT
    assert L.vndf_sample_cap_pdf(*P, P[0], *Q[1:], 64, None) == vndf.VNDF_ERR_INVALID_ARGUMENT  # alias
    assert L.vndf_sample_cap_pdf(*P, Q[0], Q[0], *Q[2:], 64, None) == vndf.VNDF_ERR_INVALID_ARGUMENT
    assert L.vndf_sample_cap_pdf(*P, *Q[:3], None, 64, None) == vndf.VNDF_ERR_INVALID_ARGUMENT
    odd = ctypes.c_void_p(x["u2"].data_ptr() + 2)
    assert L.vndf_sample_cap_pdf(*P[:6], odd, *Q, 8, None) == vndf.VNDF_ERR_INVALID_ARGUMENT
    assert L.vndf_sample_cap(*P, *Q[:3], 64, None) == vndf.VNDF_OK
    assert L.vndf_sample_heitz2018(*P, *Q[:3], None, 64, None) == vndf.VNDF_OK
    assert L.vndf_sample_cap_philox(1, 0, -5, *Q, None) == vndf.VNDF_ERR_INVALID_ARGUMENT
    assert L.vndf_sample_cap_philox(1, 0, 64, Q[0], Q[0], Q[2], Q[3], None) == vndf.VNDF_ERR_INVALID_ARGUMENT
    # histogram: 32-bit per-block partial counts bound the samples per call
    counts = torch.zeros(64, dtype=torch.int64, device=dev)
    cp = ctypes.c_void_p(counts.data_ptr())
    assert L.vndf_histogram(0, 0, 0.0, 0.0, 1.0, 0.5, 0.5, 1, 0, 1 << 62, 8, 8, cp, None) \
        == vndf.VNDF_ERR_INVALID_ARGUMENT
    assert L.vndf_histogram(0, 0, 0.0, 0.0, 1.0, 0.5, 0.5, 1, 0, 1000, 8, 8, cp, None) == vndf.VNDF_OK
    torch.cuda.synchronize()
    assert int(counts.sum().item()) == 1000


def test_heitz_philox_conditioned_parity(env):
    """The fused Heitz baseline on config-4 inputs (same generation as the cap
    kernel) against the float64 Listing 2: same error-model gate as the
    streamed baseline (reading R8)."""
    oracle, vndf, synth, dev = env
    n = 1 << 21
    out = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_heitz2018_philox(3, 77, n, *out)
    torch.cuda.synchronize()
    idx = np.arange(77, 77 + n, dtype=np.uint64)
    h_ref, p_ref, ti = oracle.batch_sample_philox(oracle.HEITZ, 3, idx)
    eh, ep = _errors([o.cpu().numpy() for o in out[:3]], out[3].cpu().numpy(), h_ref, p_ref)
    X = oracle.philox_words(3, idx, 0).astype(np.uint64)   # wi, alpha
    Y = oracle.philox_words(3, idx, 1).astype(np.uint64)   # u1, u2
    ax = 0.01 * 100.0 ** ((X[:, 2] >> 8) / 2**24)
    ay = 0.01 * 100.0 ** ((X[:, 3] >> 8) / 2**24)
    u1, u2 = (Y[:, 0] >> 8) / 2**24, (Y[:, 1] >> 8) / 2**24
    N = 1.0 / np.sqrt((h_ref[0] / ax) ** 2 + (h_ref[1] / ay) ** 2 + h_ref[2] ** 2)
    rim = 1.0 - u2 * np.cos(2 * np.pi * u1) ** 2
    with np.errstate(divide="ignore"):
        est = 1e-6 * (1.0 / ti + 1.0 / np.sqrt(np.maximum(rim, 0))) / N
    good = est <= TOL_H
    assert good.mean() > 0.5
    assert eh[good].max() <= TOL_H and ep[good].max() <= TOL_PDF, (float(eh[good].max()), float(ep[good].max()))
    assert ((eh <= TOL_H) & (ep <= TOL_PDF)).mean() >= 0.98


@pytest.mark.parametrize("cfg", [(0, 0, 0), (8, 128, 1), (8, 256, 2), (4, 64, 0), (1, 128, 0), (0, 0, -1)])
def test_launch_configurations_bit_identical(env, cfg):
    """Persistent grid-stride grids (many chunks per thread and block), other
    block sizes and vector widths give bit-identical results (the tuning knob
    of vndf.h changes scheduling only; queue overflow: test_overflow_gpu.py)."""
    oracle, vndf, synth, dev = env
    n = (1 << 21) + 13
    x = synth.fill(5, 4, n, device=dev)
    ref = _stream_run(vndf, x, synth.PLANES)
    try:
        vndf.vndf_set_launch_config(*cfg)
        got = _stream_run(vndf, x, synth.PLANES)
        p1 = vndf.empty_outputs(n, dev)
        vndf.vndf_sample_cap_philox(3, 0, n, *p1)
    finally:
        vndf.vndf_set_launch_config(0, 0, 0)
    p0 = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_philox(3, 0, n, *p0)
    torch.cuda.synchronize()
    for a, b in zip(ref, got):
        assert torch.equal(a, b)
    for a, b in zip(p0, p1):
        assert torch.equal(a, b)


@pytest.mark.parametrize("n", [(1 << 16) + 9, (1 << 17) + 3, (1 << 18) + 5, (1 << 19) + 7, (1 << 22) + 1])
def test_default_shapes_across_sizes(env, n):
    """The size-dependent default launch shape (1 x 64, 1 x 256, 4 x 128, 8 x 128
    by samples per SM; vndf.cu stream_shape) on the config-5 edge mix: every
    sample within tolerance of the float64 oracle, and bit-identical to the
    8 x 128 shape, cap and Heitz."""
    oracle, vndf, synth, dev = env
    x = synth.fill(5, 4, n, device=dev)
    out = _stream_run(vndf, x, synth.PLANES)
    heitz = _stream_run(vndf, x, synth.PLANES, kernel="heitz")
    try:
        vndf.vndf_set_launch_config(8, 128, 0)
        ref = _stream_run(vndf, x, synth.PLANES)
        href = _stream_run(vndf, x, synth.PLANES, kernel="heitz")
    finally:
        vndf.vndf_set_launch_config(0, 0, 0)
    for a, b in zip(list(out) + list(heitz), list(ref) + list(href)):
        assert torch.equal(a, b)
    host = _host(x, synth.PLANES)
    h_ref, p_ref, _ = oracle.batch_sample(oracle.CAP, *host, pdf=True)
    eh, ep = _errors([o.cpu().numpy() for o in out[:3]], out[3].cpu().numpy(), h_ref, p_ref)
    assert eh.max() <= TOL_H and ep.max() <= TOL_PDF, (float(eh.max()), float(ep.max()))
