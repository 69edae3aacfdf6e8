"""NEXT-4: the standalone VNDF pdf kernel (Eq. 1) against the
float64 oracle at identical fp32 inputs; tolerance 1e-4 relative (exact zero
where the oracle's pdf is zero: back-facing h, h below the horizon)."""
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
    import oracle
    import paper_2306_05044_b200 as vndf
    import synth
    return oracle, vndf, synth, torch.device("cuda:0")


def _check(oracle, vndf, dev, h, wi, ax, ay):
    n = h.shape[1]
    t = [torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).to(dev) for v in (*h, *wi, ax, ay)]
    out = torch.empty(n, dtype=torch.float32, device=dev)
    vndf.vndf_pdf(*t, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy().astype(np.float64)
    hh = np.stack([x.cpu().numpy() for x in t[:3]]).astype(np.float64)
    ww = np.stack([x.cpu().numpy() for x in t[3:6]]).astype(np.float64)
    nh = hh / np.linalg.norm(hh, axis=0)
    ref = oracle.batch_pdf(nh, ww, t[6].cpu().numpy().astype(np.float64), t[7].cpu().numpy().astype(np.float64))
    zero = ref == 0
    assert np.all(got[zero] == 0)
    rel = np.abs(got[~zero] - ref[~zero]) / ref[~zero]
    return rel


@pytest.mark.parametrize("cid", [2, 5])
def test_pdf_at_sampled_h(env, cid):
    oracle, vndf, synth, dev = env
    cfg = synth.CONFIGS[cid]
    n = 1 << 21
    x = synth.fill(cfg.recipe, cfg.seed, n, device=dev)
    hx, hy, hz, p = vndf.empty_outputs(n, dev)
    vndf.vndf_sample_cap_pdf(*[x[k] for k in synth.PLANES], hx, hy, hz, p)
    torch.cuda.synchronize()
    h = np.stack([hx.cpu().numpy(), hy.cpu().numpy(), hz.cpu().numpy()])
    wi = np.stack([x[k].cpu().numpy() for k in ("wi_x", "wi_y", "wi_z")])
    rel = _check(oracle, vndf, dev, h, wi, x["alpha_x"].cpu().numpy(), x["alpha_y"].cpu().numpy())
    print(f"config {cid}: max rel {rel.max():.2e}")
    assert rel.max() <= 1e-4


def test_pdf_random_directions_ragged(env):
    """Arbitrary (non-unit, back-facing, below-horizon) h and wi, ragged n."""
    oracle, vndf, synth, dev = env
    rng = np.random.default_rng(44)
    n = 100003
    h = rng.normal(size=(3, n)) * rng.uniform(0.5, 2.0, n)
    wi = rng.normal(size=(3, n)) * rng.uniform(0.5, 2.0, n)
    ax = np.exp(rng.uniform(np.log(1e-3), 0, n))
    ay = np.exp(rng.uniform(np.log(1e-3), 0, n))
    rel = _check(oracle, vndf, dev, h, wi, ax, ay)
    assert rel.max() <= 1e-4
