"""NEXT-3 pins: the paper's native handling of incidence below the horizon
(Fig. 4, theta_i = 130 deg; sigma_std = (1 + z_i)/2 on [-1, 1], Eq. 4)."""
import numpy as np
import pytest

from oracle import stats

CAP, HEITZ = 0, 1
CASES = [(110, 0, 1.0, 1.0), (130, 20, 0.3, 0.3), (130, 60, 0.5, 0.1), (160, 45, 0.6, 0.6), (100, 10, 0.05, 0.3)]


def _wi(t, p):
    t, p = np.radians(t), np.radians(p)
    return np.array([np.sin(t) * np.cos(p), np.sin(t) * np.sin(p), np.cos(t)])


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
def test_native_pdf_normalises(orc, case):
    t, p, ax, ay = case
    m = stats.bin_masses(_wi(t, p), ax, ay, native=True)
    assert m.sum() == pytest.approx(1.0, abs=3e-4)


def test_native_equals_flip_above_horizon(orc):
    """For wi.z >= 0 the native and flipped forms coincide."""
    rng = np.random.default_rng(30)
    for _ in range(500):
        wi = rng.normal(size=3); wi[2] = abs(wi[2]); wi /= np.linalg.norm(wi)
        ax, ay = np.exp(rng.uniform(np.log(0.01), 0, 2))
        u1, u2 = rng.uniform(0, 1, 2)
        for m in (CAP, HEITZ):
            # the native cap is evaluated in binary128 (reading R17): equal to rounding
            np.testing.assert_allclose(orc.sample_vndf_native(m, wi, ax, ay, u1, u2),
                                       orc.sample_vndf(m, wi, ax, ay, u1, u2), atol=1e-10)
        h = orc.sample_vndf(CAP, wi, ax, ay, u1, u2)
        assert orc.pdf_vndf_native(h, wi, ax, ay) == orc.pdf_vndf(h, wi, ax, ay)


def test_native_quad_cap_resolves_straight_below(orc):
    """Reading R17: at ws.z = -1 + 1e-8 the binary128 evaluation keeps h.z =
    (1 - u2)(1 + ws.z) (the exact algebraic value of z + ws.z, Listing 3)."""
    ax = ay = 1e-3
    wi = np.array([0.187, -0.0439, -0.9813727])
    wi /= np.linalg.norm(wi)
    u1, u2 = 0.46373, 1 - 2**-24
    h = orc.sample_vndf_native(CAP, wi, ax, ay, u1, u2)
    t = np.array([ax * wi[0], ay * wi[1], wi[2]])
    L = np.linalg.norm(t)
    ws = t / L
    a = (ws[0] ** 2 + ws[1] ** 2) / (1 - ws[2])       # 1 + ws.z without cancellation
    hz = (1 - u2) * a
    st = np.sqrt(u2 * ((1 - u2) * a * a + ws[0] ** 2 + ws[1] ** 2))
    hs = np.array([st * np.cos(2 * np.pi * u1) + ws[0], st * np.sin(2 * np.pi * u1) + ws[1], hz])
    m = np.array([ax * hs[0], ay * hs[1], hs[2]])
    np.testing.assert_allclose(h, m / np.linalg.norm(m), atol=1e-9)


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
@pytest.mark.parametrize("method", [CAP, HEITZ], ids=["cap", "heitz"])
def test_native_chi2_and_invariants(orc, case, method):
    t, p, ax, ay = case
    wi = _wi(t, p)
    n = 1 << 20
    rng = np.random.default_rng(31 + method)
    u = rng.random((2, n), dtype=np.float32)
    wi32 = wi.astype(np.float32)
    h, _ = orc.batch_sample_native(method, np.full(n, wi32[0]), np.full(n, wi32[1]), np.full(n, wi32[2]),
                                   np.full(n, ax, np.float32), np.full(n, ay, np.float32), u[0], u[1],
                                   pdf=False)
    assert h[2].min() >= -1e-12                       # upper-hemisphere normals
    assert (wi32.astype(np.float64) @ h).min() >= -1e-9  # visible from wi
    _, _, pv = stats.pearson(stats.histogram(h), stats.bin_masses(wi32.astype(np.float64), ax, ay, native=True))
    assert pv > 1e-3


@pytest.mark.parametrize("case", [(130, 20, 0.3, 0.3), (110, 0, 1.0, 1.0), (100, 10, 0.05, 0.3)])
def test_native_raycast_definition(orc, case):
    """The definition with rays from below: same distribution."""
    t, p, ax, ay = case
    wi = _wi(t, p)
    hr, trials = orc.batch_raycast_native(wi, ax, ay, seed=5, n=1 << 18)
    _, _, pv = stats.pearson(stats.histogram(hr), stats.bin_masses(wi, ax, ay, native=True))
    assert pv > 1e-3
