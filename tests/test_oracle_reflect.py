"""Pins of the oracle's NEXT-2 functions: BRDF importance sampling with the VNDF
(appendix): reflection (Eq. 5), the reflected-direction pdf
(Eq. 20), height-correlated Smith G2 (Eq. 13-14), the Cook-Torrance BRDF
(Eq. 11, F = 1) and the Monte Carlo estimator (Eq. 19)."""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_values.json")))
CAP, HEITZ = 0, 1


def _dir(theta_deg, phi_deg=0.0):
    t, p = np.radians(theta_deg), np.radians(phi_deg)
    return np.array([np.sin(t) * np.cos(p), np.sin(t) * np.sin(p), np.cos(t)])


def test_spec_worked_values(orc):
    e = GOLD["G2_combination"]
    pole = [0, 0, 1]
    # G1 = 1 at the pole; G1 = 2z/(1+z) = 0.5 at z = 1/3 with alpha = 1 (Eq. 17)
    z = 1.0 / 3.0
    wo = [np.sqrt(1 - z * z), 0, z]
    assert orc.G2(pole, pole, pole, 1, 1) == pytest.approx(e[0]["value"])
    assert orc.G1(pole, wo, 1, 1) == pytest.approx(0.5)
    assert orc.G2(pole, pole, wo, 1, 1) == pytest.approx(e[1]["value"])
    b = GOLD["brdf"][0]
    assert orc.brdf_cos(b["wi"], b["wo"], *b["alpha"]) == pytest.approx(b["value"], abs=1e-7)
    p = GOLD["pdf_reflected"][0]
    assert orc.pdf_reflect(p["wa"], p["wb"], *p["alpha"]) == pytest.approx(p["value"], abs=1e-7)
    r = GOLD["reflect_sample_pole"][0]
    out = orc.sample_reflect(CAP, r["wa"], *r["alpha"], *r["u"])
    np.testing.assert_allclose(out[:3], r["wb"], atol=1e-12)
    assert out[4] == pytest.approx(r["weight"])


def test_eq20_equals_vndf_times_reflection_jacobian(orc):
    """Eq. 20 (G1 D / 4cos) == Eq. 1 x Eq. 8 (D_vis / (4 |wb.wm|))."""
    rng = np.random.default_rng(20)
    for _ in range(3000):
        wa = rng.normal(size=3); wa[2] = abs(wa[2]) + 1e-2; wa /= np.linalg.norm(wa)
        wb = rng.normal(size=3); wb /= np.linalg.norm(wb)
        if np.linalg.norm(wa + wb) < 1e-3:
            continue
        ax, ay = np.exp(rng.uniform(np.log(0.02), 0, 2))
        wm = orc.half_vector(wa, wb)
        want = orc.pdf_vndf(wm, wa, ax, ay) * orc.reflect_jacobian(wb, wm)
        assert orc.pdf_reflect(wa, wb, ax, ay) == pytest.approx(want, rel=1e-9, abs=1e-300)


@pytest.mark.parametrize("za", [0.3, 0.7, 1.0])
@pytest.mark.parametrize("alpha", [(0.1, 0.1), (0.5, 0.5), (1.0, 1.0), (0.1, 0.6)])
def test_eq20_integrates_to_one(orc, za, alpha):
    """the reflected-direction pdf is normalised over the whole sphere."""
    wa = np.array([np.sqrt(1 - za * za), 0.0, za])
    dirs, w = orc.sphere_quadrature(nz=768, nphi=768)
    tot = float((orc.batch_pdf_reflect(wa, *alpha, dirs) * w).sum())
    assert tot == pytest.approx(1.0, abs=2e-3)


def test_brdf_reciprocity(orc):
    """f_r(wi, wo) = f_r(wo, wi): compare brdf_cos / cos(theta_o)."""
    rng = np.random.default_rng(21)
    for _ in range(2000):
        wi, wo = rng.normal(size=(2, 3))
        wi[2], wo[2] = abs(wi[2]) + 1e-2, abs(wo[2]) + 1e-2
        wi /= np.linalg.norm(wi); wo /= np.linalg.norm(wo)
        ax, ay = np.exp(rng.uniform(np.log(0.05), 0, 2))
        a = orc.brdf_cos(wi, wo, ax, ay) / wo[2]
        b = orc.brdf_cos(wo, wi, ax, ay) / wi[2]
        assert a == pytest.approx(b, rel=1e-10)


@pytest.mark.parametrize("method", [CAP, HEITZ])
def test_weight_is_g2_over_g1(orc, method):
    """f_r |cos| / PDF reduces to G2/G1 in [0, 1]; zero below the horizon."""
    rng = np.random.default_rng(22 + method)
    for _ in range(2000):
        wa = rng.normal(size=3); wa[2] = abs(wa[2]) + 1e-3; wa /= np.linalg.norm(wa)
        ax, ay = np.exp(rng.uniform(np.log(0.01), 0, 2))
        u1, u2 = rng.uniform(0, 1, 2)
        r = orc.sample_reflect(method, wa, ax, ay, u1, u2)
        wb = r[:3]
        wm = orc.sample_vndf(method, wa, ax, ay, u1, u2)
        np.testing.assert_allclose(wb, orc.reflect(wa, wm), atol=1e-12)
        if wb[2] > 0:
            want = orc.G2(wm, wa, wb, ax, ay) / orc.G1(wm, wa, ax, ay)
            assert r[4] == pytest.approx(want, rel=1e-9)
        else:
            assert r[4] == 0.0
        assert 0.0 <= r[4] <= 1.0 + 1e-12


@pytest.mark.parametrize("theta,alpha", [(0, (0.1, 0.1)), (45, (0.5, 0.5)), (75, (0.3, 0.05)),
                                         (60, (1.0, 1.0))])
def test_furnace_estimator_converges_to_albedo(orc, theta, alpha):
    """Eq. 19 with L = 1 is an unbiased estimator of the directional albedo
    int f_r cos dwo (Eq. 18): the oracle's MC mean agrees with quadrature within
    5 standard errors, for both samplers, and both samplers show the same
    variance ("the same variance reduction")."""
    wa = _dir(theta, 20)
    dirs, w = orc.sphere_quadrature(nz=1024, nphi=1024, upper_only=True)
    albedo = float((orc.batch_brdf_cos(wa, *alpha, dirs) * w).sum())
    n = 1 << 17
    stats = []
    for method in (CAP, HEITZ):
        s, sq = orc.furnace(method, wa, *alpha, seed=7 + method, n=n)
        mean = s / n
        var = sq / n - mean * mean
        se = np.sqrt(var / n)
        assert abs(mean - albedo) <= 5 * se + 1e-6, (method, mean, albedo, se)
        stats.append((mean, var))
    (m0, v0), (m1, v1) = stats
    if v0 > 1e-12:
        # ratio of sample variances of the same distribution: relative sd ~ sqrt(2/n) * kurtosis factor
        assert abs(v1 / v0 - 1) < 0.05
    if theta == 0 and alpha == (0.1, 0.1):
        assert m0 >= 0.95  # near-specular single-scatter albedo at normal incidence


@pytest.mark.parametrize("method", [CAP, HEITZ], ids=["cap", "heitz"])
@pytest.mark.parametrize("theta,alpha", [(30, (0.4, 0.4)), (70, (0.3, 0.6)), (0, (1.0, 1.0))])
def test_reflected_directions_follow_eq20(orc, method, theta, alpha):
    """The appendix's sampling steps (1)-(2) produce directions distributed as
    Eq. 20 over the whole sphere (below-horizon reflections included)."""
    from oracle import stats
    wa = _dir(theta, 40)
    n = 1 << 19
    rng = np.random.default_rng(60 + method + theta)
    u = rng.random((2, n), dtype=np.float32)
    wa32 = wa.astype(np.float32)
    out = orc.batch_sample_reflect(method, np.full(n, wa32[0]), np.full(n, wa32[1]), np.full(n, wa32[2]),
                                   np.full(n, alpha[0], np.float32), np.full(n, alpha[1], np.float32), u[0], u[1])
    masses = stats.sphere_bin_masses(lambda d: orc.batch_pdf_reflect(wa32.astype(np.float64), *alpha, d))
    assert masses.sum() == pytest.approx(1.0, abs=2e-3)
    _, _, pv = stats.pearson(stats.sphere_histogram(out[:3]), masses)
    assert pv > 1e-3, pv


def test_batch_reflect_philox_driver(orc):
    """The Philox batch driver is orc_sample_reflect on orc_c4_inputs, index by
    index (no arithmetic of its own), for both methods and 64-bit indices."""
    idx = np.array([0, 1, 7, 4095, (1 << 32) - 1, 1 << 32, (1 << 40) + 3], dtype=np.uint64)
    for method in (orc.CAP, orc.HEITZ):
        got = orc.batch_sample_reflect_philox(method, 9, idx, threads=3)
        for k, i in enumerate(idx):
            x = orc.c4_inputs(9, int(i))
            want = orc.sample_reflect(method, x[:3], x[3], x[4], x[5], x[6])
            np.testing.assert_array_equal(got[:, k], want)


# --------------------------------------------------------------- G2 pins --
def test_G2_height_correlated_at_half_half(orc):
    """Eq. 13-14: G2 = Gi Go / (Gi + Go - Gi Go).  With alpha = 1,
    wm = pole and z_i = z_o = 1/3, Eq. 17 gives Gi = Go = 2z/(1+z) = 1/2, so
    G2 = (1/4) / (3/4) = 1/3 -- the separable product Gi Go would give 1/4."""
    z = 1.0 / 3.0
    s = np.sqrt(1 - z * z)
    wi = [s, 0.0, z]
    wo = [-s * 0.6, s * 0.8, z]
    pole = [0.0, 0.0, 1.0]
    assert orc.G1(pole, wi, 1, 1) == pytest.approx(0.5, abs=1e-15)
    assert orc.G1(pole, wo, 1, 1) == pytest.approx(0.5, abs=1e-15)
    assert orc.G2(pole, wi, wo, 1, 1) == pytest.approx(1.0 / 3.0, abs=1e-14)


def _lambda_heitz2014(w, ax, ay):
    """Smith Lambda of the anisotropic GGX NDF (Heitz 2014, 'Understanding the
    masking-shadowing function', eq. 86 with alpha_o^2 = ax^2 cos^2 phi +
    ay^2 sin^2 phi): Lambda = (-1 + sqrt(1 + (ax^2 x^2 + ay^2 y^2) / z^2)) / 2."""
    x, y, zz = w
    a2t2 = (ax * ax * x * x + ay * ay * y * y) / (zz * zz)
    return 0.5 * (-1.0 + np.sqrt(1.0 + a2t2))


def test_G2_matches_heitz2014_height_correlated_form(orc):
    """Independent textbook form of the height-correlated Smith term (Heitz 2014,
    eq. 99): G2 = chi+(wi.wm) chi+(wo.wm) / (1 + Lambda(wi) + Lambda(wo)).
    Random (wi, wo, alpha), wm the half vector (positive chi+ on both sides)."""
    rng = np.random.default_rng(1314)
    checked = 0
    for _ in range(4000):
        wi = rng.normal(size=3); wi[2] = abs(wi[2]) + 1e-3; wi /= np.linalg.norm(wi)
        wo = rng.normal(size=3); wo[2] = abs(wo[2]) + 1e-3; wo /= np.linalg.norm(wo)
        ax, ay = np.exp(rng.uniform(np.log(0.01), 0, 2))
        wm = orc.half_vector(wi, wo)
        want = 1.0 / (1.0 + _lambda_heitz2014(wi, ax, ay) + _lambda_heitz2014(wo, ax, ay))
        got = orc.G2(wm, wi, wo, ax, ay)
        assert got == pytest.approx(want, rel=1e-10, abs=1e-15)
        # and the separable product is measurably different here
        gi, go = orc.G1(wm, wi, ax, ay), orc.G1(wm, wo, ax, ay)
        if want > 1e-3 and max(gi, go) < 0.9:
            assert abs(gi * go - want) > 1e-4 * want
        checked += 1
    assert checked == 4000
