"""Pins of the float64 oracle against closed forms, textbook formulas, worked
values and invariants that the paper and the mathematics fix.

Each test names the passage it pins.  P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_values.json")))
CAP, HEITZ = 0, 1


# ------------------------------------------------------------ worked values ---
def test_spec_worked_values(orc):
    for e in GOLD["sigma_std"]:
        assert orc.sigma_std(e["wi"][2]) == pytest.approx(e["value"], abs=1e-7), e["cite"]
    for e in GOLD["D_std"]:
        assert orc.D_std(e["wm"][2]) == pytest.approx(e["value"], abs=1e-7), e["cite"]
    for e in GOLD["Dvis_std"]:
        assert orc.Dvis_std(e["wm"], e["wi"]) == pytest.approx(e["value"], abs=1e-7), e["cite"]
    for e in GOLD["pdf_vndf_ggx"]:
        assert orc.pdf_vndf(e["wm"], e["wi"], *e["alpha"]) == pytest.approx(e["value"], abs=1e-7)
    for e in GOLD["cap_samples_normal_incidence"]:
        h = orc.sample_vndf(CAP, e["wi"], 1.0, 1.0, *e["u"])
        np.testing.assert_allclose(h, e["h"], atol=1e-7, err_msg=e["cite"])
    for e in GOLD["ggx_pole_fixed_point"]:
        h = orc.sample_vndf(CAP, e["wi"], *e["alpha"], *e["u"])
        np.testing.assert_allclose(h, e["h"], atol=1e-12, err_msg=e["cite"])
    for e in GOLD["reflect"]:
        np.testing.assert_allclose(orc.reflect(e["wi"], e["wm"]), e["wo"], atol=1e-7)
    for e in GOLD["reflect_jacobian"]:
        assert orc.reflect_jacobian(e["wo"], e["wh"]) == pytest.approx(e["value"])
    for e in GOLD["cap_density"]:
        assert orc.cap_density(e["wo"], e["wi"]) == pytest.approx(e["value"], abs=1e-7), e["cite"]
    for e in GOLD["D_ggx"]:
        assert orc.D_ggx(e["wm"], *e["alpha"]) == pytest.approx(e["value"], abs=1e-7), e["cite"]
    for e in GOLD["G1"]:
        wm = np.asarray(e["wm"]) / np.linalg.norm(e["wm"])
        assert orc.G1(wm, e["wk"], *e["alpha"]) == pytest.approx(e["value"], abs=1e-7), e["cite"]


# -------------------------------------------------- normal-incidence closed form
def _ggx_inversion(ax, ay, u1, u2):
    """Textbook anisotropic GGX NDF inversion (Walter et al. 2007 with the
    anisotropic stretch): slope = (ax sqrt(u2) cos 2pi u1, ay sqrt(u2) sin 2pi u1)
    / sqrt(1 - u2); h = normalize(-slope..., 1) up to the sign convention of the
    slope, i.e. h = normalize(ax sqrt(u2) cos, ay sqrt(u2) sin, sqrt(1 - u2))."""
    v = np.array([ax * np.sqrt(u2) * np.cos(2 * np.pi * u1),
                  ay * np.sqrt(u2) * np.sin(2 * np.pi * u1),
                  np.sqrt(1 - u2)])
    return v / np.linalg.norm(v)


def _textbook_D(h, ax, ay):
    """GGX NDF in theta/phi form (Walter 2007; Heitz 2014 eq. 85)."""
    th = np.arccos(np.clip(h[2], -1, 1))
    ph = np.arctan2(h[1], h[0])
    if h[2] <= 0:
        return 0.0
    t2 = np.tan(th) ** 2
    return 1.0 / (np.pi * ax * ay * np.cos(th) ** 4
                  * (1 + t2 * (np.cos(ph) ** 2 / ax ** 2 + np.sin(ph) ** 2 / ay ** 2)) ** 2)


def _textbook_G1(w, ax, ay):
    """Smith GGX masking via Lambda (Heitz 2014, eq. 86 with projected roughness)."""
    th = np.arccos(np.clip(w[2], -1, 1))
    ph = np.arctan2(w[1], w[0])
    a2 = np.cos(ph) ** 2 * ax ** 2 + np.sin(ph) ** 2 * ay ** 2
    lam = (-1 + np.sqrt(1 + a2 * np.tan(th) ** 2)) / 2
    return 1.0 / (1.0 + lam)


def _textbook_vndf(h, w, ax, ay):
    """Heitz & d'Eon 2014 definition D_w(h) = G1(w) max(0, w.h) D(h) / cos(theta_w)."""
    return _textbook_G1(w, ax, ay) * max(0.0, float(np.dot(w, h))) * _textbook_D(h, ax, ay) / w[2]


def test_normal_incidence_is_textbook_ggx_inversion(orc):
    """P3: at wi = (0,0,1) both samplers reduce per sample to GGX NDF inversion,
    and the VNDF reduces to D(h) h.z (G1 = 1)."""
    rng = np.random.default_rng(1)
    for _ in range(2000):
        ax, ay = np.exp(rng.uniform(np.log(1e-3), 0, 2))
        u1, u2 = rng.uniform(0, 1, 2)
        want = _ggx_inversion(ax, ay, u1, u2)
        for m in (CAP, HEITZ):
            h = orc.sample_vndf(m, [0, 0, 1], ax, ay, u1, u2)
            np.testing.assert_allclose(h, want, atol=1e-11)
        p = orc.pdf_vndf(want, [0, 0, 1], ax, ay)
        assert p == pytest.approx(_textbook_D(want, ax, ay) * want[2], rel=1e-9)


def test_isotropic_theta_closed_form(orc):
    """P3 (isotropic): theta_h = atan(alpha sqrt(u2 / (1 - u2)))."""
    for a in (1e-3, 0.05, 0.3, 1.0):
        for u2 in (0.0, 0.1, 0.5, 0.9, 1 - 2**-24):
            h = orc.sample_vndf(CAP, [0, 0, 1], a, a, 0.3, u2)
            assert np.arccos(h[2]) == pytest.approx(np.arctan(a * np.sqrt(u2 / (1 - u2))), abs=1e-9)


def test_alpha_one_pole_is_cosine_weighted(orc):
    """P4: alpha = (1,1), wi = pole: h = (sqrt(u2) cos, sqrt(u2) sin, sqrt(1-u2)), pdf = h.z/pi."""
    rng = np.random.default_rng(2)
    for u1, u2 in rng.uniform(0, 1, (500, 2)):
        h = orc.sample_vndf(CAP, [0, 0, 1], 1.0, 1.0, u1, u2)
        want = [np.sqrt(u2) * np.cos(2 * np.pi * u1), np.sqrt(u2) * np.sin(2 * np.pi * u1), np.sqrt(1 - u2)]
        np.testing.assert_allclose(h, want, atol=1e-12)
        assert orc.pdf_vndf(h, [0, 0, 1], 1, 1) == pytest.approx(h[2] / np.pi, rel=1e-12)


# ----------------------------------------------------------------- the pdf ---
def _rand_dir_upper(rng):
    v = rng.normal(size=3)
    v[2] = abs(v[2]) + 1e-3
    return v / np.linalg.norm(v)


def test_G1_smith_form_and_chi_plus(orc):
    """Eq. 16-17: G1(wm, wi) equals Heitz 2014's Smith masking
    1/(1 + Lambda(wi)) for every front-facing microfacet (wi.wm > 0, the same
    sign in std space since (M^-1 wi).(M^T wm) = wi.wm) and is 0 for
    back-facing ones (the chi+ factor)."""
    rng = np.random.default_rng(1617)
    front = back = 0
    for _ in range(400):
        ax, ay = np.exp(rng.uniform(np.log(0.01), 0.0, 2))
        wi = rng.normal(size=3)
        wi[2] = abs(wi[2]) + 1e-3
        wi /= np.linalg.norm(wi)
        wm = rng.normal(size=3)
        wm[2] = abs(wm[2]) + 1e-3
        wm /= np.linalg.norm(wm)
        g = orc.G1(wm, wi, ax, ay)
        if float(np.dot(wi, wm)) > 1e-9:
            assert g == pytest.approx(_textbook_G1(wi, ax, ay), rel=1e-9, abs=1e-12)
            front += 1
        elif float(np.dot(wi, wm)) < -1e-9:
            assert g == 0.0
            back += 1
    assert front > 50 and back > 50


def test_pdf_three_forms_agree(orc):
    """Eq. 1 == G1 max(0,wi.h) D / wi.z via Eq. 12 + Eq. 16-17
    == the textbook Smith/Lambda + theta/phi GGX forms (Heitz 2014)."""
    rng = np.random.default_rng(3)
    for _ in range(3000):
        wi = _rand_dir_upper(rng)
        h = _rand_dir_upper(rng)
        ax, ay = np.exp(rng.uniform(np.log(1e-2), 0, 2))
        p1 = orc.pdf_vndf(h, wi, ax, ay)
        p2 = orc.pdf_vndf_g1d(h, wi, ax, ay)
        p3 = _textbook_vndf(h, wi, ax, ay)
        assert p1 == pytest.approx(p2, rel=1e-9, abs=1e-300)
        assert p1 == pytest.approx(p3, rel=1e-8, abs=1e-300)


def test_pdf_support(orc):
    """D_std = 0 below the horizon (Eq. 3) and max(wm.wi, 0) (Eq. 2): pdf vanishes
    for h.z <= 0 and for back-facing h."""
    rng = np.random.default_rng(4)
    for _ in range(500):
        wi = _rand_dir_upper(rng)
        h = _rand_dir_upper(rng)
        ax, ay = np.exp(rng.uniform(np.log(1e-2), 0, 2))
        hb = h * np.array([1, 1, -1])
        assert orc.pdf_vndf(hb, wi, ax, ay) == 0.0
        if np.dot(h, wi) < 0:
            assert orc.pdf_vndf(h, wi, ax, ay) == 0.0


@pytest.mark.parametrize("wi_deg,ax,ay", [(0, 1, 1), (0, 0.5, 0.5), (45, 0.2, 0.2), (80, 0.5, 0.5),
                                          (70, 0.05, 0.3), (85, 0.3, 0.05), (60, 1.0, 0.1),
                                          (89.9, 0.1, 0.1)])
def test_pdf_normalises(orc, wi_deg, ax, ay):
    """The VNDF is a pdf over directions (Eq. 1 is a linearly transformed
    distribution): its integral over the hemisphere is 1.
    Catches dropped Jacobian / normalisation factors."""
    from oracle.stats import bin_masses
    t = np.radians(wi_deg)
    wi = [np.sin(t) * np.cos(0.4), np.sin(t) * np.sin(0.4), np.cos(t)]
    m = bin_masses(wi, ax, ay, nt=64, npb=64, q=16)
    assert m.sum() == pytest.approx(1.0, abs=2e-4)


# ------------------------------------------------------- sampler invariants ---
def _random_inputs(rng, n):
    out = []
    for k in range(n):
        kind = k % 4
        if kind == 0:
            wi = _rand_dir_upper(rng)
        elif kind == 1:  # grazing
            z = rng.uniform(1e-4, 0.05)
            p = rng.uniform(0, 2 * np.pi)
            wi = np.array([np.sqrt(1 - z * z) * np.cos(p), np.sqrt(1 - z * z) * np.sin(p), z])
        elif kind == 2:  # back side
            wi = _rand_dir_upper(rng) * np.array([1, 1, -1])
        else:  # non-unit incidence (P:419 normalises after the stretch)
            wi = _rand_dir_upper(rng) * rng.uniform(0.5, 2.0)
        ax, ay = rng.choice([1e-3, 0.05, 0.3, 1.0], 2) if k % 3 == 0 else np.exp(rng.uniform(np.log(1e-3), 0, 2))
        u1, u2 = rng.uniform(0, 1, 2)
        if k % 17 == 0:
            u2 = 1 - 2**-24
        if k % 19 == 0:
            u1 = 0.0
        if k % 23 == 0:
            u2 = 0.0
        out.append((wi, ax, ay, u1, u2))
    return out


@pytest.mark.parametrize("method", [CAP, HEITZ])
def test_sampler_invariants(orc, method):
    """P6: |h| = 1, s h.z >= 0, wi.h >= 0 (visible normal), for grazing, back-side,
    non-unit incidence and alpha down to 1e-3."""
    rng = np.random.default_rng(5 + method)
    for wi, ax, ay, u1, u2 in _random_inputs(rng, 4000):
        h = orc.sample_vndf(method, wi, ax, ay, u1, u2)
        s = -1.0 if wi[2] < 0 else 1.0
        assert abs(np.linalg.norm(h) - 1) < 1e-12
        assert s * h[2] >= -1e-12
        assert np.dot(wi, h) >= -1e-12 * np.linalg.norm(wi)


def test_cap_inverse_map(orc):
    """Per-sample pin of Listing 1 + Listing 3 away from normal incidence.
    Undo the unstretch with M^T, reflect ws about the std-space
    normal (Eq. 5): the result must be the cap direction c with
    c.z = (1 - u2)(1 + ws.z) - ws.z and azimuth 2 pi u1.  Catches a
    transposed warp, swapped uniforms and sign errors."""
    rng = np.random.default_rng(6)
    checked = 0
    for wi, ax, ay, u1, u2 in _random_inputs(rng, 4000):
        h = orc.sample_vndf(CAP, wi, ax, ay, u1, u2)
        s = -1.0 if wi[2] < 0 else 1.0
        w = s * np.asarray(wi)
        ws = np.array([ax * w[0], ay * w[1], w[2]])
        ws /= np.linalg.norm(ws)
        hh = s * h
        hs = np.array([hh[0] / ax, hh[1] / ay, hh[2]])
        hs /= np.linalg.norm(hs)
        c = 2 * np.dot(hs, ws) * hs - ws
        zc = (1 - u2) * (1 + ws[2]) - ws[2]
        cond = np.linalg.norm(hs * 0 + (c + ws))  # |c + ws| = |hs_unnormalised|
        if cond < 1e-3:
            continue  # c ~ -ws: the reflection is ill-conditioned
        checked += 1
        tol = 1e-9 * max(ax, ay) / min(ax, ay) / cond
        assert c[2] == pytest.approx(zc, abs=max(tol, 1e-10))
        st = np.hypot(c[0], c[1])
        if st > 1e-4:
            dphi = np.angle(np.exp(1j * (np.arctan2(c[1], c[0]) - 2 * np.pi * u1)))
            assert abs(dphi) < max(tol / st, 1e-9)
    assert checked > 3900


def test_flip_reading(orc):
    """Reading R4 (BASELINE config 5): wi.z < 0 is sampled on the flipped
    hemisphere by whole-vector negation and flipped back; pdf(h|wi) = pdf(-h|-wi).
    wi.z = -0.0 counts as the upper side."""
    rng = np.random.default_rng(7)
    for _ in range(500):
        wi = _rand_dir_upper(rng) * np.array([1, 1, -1])
        ax, ay = np.exp(rng.uniform(np.log(1e-3), 0, 2))
        u1, u2 = rng.uniform(0, 1, 2)
        for m in (CAP, HEITZ):
            h = orc.sample_vndf(m, wi, ax, ay, u1, u2)
            g = orc.sample_vndf(m, -wi, ax, ay, u1, u2)
            np.testing.assert_array_equal(h, -g)
        assert orc.pdf_vndf(h, wi, ax, ay) == orc.pdf_vndf(-h, -wi, ax, ay)
    a = orc.sample_vndf(CAP, [0.6, 0.8, -0.0], 0.3, 0.3, 0.2, 0.7)
    b = orc.sample_vndf(CAP, [0.6, 0.8, 0.0], 0.3, 0.3, 0.2, 0.7)
    np.testing.assert_array_equal(a, b)


def test_deferred_normalisation_identity(orc):
    """normalising the half vector before the unstretch changes nothing."""
    rng = np.random.default_rng(8)
    for wi, ax, ay, u1, u2 in _random_inputs(rng, 1000):
        if wi[2] < 0:
            continue
        ws = np.array([ax * wi[0], ay * wi[1], wi[2]])
        ws /= np.linalg.norm(ws)
        hs = orc.sample_hemisphere(CAP, u1, u2, ws)
        if np.linalg.norm(hs) < 1e-6:
            continue
        hn = hs / np.linalg.norm(hs)
        a = np.array([ax * hs[0], ay * hs[1], hs[2]])
        b = np.array([ax * hn[0], ay * hn[1], hn[2]])
        np.testing.assert_allclose(a / np.linalg.norm(a), b / np.linalg.norm(b), atol=1e-12)
        np.testing.assert_allclose(orc.sample_vndf(CAP, wi, ax, ay, u1, u2), a / np.linalg.norm(a),
                                   atol=1e-8)


@pytest.mark.parametrize("entry", GOLD["fig4_cap_bottom"])
def test_fig4_cap_support(orc, entry):
    """Fig. 4: a hemispherical mirror reflects parallel rays into a cap
    cut at z = -cos(theta_i).  Native Listing 3 (no flip), alpha = 1 (std space):
    c = h - wi must lie in (-cos theta_i, 1] and approach the cut as u2 -> 1."""
    t = np.radians(entry["theta_i_deg"])
    wi = np.array([np.sin(t), 0.0, np.cos(t)])
    bottom = -np.cos(t)
    assert bottom == pytest.approx(entry["cap_bottom_z"], abs=1e-7)  # the figure's label
    zmin = 1.0
    rng = np.random.default_rng(9)
    for u1, u2 in np.vstack([rng.uniform(0, 1, (3000, 2)), [[0.3, 1 - 2**-24], [0.9, 1 - 1e-12]]]):
        c = orc.sample_hemisphere(CAP, u1, u2, wi) - wi
        assert abs(np.linalg.norm(c) - 1) < 1e-12
        assert c[2] > bottom - 1e-12
        zmin = min(zmin, c[2])
        h = orc.sample_hemisphere(CAP, u1, u2, wi)
        assert h[2] >= -1e-12 and np.dot(h, wi) >= -1e-12  # visible upper normals
    assert zmin == pytest.approx(bottom, abs=1e-6)


# ------------------------------------------------------ reflection machinery --
def test_reflect_half_vector_round_trip(orc):
    """Eq. 5 and Eq. 6 are inverse on visible normals."""
    rng = np.random.default_rng(10)
    for _ in range(1000):
        wi, wm = _rand_dir_upper(rng), _rand_dir_upper(rng)
        if np.dot(wi, wm) <= 1e-3:
            continue
        wo = orc.reflect(wi, wm)
        assert abs(np.linalg.norm(wo) - 1) < 1e-12
        np.testing.assert_allclose(orc.half_vector(wi, wo), wm, atol=1e-10)


def test_reflection_jacobian_finite_difference(orc):
    """Eq. 8 against the finite-difference solid-angle ratio of the
    map wo -> half_vector(wi, wo)."""
    rng = np.random.default_rng(11)
    for _ in range(100):
        wi = _rand_dir_upper(rng)
        wo = _rand_dir_upper(rng)
        if np.linalg.norm(wi + wo) < 0.2:
            continue
        e1 = np.cross(wo, [0.3, 0.5, 0.8]); e1 /= np.linalg.norm(e1)
        e2 = np.cross(wo, e1)
        eps = 1e-5

        def H(v):
            return orc.half_vector(wi, v / np.linalg.norm(v))
        h0 = H(wo)
        d1 = (H(wo + eps * e1) - H(wo - eps * e1)) / (2 * eps)
        d2 = (H(wo + eps * e2) - H(wo - eps * e2)) / (2 * eps)
        ratio = np.linalg.norm(np.cross(d1, d2))
        assert ratio == pytest.approx(orc.reflect_jacobian(wo, h0), rel=1e-4)


@pytest.mark.parametrize("zi", [-0.5, 0.0, 0.5, 1.0])
def test_cap_density_integrates_to_one(orc, zi):
    """Eq. 10's constant is 1/solid angle of the cap: integrate f_p
    over the sphere by midpoint quadrature in (z, phi) (uniform-area coordinates)."""
    wi = np.array([np.sqrt(1 - zi * zi), 0.0, zi])
    nz, nphi = 400, 64
    tot = 0.0
    for z in (np.arange(nz) + 0.5) / nz * 2 - 1:
        for p in (np.arange(nphi) + 0.5) / nphi * 2 * np.pi:
            r = np.sqrt(1 - z * z)
            tot += orc.cap_density([r * np.cos(p), r * np.sin(p), z], wi)
    tot *= (2.0 / nz) * (2 * np.pi / nphi)
    assert tot == pytest.approx(1.0, abs=1.5 / nz * (1 + abs(zi)) + 1e-9)


def test_heitz_inverse_map(orc):
    """Per-sample pin of Listing 1 + Listing 2 away from normal
    incidence: undo the unstretch (M^T), express the std-space
    normal in the basis (w1, w2, ws) of P:435-438 and check the disk
    parameterisation: t1 = sqrt(u2) cos(2 pi u1) and
    t2 = (1 - s) sqrt(1 - t1^2) + s sqrt(u2) sin(2 pi u1), s = (1 + ws.z)/2
    (P:443-445).  Catches a swapped or mis-signed basis vector, swapped
    uniforms and a wrong warp of the cross section."""
    rng = np.random.default_rng(12)
    checked = 0
    for wi, ax, ay, u1, u2 in _random_inputs(rng, 3000):
        h = orc.sample_vndf(HEITZ, wi, ax, ay, u1, u2)
        sgn = -1.0 if wi[2] < 0 else 1.0
        w = sgn * np.asarray(wi)
        ws = np.array([ax * w[0], ay * w[1], w[2]])
        ws /= np.linalg.norm(ws)
        hh = sgn * h
        hs = np.array([hh[0] / ax, hh[1] / ay, hh[2]])
        hs /= np.linalg.norm(hs)
        tmp = ws[0] ** 2 + ws[1] ** 2
        if tmp < 1e-12:
            continue
        w1 = np.array([-ws[1], ws[0], 0.0]) / np.sqrt(tmp)
        w2 = np.cross(ws, w1)
        t1, t2 = hs @ w1, hs @ w2
        r = np.sqrt(u2)
        s = (1 + ws[2]) / 2
        want_t1 = r * np.cos(2 * np.pi * u1)
        want_t2 = (1 - s) * np.sqrt(max(1 - want_t1 ** 2, 0)) + s * r * np.sin(2 * np.pi * u1)
        cond = max(ax, ay) / min(ax, ay)
        assert t1 == pytest.approx(want_t1, abs=1e-8 * cond)
        assert t2 == pytest.approx(want_t2, abs=1e-8 * cond)
        checked += 1
    assert checked > 2500
