"""Distribution pins of the seeded input recipes (BASELINE.json configs;
SURVEY.md s.8(d); DESIGN.md s.5, readings R12 / R16).

The recipes are prose in BASELINE.json ("wi uniform on the upper hemisphere",
"cosine-weighted", "log-uniform [a, b]", the config-5 mix).  Each is pinned here
by what the prose fixes, independently of the formulas that generate it:
  * uniform on the upper hemisphere  <=>  z = cos(theta) ~ U(0, 1] and the
    azimuth ~ U[0, 2 pi), independent (Archimedes: equal-height zones have
    equal area);
  * cosine-weighted                  <=>  z^2 ~ U(0, 1] (p(z) = 2z on [0, 1]);
  * log-uniform [a, b]               <=>  log(alpha / a) / log(b / a) ~ U[0, 1);
  * the method's uniforms u1, u2 ~ U[0, 1) and independent of the scene.
Kolmogorov-Smirnov tests on 2^17 samples (a mutant such as cosine-weighted wi
in config 4, or a swapped log-uniform range, fails at p < 1e-30), plus a
16 x 16 chi-square test of joint uniformity for pairs that must be independent.
"""
import numpy as np
import pytest
from scipy import stats

N = 1 << 17
P_MIN = 1e-4   # fixed seeds: deterministic; a correct recipe sits far above


def _ks_uniform(x, lo=0.0, hi=1.0):
    return stats.kstest(np.asarray(x, dtype=np.float64), "uniform", args=(lo, hi - lo)).pvalue


def _joint_uniform_p(a, b, bins=16):
    h, _, _ = np.histogram2d(a, b, bins=bins, range=[[0, 1], [0, 1]])
    e = h.sum() / bins**2
    chi2 = ((h - e) ** 2 / e).sum()
    return stats.chi2.sf(chi2, bins * bins - 1)


def _azimuth01(x, y):
    return np.mod(np.arctan2(y, x), 2 * np.pi) / (2 * np.pi)


# ------------------------------------------------------------------ config 4 --
@pytest.fixture(scope="module")
def c4(orc):
    return orc.batch_c4_inputs(3, np.arange(N, dtype=np.uint64))


def test_c4_wi_uniform_upper_hemisphere(c4):
    wx, wy, wz = c4[0], c4[1], c4[2]
    assert np.all(wz > 0.0)
    np.testing.assert_allclose(wx * wx + wy * wy + wz * wz, 1.0, atol=1e-14)
    assert _ks_uniform(1.0 - wz) > P_MIN                      # z ~ U(0, 1]
    assert _ks_uniform(_azimuth01(wx, wy)) > P_MIN            # phi ~ U[0, 2 pi)
    assert _joint_uniform_p(1.0 - wz, _azimuth01(wx, wy)) > P_MIN


def test_c4_wi_not_cosine_weighted(c4):
    """Power: the cosine-weighted law (z^2 uniform) is rejected on the same data."""
    assert _ks_uniform(c4[2] ** 2) < 1e-30


@pytest.mark.parametrize("row", [3, 4])
def test_c4_alpha_log_uniform(c4, row):
    a = c4[row]
    assert a.min() >= 0.01 and a.max() <= 1.0
    assert _ks_uniform(np.log(a / 0.01) / np.log(100.0)) > P_MIN
    # power: the config-3 range [0.001, 1] would be rejected
    assert _ks_uniform(np.log(a / 0.001) / np.log(1000.0)) < 1e-30


def test_c4_alpha_axes_independent(c4):
    lx = np.log(c4[3] / 0.01) / np.log(100.0)
    ly = np.log(c4[4] / 0.01) / np.log(100.0)
    assert _joint_uniform_p(lx, ly) > P_MIN
    assert abs(np.corrcoef(lx, ly)[0, 1]) < 0.02


def test_c4_method_uniforms(c4):
    u1, u2 = c4[5], c4[6]
    for u in (u1, u2):
        assert u.min() >= 0.0 and u.max() < 1.0
        assert _ks_uniform(u) > P_MIN
        # 24-bit grid (u(w) = (w >> 8) 2^-24, exact in binary32)
        assert np.all(np.float32(u) == u) and np.all(np.mod(u * 2**24, 1.0) == 0.0)
    assert _joint_uniform_p(u1, u2) > P_MIN
    # the method's uniforms are independent of the scene (wi, alpha)
    assert _joint_uniform_p(u1, 1.0 - c4[2]) > P_MIN
    assert _joint_uniform_p(u2, _azimuth01(c4[0], c4[1])) > P_MIN
    assert _joint_uniform_p(u1, np.log(c4[3] / 0.01) / np.log(100.0)) > P_MIN


def test_c4_scene_uniforms_carry_24_bits(c4):
    """SURVEY s.8(d): the incidence uniforms are 24-bit (the round-1 variant drew
    them on a 2^16 grid): 1 - z takes (almost) N distinct values."""
    assert np.unique(1.0 - c4[2]).size > 0.99 * N
    assert np.unique(_azimuth01(c4[0], c4[1])).size > 0.99 * N


def test_c4_word_layout(orc):
    """Bit layout of SURVEY s.8(d): X = block 0 -> wi, alpha; Y = block 1 -> u1, u2."""
    idx = np.array([0, 1, 2**20 + 3, 2**32 - 1, 2**32, 2**33 + 7], dtype=np.uint64)
    v = orc.batch_c4_inputs(3, idx)
    X = orc.philox_words(3, idx, 0)
    Y = orc.philox_words(3, idx, 1)
    u = lambda w: (w >> 8).astype(np.float64) * 2.0**-24
    np.testing.assert_array_equal(v[5], u(Y[:, 0]))
    np.testing.assert_array_equal(v[6], u(Y[:, 1]))
    np.testing.assert_array_equal(v[2], 1.0 - u(X[:, 0]))
    np.testing.assert_allclose(_azimuth01(v[0], v[1]), u(X[:, 1]), atol=1e-12)
    np.testing.assert_allclose(np.log(v[3] / 0.01) / np.log(100.0), u(X[:, 2]), atol=1e-12)
    np.testing.assert_allclose(np.log(v[4] / 0.01) / np.log(100.0), u(X[:, 3]), atol=1e-12)


# --------------------------------------------------- streamed configs (synth) --
@pytest.fixture(scope="module")
def planes():
    import synth
    return {cid: synth.fill_numpy(synth.CONFIGS[cid].recipe, synth.CONFIGS[cid].seed, N)
            for cid in (1, 2, 3, 5)}


def _f64(x):
    return np.asarray(x, dtype=np.float64)


@pytest.mark.parametrize("cid", [1, 3])
def test_synth_uniform_upper_hemisphere(planes, cid):
    p = planes[cid]
    wx, wy, wz = _f64(p["wi_x"]), _f64(p["wi_y"]), _f64(p["wi_z"])
    assert np.all(wz > 0.0)
    np.testing.assert_allclose(wx * wx + wy * wy + wz * wz, 1.0, atol=1e-6)
    assert _ks_uniform(1.0 - wz) > P_MIN
    assert _ks_uniform(_azimuth01(wx, wy)) > P_MIN
    assert _ks_uniform(wz ** 2) < 1e-30            # not cosine-weighted


def test_synth_config2_cosine_weighted(planes):
    p = planes[2]
    wx, wy, wz = _f64(p["wi_x"]), _f64(p["wi_y"]), _f64(p["wi_z"])
    assert np.all(wz > 0.0)
    assert _ks_uniform(wz ** 2) > P_MIN            # p(z) = 2z
    assert _ks_uniform(_azimuth01(wx, wy)) > P_MIN
    assert _ks_uniform(1.0 - wz) < 1e-30           # not uniform-hemisphere


@pytest.mark.parametrize("cid,lo", [(2, 0.01), (3, 0.001)])
def test_synth_alpha_log_uniform(planes, cid, lo):
    for k in ("alpha_x", "alpha_y"):
        a = _f64(planes[cid][k])
        assert a.min() >= lo * (1 - 1e-6) and a.max() <= 1.0 + 1e-6
        assert _ks_uniform(np.log(a / lo) / np.log(1.0 / lo)) > 1e-3
    lx = np.log(_f64(planes[cid]["alpha_x"]) / lo) / np.log(1.0 / lo)
    ly = np.log(_f64(planes[cid]["alpha_y"]) / lo) / np.log(1.0 / lo)
    assert _joint_uniform_p(np.clip(lx, 0, 1 - 1e-12), np.clip(ly, 0, 1 - 1e-12)) > P_MIN


def test_synth_config1_isotropic_half(planes):
    assert np.all(planes[1]["alpha_x"] == np.float32(0.5))
    assert np.all(planes[1]["alpha_y"] == np.float32(0.5))


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_synth_method_uniforms(planes, cid):
    p = planes[cid]
    u1, u2 = _f64(p["u1"]), _f64(p["u2"])
    assert _ks_uniform(u1) > P_MIN and _ks_uniform(u2) > P_MIN
    assert _joint_uniform_p(u1, u2) > P_MIN
    wz = _f64(p["wi_z"])
    scene = wz ** 2 if cid == 2 else 1.0 - wz      # the uniform behind wi.z
    assert _joint_uniform_p(u1, scene) > P_MIN
    assert _joint_uniform_p(u2, _azimuth01(_f64(p["wi_x"]), _f64(p["wi_y"]))) > P_MIN


def test_synth_config5_edge_mix(planes):
    """BASELINE config 5: 40% grazing z in [1e-4, 0.05], 20% below the horizon,
    40% uniform upper; alpha per axis from {1e-3, .05, .3, 1} uniformly and
    independently; u1 = 0, u2 = 0 and the rim u2 = 1 - 2^-24 injected 1/64 each
    (the rim rule wins over u2 = 0)."""
    p = planes[5]
    wz = _f64(p["wi_z"])
    n = wz.size
    below = wz < 0
    band = (wz >= 1e-4) & (wz <= 0.05)

    def binom_ok(count, prob):
        return stats.binomtest(int(count), n, prob).pvalue > P_MIN

    assert binom_ok(below.sum(), 0.2)
    # grazing (all of it in the band) + the uniform-upper share that falls in it
    assert binom_ok(band.sum(), 0.4 + 0.4 * (0.05 - 1e-4))
    assert _ks_uniform(-wz[below]) > P_MIN                      # back side: -z ~ U(0, 1]
    up = ~below & ~band
    # uniform-upper outside the band: 1 - z uniform on [0, 0.95)
    assert _ks_uniform(1.0 - wz[up & (wz > 0.05)], 0.0, 0.95) > P_MIN
    # grazing z is uniform in its band (the upper share there is uniform too)
    assert _ks_uniform(wz[band], 1e-4, 0.05) > P_MIN
    T = np.array([1e-3, 0.05, 0.3, 1.0], dtype=np.float32)
    for k in ("alpha_x", "alpha_y"):
        a = p[k]
        assert np.all(np.isin(a, T))
        cnt = np.array([(a == t).sum() for t in T])
        assert stats.chisquare(cnt).pvalue > P_MIN
    jx = np.searchsorted(T, p["alpha_x"])
    jy = np.searchsorted(T, p["alpha_y"])
    tab = np.zeros((4, 4))
    np.add.at(tab, (jx, jy), 1)
    assert stats.chi2_contingency(tab).pvalue > P_MIN
    u1, u2 = _f64(p["u1"]), _f64(p["u2"])
    assert binom_ok((u1 == 0.0).sum(), 1 / 64)
    assert binom_ok((u2 == 0.0).sum(), (1 / 64) * (63 / 64))
    assert binom_ok((u2 == 1.0 - 2.0**-24).sum(), 1 / 64)
    rest = (u1 > 0) & (u2 > 0) & (u2 < 1 - 2.0**-24)
    assert _ks_uniform(u1[rest]) > P_MIN and _ks_uniform(u2[rest]) > P_MIN
