"""Distributional pins of the oracle samplers.

* The theorem (Eq. 10) and its corollary: cap samples are
  distributed as the VNDF, Eq. 1.  Pinned by a chi-square test of
  oracle cap samples against quadrature masses of the analytic pdf (which is
  itself pinned by tests/test_oracle_closed_forms.py).
* Listing 2 (Heitz) samples the same distribution.
* The brute-force ray-cast sampler built from the DEFINITION of the VNDF
   agrees with the analytic pdf and with the cap sampler.
* Power: the test rejects a 3% roughness error.
Histogram layout: reading R14 (oracle/stats.py).
"""
import numpy as np
import pytest

from oracle import stats

CAP, HEITZ = 0, 1
# (theta_i deg, phi_i deg; ax, ay) -- BASELINE config 2's eight chi-square pairs
PAIRS = [(0, 0, 1, 1), (0, 0, .5, .5), (45, 0, .2, .2), (80, 30, .5, .5),
         (70, 20, .05, .3), (85, 60, .3, .05), (45, 0, .01, .01), (60, 135, 1, .1)]
N = 1 << 20


def _wi(t, p):
    t, p = np.radians(t), np.radians(p)
    return np.array([np.sin(t) * np.cos(p), np.sin(t) * np.sin(p), np.cos(t)])


def _samples(orc, method, wi, ax, ay, n, seed):
    rng = np.random.default_rng(seed)
    u = rng.random((2, n), dtype=np.float32)
    wi32 = np.asarray(wi, dtype=np.float32)
    planes = [np.full(n, wi32[0]), np.full(n, wi32[1]), np.full(n, wi32[2]),
              np.full(n, ax, np.float32), np.full(n, ay, np.float32), u[0], u[1]]
    h, _, _ = orc.batch_sample(method, *planes, pdf=False)
    return h, wi32.astype(np.float64)


_MASS = {}


def _masses(wi, ax, ay):
    key = (tuple(np.round(wi, 12)), ax, ay)
    if key not in _MASS:
        _MASS[key] = stats.bin_masses(wi, ax, ay)
    return _MASS[key]


@pytest.mark.parametrize("pair", PAIRS, ids=[f"{p}" for p in PAIRS])
@pytest.mark.parametrize("method", [CAP, HEITZ], ids=["cap", "heitz"])
def test_chi2_against_analytic_vndf(orc, pair, method):
    t, p, ax, ay = pair
    h, wi = _samples(orc, method, _wi(t, p), ax, ay, N, seed=1000 + 7 * method + PAIRS.index(pair))
    chi2, dof, pv = stats.pearson(stats.histogram(h), _masses(wi, ax, ay))
    assert pv > 1e-3, (chi2, dof, pv)


@pytest.mark.parametrize("pair", [(0, 0, .5, .5), (70, 20, .05, .3), (60, 135, 1, .1), (85, 60, .3, .05)])
def test_raycast_definition_matches_analytic_and_cap(orc, pair):
    t, p, ax, ay = pair
    wi = _wi(t, p)
    n = 1 << 18
    hr, trials = orc.batch_raycast(wi, ax, ay, seed=77, n=n)
    assert trials >= n
    _, _, pv = stats.pearson(stats.histogram(hr), _masses(wi, ax, ay))
    assert pv > 1e-3
    hc, _ = _samples(orc, CAP, wi, ax, ay, n, seed=5)
    _, _, pv2 = stats.two_sample(stats.histogram(hr), stats.histogram(hc))
    assert pv2 > 1e-3


def test_chi2_has_power(orc):
    """A 3% roughness error must be rejected."""
    wi = _wi(45, 0)
    h, wi32 = _samples(orc, CAP, wi, 0.2, 0.2, N, seed=3)
    _, _, pv = stats.pearson(stats.histogram(h), stats.bin_masses(wi32, 0.206, 0.206))
    assert pv < 1e-6
    # and a swapped anisotropy is rejected outright
    h, wi32 = _samples(orc, CAP, _wi(70, 20), 0.05, 0.3, N, seed=4)
    _, _, pv = stats.pearson(stats.histogram(h), stats.bin_masses(wi32, 0.3, 0.05))
    assert pv < 1e-12


@pytest.mark.parametrize("method", [CAP, HEITZ], ids=["cap", "heitz"])
@pytest.mark.parametrize("theta", [0, 40, 75, 89])
def test_reflected_directions_fill_the_cap_uniformly(orc, method, theta):
    """Eq. 10: reflecting wi about visible normals of the hemisphere
    (std space, alpha = 1) gives z_o uniform on (-z_i, 1] and phi_o uniform.
    A real test for Listing 2; for Listing 3 it checks the implementation."""
    from scipy import stats as st
    wi = _wi(theta, 30)
    n = 1 << 18
    h, wi = _samples(orc, method, wi, 1.0, 1.0, n, seed=11 + theta)
    d = (h * wi[:, None]).sum(0)
    wo = 2 * d * h - wi[:, None]
    zi = wi[2]
    zo = wo[2]
    assert zo.min() > -zi - 1e-6
    pz = st.kstest((zo + zi) / (1 + zi), "uniform").pvalue
    pp = st.kstest(np.mod(np.arctan2(wo[1], wo[0]), 2 * np.pi) / (2 * np.pi), "uniform").pvalue
    assert pz > 1e-3 and pp > 1e-3, (pz, pp)
