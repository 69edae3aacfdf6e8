"""Chi-square machinery for the distributional tests (test infrastructure).

Histogram layout (reading R14): 64 x 64
bins in (theta, phi) of the sampled normal h, theta uniform on [0, pi/2],
phi uniform on [0, 2 pi).  Expected bin masses come from 16 x 16
Gauss-Legendre quadrature of the oracle's Eq. 1 pdf times the
solid-angle Jacobian sin(theta).  Bins with expected count < 5 are pooled
into one bin; the test passes when the Pearson p-value exceeds 1e-3.
"""
from __future__ import annotations

import numpy as np
from scipy import stats as _st

from . import batch_pdf, batch_pdf_native

NT = 64
NP = 64


def bin_masses(wi, ax: float, ay: float, nt: int = NT, npb: int = NP, q: int = 16,
               native: bool = False) -> np.ndarray:
    """Quadrature of pdf(h | wi) sin(theta) over each (theta, phi) bin (upper
    hemisphere of h).  native=True evaluates Eq. 1 without the flip (NEXT-3)."""
    x, w = np.polynomial.legendre.leggauss(q)
    tb = np.linspace(0.0, np.pi / 2, nt + 1)
    pb = np.linspace(0.0, 2 * np.pi, npb + 1)
    # nodes per bin
    th = (0.5 * (tb[1:] - tb[:-1]))[:, None] * x[None, :] + (0.5 * (tb[1:] + tb[:-1]))[:, None]
    ph = (0.5 * (pb[1:] - pb[:-1]))[:, None] * x[None, :] + (0.5 * (pb[1:] + pb[:-1]))[:, None]
    wt = (0.5 * (tb[1] - tb[0])) * w
    wp = (0.5 * (pb[1] - pb[0])) * w
    T = th.reshape(-1)  # nt*q
    P = ph.reshape(-1)  # np*q
    TT, PP = np.meshgrid(T, P, indexing="ij")
    st = np.sin(TT)
    h = np.stack([st * np.cos(PP), st * np.sin(PP), np.cos(TT)]).reshape(3, -1)
    wi = np.asarray(wi, dtype=np.float64).reshape(3, 1)
    if native:
        f = batch_pdf_native(h, wi[:, 0], ax, ay).reshape(TT.shape) * st
    else:
        f = batch_pdf(h, np.repeat(wi, h.shape[1], axis=1), ax, ay).reshape(TT.shape) * st
    f = f.reshape(nt, q, npb, q)
    m = np.einsum("aibj,i,j->ab", f, wt, wp)
    return m


def histogram(h: np.ndarray, nt: int = NT, npb: int = NP) -> np.ndarray:
    h = np.asarray(h, dtype=np.float64).reshape(3, -1)
    th = np.arccos(np.clip(h[2] / np.linalg.norm(h, axis=0), -1.0, 1.0))
    ph = np.mod(np.arctan2(h[1], h[0]), 2 * np.pi)
    it = np.clip((th / (np.pi / 2) * nt).astype(np.int64), 0, nt - 1)
    ip = np.clip((ph / (2 * np.pi) * npb).astype(np.int64), 0, npb - 1)
    out = np.zeros((nt, npb), dtype=np.int64)
    np.add.at(out, (it, ip), 1)
    return out


def pearson(counts: np.ndarray, masses: np.ndarray, min_expected: float = 5.0):
    """Pearson chi-square with pooling of low-expectation bins.  Returns (chi2, dof, p)."""
    c = np.asarray(counts, dtype=np.float64).reshape(-1)
    m = np.asarray(masses, dtype=np.float64).reshape(-1)
    n = c.sum()
    m = m / m.sum()  # quadrature mass is 1 to ~1e-6; renormalise exactly
    e = n * m
    keep = e >= min_expected
    cc = list(c[keep]) + ([c[~keep].sum()] if (~keep).any() else [])
    ee = list(e[keep]) + ([e[~keep].sum()] if (~keep).any() else [])
    cc, ee = np.asarray(cc), np.asarray(ee)
    ok = ee > 0
    chi2 = float(((cc[ok] - ee[ok]) ** 2 / ee[ok]).sum())
    dof = int(ok.sum() - 1)
    return chi2, dof, float(_st.chi2.sf(chi2, dof))


def two_sample(c1: np.ndarray, c2: np.ndarray, min_expected: float = 5.0):
    """Chi-square homogeneity test of two histograms (pooling sparse bins)."""
    a = np.asarray(c1, dtype=np.float64).reshape(-1)
    b = np.asarray(c2, dtype=np.float64).reshape(-1)
    na, nb = a.sum(), b.sum()
    tot = a + b
    ea = tot * na / (na + nb)
    eb = tot * nb / (na + nb)
    keep = (ea >= min_expected) & (eb >= min_expected)
    A = list(a[keep]) + ([a[~keep].sum()] if (~keep).any() else [])
    B = list(b[keep]) + ([b[~keep].sum()] if (~keep).any() else [])
    A, B = np.asarray(A), np.asarray(B)
    T = A + B
    EA, EB = T * na / (na + nb), T * nb / (na + nb)
    ok = T > 0
    chi2 = float((((A - EA) ** 2 / EA)[ok]).sum() + (((B - EB) ** 2 / EB)[ok]).sum())
    dof = int(ok.sum() - 1)
    return chi2, dof, float(_st.chi2.sf(chi2, dof))


def sphere_bin_masses(pdf_dirs, nz: int = 32, nphi: int = 64, q: int = 12) -> np.ndarray:
    """Masses of a density over the whole sphere in nz x nphi bins of
    (z = cos theta uniform on [-1, 1], phi uniform on [0, 2 pi)), by q x q
    Gauss-Legendre per bin (z is the uniform-area coordinate).  pdf_dirs maps a
    (3, k) array of unit directions to k densities."""
    x, w = np.polynomial.legendre.leggauss(q)
    zb = np.linspace(-1.0, 1.0, nz + 1)
    pb = np.linspace(0.0, 2 * np.pi, nphi + 1)
    zz = (0.5 * (zb[1:] - zb[:-1]))[:, None] * x[None, :] + (0.5 * (zb[1:] + zb[:-1]))[:, None]
    pp = (0.5 * (pb[1:] - pb[:-1]))[:, None] * x[None, :] + (0.5 * (pb[1:] + pb[:-1]))[:, None]
    Z, P = np.meshgrid(zz.reshape(-1), pp.reshape(-1), indexing="ij")
    r = np.sqrt(np.clip(1 - Z * Z, 0, None))
    d = np.stack([r * np.cos(P), r * np.sin(P), Z]).reshape(3, -1)
    f = pdf_dirs(d).reshape(nz, q, nphi, q)
    return np.einsum("aibj,i,j->ab", f, 0.5 * (zb[1] - zb[0]) * w, 0.5 * (pb[1] - pb[0]) * w)


def sphere_histogram(v: np.ndarray, nz: int = 32, nphi: int = 64) -> np.ndarray:
    v = np.asarray(v, dtype=np.float64).reshape(3, -1)
    v = v / np.linalg.norm(v, axis=0)
    iz = np.clip(((v[2] + 1) * 0.5 * nz).astype(np.int64), 0, nz - 1)
    ip = np.clip((np.mod(np.arctan2(v[1], v[0]), 2 * np.pi) / (2 * np.pi) * nphi).astype(np.int64), 0, nphi - 1)
    out = np.zeros((nz, nphi), dtype=np.int64)
    np.add.at(out, (iz, ip), 1)
    return out
