"""Float64 CPU oracle for GGX VNDF spherical-cap sampling (arXiv 2306.05044).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package.  It shares no code with the CUDA path in
``paper_2306_05044_b200/`` and never imports it.

The arithmetic lives in ``oracle.c`` (plain C, float64, every function cites
the PAPER.md passage it follows); this module only loads it with ctypes and
marshals numpy arrays.  ``stats.py`` holds the chi-square / quadrature
machinery used by the distributional tests.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# Plain scalar float64 build: -O2, no -ffast-math, no vectorisation tricks
# that could change rounding (-ffp-contract=off keeps a*b+c as two roundings
# unless the source calls fma() explicitly, as Listing 3 line 6 does).
CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-ffp-contract=off"]


def _stale() -> bool:
    return not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC)


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc).  Returns the library path.
    Concurrent callers (several processes) serialise on a lock file."""
    import fcntl
    if not (force or _stale()):
        return _LIB
    with open(_LIB + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if force or _stale():
            cmd = ["gcc", *CFLAGS, _SRC, "-o", _LIB + ".tmp", "-lquadmath", "-lm"]
            subprocess.run(cmd, check=True)
            os.replace(_LIB + ".tmp", _LIB)
        fcntl.flock(lk, fcntl.LOCK_UN)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        d, u32, u64, i64, i32 = (ctypes.c_double, ctypes.c_uint32, ctypes.c_uint64,
                                  ctypes.c_int64, ctypes.c_int)
        P = ctypes.c_void_p
        L.orc_philox4x32_10.argtypes = [P, P, P]
        L.orc_philox_block.argtypes = [u64, u64, u32, P]
        L.orc_u01.argtypes = [u32]
        L.orc_u01.restype = d
        L.orc_sample_vndf.argtypes = [i32, P, d, d, d, d, P, P]
        L.orc_sample_hemisphere.argtypes = [i32, d, d, P, P]
        for name in ("orc_sigma_std", "orc_D_std"):
            getattr(L, name).argtypes = [d]
            getattr(L, name).restype = d
        L.orc_Dvis_std.argtypes = [P, P]
        L.orc_Dvis_std.restype = d
        for name in ("orc_pdf_vndf", "orc_pdf_vndf_g1d", "orc_G1"):
            getattr(L, name).argtypes = [P, P, d, d]
            getattr(L, name).restype = d
        L.orc_D_ggx.argtypes = [P, d, d]
        L.orc_D_ggx.restype = d
        L.orc_reflect.argtypes = [P, P, P]
        L.orc_half_vector.argtypes = [P, P, P]
        L.orc_reflect_jacobian.argtypes = [P, P]
        L.orc_reflect_jacobian.restype = d
        L.orc_cap_density.argtypes = [P, P]
        L.orc_cap_density.restype = d
        L.orc_sample_raycast.argtypes = [P, d, d, u64, u64, P]
        L.orc_sample_raycast.restype = u64
        L.orc_c4_inputs.argtypes = [u64, u64, P]
        L.orc_batch_c4_inputs.argtypes = [u64, i64, P, P]
        L.orc_batch_sample.argtypes = [i32, i64] + [P] * 7 + [P] * 5 + [i32]
        L.orc_batch_sample_philox.argtypes = [i32, u64, i64, P] + [P] * 5 + [i32]
        L.orc_batch_pdf.argtypes = [i64] + [P] * 9
        L.orc_batch_philox_words.argtypes = [u64, i64, P, u32, P]
        L.orc_batch_raycast.argtypes = [P, d, d, u64, i64, P, P, P]
        L.orc_batch_raycast.restype = u64
        L.orc_batch_microbench.argtypes = [i32, u64, i64, i32, P]
        L.orc_batch_microbench_trace.argtypes = [i32, u64, i64, i32, P]
        L.orc_G2.argtypes = [P, P, P, d, d]
        L.orc_G2.restype = d
        L.orc_brdf_cos.argtypes = [P, P, d, d]
        L.orc_brdf_cos.restype = d
        L.orc_pdf_reflect.argtypes = [P, P, d, d]
        L.orc_pdf_reflect.restype = d
        L.orc_sample_reflect.argtypes = [i32, P, d, d, d, d, P]
        L.orc_batch_sample_reflect.argtypes = [i32, i64] + [P] * 7 + [P]
        L.orc_batch_sample_reflect_philox.argtypes = [i32, u64, i64, P, P, i32]
        L.orc_furnace.argtypes = [i32, P, d, d, u64, u64, i64, P]
        L.orc_batch_pdf_reflect.argtypes = [i64, P, d, d, P, P, P, P]
        L.orc_sample_vndf_native.argtypes = [i32, P, d, d, d, d, P]
        L.orc_pdf_vndf_native.argtypes = [P, P, d, d]
        L.orc_pdf_vndf_native.restype = d
        L.orc_batch_raycast_native.argtypes = [P, d, d, u64, i64, P, P, P]
        L.orc_batch_raycast_native.restype = u64
        L.orc_batch_sample_native.argtypes = [i32, i64] + [P] * 7 + [P] * 4
        L.orc_batch_pdf_native.argtypes = [i64, P, P, P, P, d, d, P]
        L.orc_batch_brdf_cos.argtypes = [i64, P, d, d, P, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray) -> ctypes.c_void_p:
    # data_as keeps a reference to `a`, so temporaries outlive the C call
    return a.ctypes.data_as(ctypes.c_void_p)


def _vec(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(3))


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ---------------------------------------------------------------- Philox ---
def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(np.asarray(ctr, dtype=np.uint32).reshape(4))
    k = np.ascontiguousarray(np.asarray(key, dtype=np.uint32).reshape(2))
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def philox_words(seed: int, indices, block: int) -> np.ndarray:
    idx = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64).reshape(-1))
    out = np.zeros((idx.size, 4), dtype=np.uint32)
    lib().orc_batch_philox_words(seed, idx.size, _p(idx), block, _p(out))
    return out


def u01(word: int) -> float:
    return lib().orc_u01(word)


def c4_inputs(seed: int, index: int) -> np.ndarray:
    out = np.zeros(7, dtype=np.float64)
    lib().orc_c4_inputs(seed, index, _p(out))
    return out


def batch_c4_inputs(seed: int, indices) -> np.ndarray:
    """Config-4 inputs (wi.xyz, ax, ay, u1, u2) at global indices, shape (7, n)."""
    idx = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64).reshape(-1))
    out = np.empty((idx.size, 7), dtype=np.float64)
    lib().orc_batch_c4_inputs(seed, idx.size, _p(idx), _p(out))
    return out.T.copy()


# --------------------------------------------------------------- scalars ---
CAP, HEITZ = 0, 1


def sample_vndf(method: int, wi, ax: float, ay: float, u1: float, u2: float):
    """Listing 1 + Listing 3 (method CAP) or Listing 2 (HEITZ); float64."""
    w = _vec(wi)
    h = np.zeros(3)
    ti = np.zeros(1)
    lib().orc_sample_vndf(method, _p(w), ax, ay, u1, u2, _p(h), _p(ti))
    return h


def sample_hemisphere(method: int, u1: float, u2: float, wi) -> np.ndarray:
    """Listing 3 (unnormalised c + wi) or Listing 2 alone; native, no flip."""
    h = np.zeros(3)
    lib().orc_sample_hemisphere(method, u1, u2, _p(_vec(wi)), _p(h))
    return h


def pdf_vndf(h, wi, ax, ay) -> float:
    return lib().orc_pdf_vndf(_p(_vec(h)), _p(_vec(wi)), ax, ay)


def pdf_vndf_g1d(h, wi, ax, ay) -> float:
    return lib().orc_pdf_vndf_g1d(_p(_vec(h)), _p(_vec(wi)), ax, ay)


def D_ggx(h, ax, ay) -> float:
    return lib().orc_D_ggx(_p(_vec(h)), ax, ay)


def G1(h, wi, ax, ay) -> float:
    return lib().orc_G1(_p(_vec(h)), _p(_vec(wi)), ax, ay)


def sigma_std(zi: float) -> float:
    return lib().orc_sigma_std(zi)


def D_std(zm: float) -> float:
    return lib().orc_D_std(zm)


def Dvis_std(wm, wi) -> float:
    return lib().orc_Dvis_std(_p(_vec(wm)), _p(_vec(wi)))


def reflect(wi, wm) -> np.ndarray:
    out = np.zeros(3)
    lib().orc_reflect(_p(_vec(wi)), _p(_vec(wm)), _p(out))
    return out


def half_vector(wi, wo) -> np.ndarray:
    out = np.zeros(3)
    lib().orc_half_vector(_p(_vec(wi)), _p(_vec(wo)), _p(out))
    return out


def reflect_jacobian(wo, wh) -> float:
    return lib().orc_reflect_jacobian(_p(_vec(wo)), _p(_vec(wh)))


def cap_density(wo, wi) -> float:
    return lib().orc_cap_density(_p(_vec(wo)), _p(_vec(wi)))


# --------------------------------------------------------------- batches ---
def batch_sample(method: int, wx, wy, wz, ax, ay, u1, u2, *, pdf: bool = True,
                 threads: int | None = None):
    """Oracle over fp32 SoA planes.  Returns (h[3,n] float64, pdf[n] or None, aux[n])."""
    planes = [np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(-1))
              for a in (wx, wy, wz, ax, ay, u1, u2)]
    n = planes[0].size
    h = np.empty((3, n), dtype=np.float64)
    p = np.empty(n, dtype=np.float64) if pdf else None
    aux = np.empty(n, dtype=np.float64)
    lib().orc_batch_sample(method, n, *[_p(a) for a in planes],
                           _p(h[0]), _p(h[1]), _p(h[2]),
                           _p(p) if pdf else None, _p(aux),
                           threads or default_threads())
    return h, p, aux


def batch_sample_philox(method: int, seed: int, indices, *, threads: int | None = None):
    idx = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64).reshape(-1))
    n = idx.size
    h = np.empty((3, n), dtype=np.float64)
    p = np.empty(n, dtype=np.float64)
    aux = np.empty(n, dtype=np.float64)
    lib().orc_batch_sample_philox(method, seed, n, _p(idx), _p(h[0]), _p(h[1]), _p(h[2]),
                                  _p(p), _p(aux), threads or default_threads())
    return h, p, aux


def batch_pdf(h, wi, ax, ay) -> np.ndarray:
    h = np.ascontiguousarray(np.asarray(h, dtype=np.float64).reshape(3, -1))
    wi = np.ascontiguousarray(np.asarray(wi, dtype=np.float64).reshape(3, -1))
    n = h.shape[1]
    ax = np.ascontiguousarray(np.broadcast_to(np.asarray(ax, dtype=np.float64), (n,)))
    ay = np.ascontiguousarray(np.broadcast_to(np.asarray(ay, dtype=np.float64), (n,)))
    out = np.empty(n, dtype=np.float64)
    lib().orc_batch_pdf(n, _p(h[0]), _p(h[1]), _p(h[2]), _p(wi[0]), _p(wi[1]), _p(wi[2]),
                        _p(ax), _p(ay), _p(out))
    return out


def batch_raycast(wi, ax, ay, seed: int, n: int):
    """Brute-force ray-cast VNDF samples (definition). Returns (h[3,n], trials)."""
    h = np.empty((3, n), dtype=np.float64)
    trials = lib().orc_batch_raycast(_p(_vec(wi)), ax, ay, seed, n, _p(h[0]), _p(h[1]), _p(h[2]))
    return h, trials


def batch_microbench(method: int, seed: int, lanes: int, iters: int) -> np.ndarray:
    """NEXT-1 microbenchmark checksums replayed in float64 (see oracle.c)."""
    out = np.empty(lanes, dtype=np.float64)
    lib().orc_batch_microbench(method, seed, lanes, iters, _p(out))
    return out


def batch_microbench_trace(method: int, seed: int, lanes: int, iters: int) -> np.ndarray:
    """NEXT-1: h of every call of lanes [0, lanes), float64, shape (lanes, iters, 3)."""
    out = np.empty((lanes, iters, 3), dtype=np.float64)
    lib().orc_batch_microbench_trace(method, seed, lanes, iters, _p(out))
    return out


# ------------------------------------------------------------------ NEXT-2 ---
def G2(wm, wi, wo, ax, ay) -> float:
    return lib().orc_G2(_p(_vec(wm)), _p(_vec(wi)), _p(_vec(wo)), ax, ay)


def brdf_cos(wi, wo, ax, ay) -> float:
    """Eq. 11 x cos(theta_o) with F = 1."""
    return lib().orc_brdf_cos(_p(_vec(wi)), _p(_vec(wo)), ax, ay)


def pdf_reflect(wa, wb, ax, ay) -> float:
    """Eq. 20."""
    return lib().orc_pdf_reflect(_p(_vec(wa)), _p(_vec(wb)), ax, ay)


def sample_reflect(method, wa, ax, ay, u1, u2) -> np.ndarray:
    out = np.zeros(5)
    lib().orc_sample_reflect(method, _p(_vec(wa)), ax, ay, u1, u2, _p(out))
    return out


def batch_sample_reflect(method, wx, wy, wz, ax, ay, u1, u2) -> np.ndarray:
    """(5, n): wb.xyz, pdf (Eq. 20), weight (f_r cos / pdf)."""
    planes = [np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(-1))
              for a in (wx, wy, wz, ax, ay, u1, u2)]
    n = planes[0].size
    out = np.empty((n, 5), dtype=np.float64)
    lib().orc_batch_sample_reflect(method, n, *[_p(a) for a in planes], _p(out))
    return out.T.copy()


def batch_sample_reflect_philox(method, seed: int, indices, *, threads: int | None = None) -> np.ndarray:
    """(5, n) reflection outputs on config-4 inputs (orc_c4_inputs) at global indices."""
    idx = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64).reshape(-1))
    out = np.empty((idx.size, 5), dtype=np.float64)
    lib().orc_batch_sample_reflect_philox(method, seed, idx.size, _p(idx), _p(out), threads or default_threads())
    return out.T.copy()


def furnace(method, wa, ax, ay, seed, n, first=0):
    """Eq. 19 white-furnace estimator: (sum, sum of squares) of the weights."""
    out = np.zeros(2)
    lib().orc_furnace(method, _p(_vec(wa)), ax, ay, seed, first, n, _p(out))
    return out


def _batch_dirs(fn, wa, ax, ay, wb):
    wb = np.ascontiguousarray(np.asarray(wb, dtype=np.float64).reshape(3, -1))
    out = np.empty(wb.shape[1])
    fn(wb.shape[1], _p(_vec(wa)), ax, ay, _p(wb[0]), _p(wb[1]), _p(wb[2]), _p(out))
    return out


def batch_pdf_reflect(wa, ax, ay, wb) -> np.ndarray:
    return _batch_dirs(lib().orc_batch_pdf_reflect, wa, ax, ay, wb)


def batch_brdf_cos(wa, ax, ay, wb) -> np.ndarray:
    return _batch_dirs(lib().orc_batch_brdf_cos, wa, ax, ay, wb)


def sphere_quadrature(nz: int = 512, nphi: int = 512, upper_only: bool = False):
    """Directions and weights of a product rule on the sphere: Gauss-Legendre in
    z = cos(theta) (uniform-area coordinate) times the midpoint rule in phi."""
    x, w = np.polynomial.legendre.leggauss(nz)
    if upper_only:
        z, wz = 0.5 * (x + 1), 0.5 * w
    else:
        z, wz = x, w
    phi = (np.arange(nphi) + 0.5) * (2 * np.pi / nphi)
    Z, P = np.meshgrid(z, phi, indexing="ij")
    r = np.sqrt(np.clip(1 - Z * Z, 0, None))
    dirs = np.stack([r * np.cos(P), r * np.sin(P), Z]).reshape(3, -1)
    weights = (wz[:, None] * np.full(nphi, 2 * np.pi / nphi)[None, :]).reshape(-1)
    return dirs, weights


# ------------------------------------------------------------------ NEXT-3 ---
def sample_vndf_native(method, wi, ax, ay, u1, u2) -> np.ndarray:
    h = np.zeros(3)
    lib().orc_sample_vndf_native(method, _p(_vec(wi)), ax, ay, u1, u2, _p(h))
    return h


def pdf_vndf_native(h, wi, ax, ay) -> float:
    return lib().orc_pdf_vndf_native(_p(_vec(h)), _p(_vec(wi)), ax, ay)


def batch_raycast_native(wi, ax, ay, seed: int, n: int):
    h = np.empty((3, n), dtype=np.float64)
    trials = lib().orc_batch_raycast_native(_p(_vec(wi)), ax, ay, seed, n, _p(h[0]), _p(h[1]), _p(h[2]))
    return h, trials


def batch_sample_native(method, wx, wy, wz, ax, ay, u1, u2, pdf=True):
    planes = [np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(-1))
              for a in (wx, wy, wz, ax, ay, u1, u2)]
    n = planes[0].size
    h = np.empty((3, n), dtype=np.float64)
    p = np.empty(n, dtype=np.float64) if pdf else None
    lib().orc_batch_sample_native(method, n, *[_p(a) for a in planes], _p(h[0]), _p(h[1]), _p(h[2]),
                                  _p(p) if pdf else None)
    return h, p


def batch_pdf_native(h, wi, ax, ay) -> np.ndarray:
    h = np.ascontiguousarray(np.asarray(h, dtype=np.float64).reshape(3, -1))
    out = np.empty(h.shape[1])
    lib().orc_batch_pdf_native(h.shape[1], _p(h[0]), _p(h[1]), _p(h[2]), _p(_vec(wi)), ax, ay, _p(out))
    return out
