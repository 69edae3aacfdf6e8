"""Seeded synthetic inputs for the five BASELINE.json configs (DESIGN.md s.5).

Shared by both sides of the parity tests and by bench.py.  Holds NONE of the
method's arithmetic: only the input recipes (directions, roughness, uniforms).
The GPU generator (csrc/synth.cu -> libvndf_synth.so) fills device planes; the
numpy generator below implements the same counter-based recipe on the host for
CPU-only tests (values agree to fp32 rounding, not bit for bit).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "synth.cu")
LIB = os.path.join(HERE, "libvndf_synth.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config (index = position + 1)."""
    cid: int
    n: int
    recipe: int       # synth recipe; 4 = in-kernel Philox (no streamed inputs)
    seed: int
    pdf: bool
    kernel: str
    label: str


CONFIGS = {
    1: Config(1, 1 << 16, 1, 0, True, "vndf_sample_cap_pdf",
              "2^16, wi uniform upper hemisphere, alpha 0.5, h + pdf"),
    2: Config(2, 1 << 24, 2, 1, True, "vndf_sample_cap_pdf",
              "2^24, wi cosine-weighted, alpha log-uniform [0.01, 1], h + pdf"),
    3: Config(3, 1 << 28, 3, 2, False, "vndf_sample_cap",
              "2^28 streamed, wi uniform upper hemisphere, alpha log-uniform [0.001, 1], h only"),
    4: Config(4, 1 << 30, 4, 3, True, "vndf_sample_cap_philox",
              "2^30 fused Philox4x32-10, wi uniform upper, alpha log-uniform [0.01, 1], h + pdf"),
    5: Config(5, 1 << 26, 5, 4, True, "vndf_sample_cap_pdf",
              "2^26 path-tracer edge mix: 40% grazing, 20% back side, 40% upper; alpha in "
              "{1e-3, .05, .3, 1}; u = 0 and rim injections; h + pdf"),
}

PLANES = ("wi_x", "wi_y", "wi_z", "alpha_x", "alpha_y", "u1", "u2")


def build(force: bool = False) -> str:
    """nvcc sm_100a build of libvndf_synth.so; concurrent callers serialise on a lock file."""
    import fcntl
    if not (force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC)):
        return LIB
    with open(LIB + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            return _build_locked(force)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)


def _build_locked(force: bool) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
               "-shared", "-Xcompiler", "-fPIC", "-cudart", "static", SRC, "-o", LIB + ".tmp"]
        subprocess.run(cmd, check=True, capture_output=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        P = ctypes.c_void_p
        L.synth_fill.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64] + [P] * 9
        L.synth_fill.restype = ctypes.c_int
        _lib = L
    return _lib


def fill(recipe: int, seed: int, n: int, *, first: int = 0, device="cuda", out=None,
         fixed=None, stream=None):
    """Generate n samples' input planes on the GPU.  Returns a dict of 7 float32
    tensors (or fills `out`, a dict of preallocated tensors)."""
    import torch
    if out is None:
        out = {k: torch.empty(n, dtype=torch.float32, device=device) for k in PLANES}
    dev = out["wi_x"].device
    fx = None
    if fixed is not None:
        fx = np.ascontiguousarray(np.asarray(fixed, dtype=np.float32).reshape(5))
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    rc = _load().synth_fill(recipe, seed, first, n, *[ctypes.c_void_p(out[k].data_ptr()) for k in PLANES],
                            fx.ctypes.data_as(ctypes.c_void_p) if fx is not None else None,
                            ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"synth_fill failed ({rc})")
    return out


# ------------------------------------------------------------- host twin ----
_M0, _M1, _W0, _W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85


def _philox_np(c0, c1, c2, c3, k0, k1):
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) for x in (c0, c1, c2, c3))
    k0, k1 = np.uint64(k0), np.uint64(k1)
    mask = np.uint64(0xFFFFFFFF)
    for _ in range(10):
        p0 = np.uint64(_M0) * c0
        p1 = np.uint64(_M1) * c2
        c0, c1, c2, c3 = ((p1 >> np.uint64(32)) ^ c1 ^ k0, p1 & mask,
                          (p0 >> np.uint64(32)) ^ c3 ^ k1, p0 & mask)
        k0 = (k0 + np.uint64(_W0)) & mask
        k1 = (k1 + np.uint64(_W1)) & mask
    return c0, c1, c2, c3


def _u(w):
    return (np.asarray(w, dtype=np.uint64) >> np.uint64(8)).astype(np.float64) * 2.0**-24


def fill_numpy(recipe: int, seed: int, n: int, *, first: int = 0, fixed=None):
    """Host version of `fill` (float64 arithmetic rounded once to float32)."""
    i = np.arange(first, first + n, dtype=np.uint64)
    lo, hi = i & np.uint64(0xFFFFFFFF), i >> np.uint64(32)
    k0, k1 = seed & 0xFFFFFFFF, seed >> 32
    z0 = np.zeros_like(i)
    X = _philox_np(lo, hi, z0, z0, k0, k1)
    Y = _philox_np(lo, hi, z0 + np.uint64(1), z0, k0, k1)
    u1, u2 = _u(Y[0]), _u(Y[1])
    if recipe == 0:
        f = np.asarray(fixed, dtype=np.float64)
        wx, wy, wz = (np.full(n, f[k]) for k in range(3))
        ax, ay = np.full(n, f[3]), np.full(n, f[4])
    else:
        ua = _u(X[0])
        phi = 2 * np.pi * _u(X[1])
        if recipe == 2:
            r, z = np.sqrt(ua), np.sqrt(1 - ua)
        elif recipe == 5:
            v = _u(Y[2])
            z = np.where(v < 0.4, 1e-4 + ua * (0.05 - 1e-4), np.where(v < 0.6, -(1 - ua), 1 - ua))
            r = np.sqrt(np.maximum((1 - z) * (1 + z), 0))
        else:
            z, r = 1 - ua, np.sqrt(ua * (2 - ua))
        wx, wy, wz = r * np.cos(phi), r * np.sin(phi), z
        if recipe == 1:
            ax = ay = np.full(n, 0.5)
        elif recipe == 2:
            ax, ay = 0.01 * 100.0 ** _u(X[2]), 0.01 * 100.0 ** _u(X[3])
        elif recipe == 3:
            ax, ay = 0.001 * 1000.0 ** _u(X[2]), 0.001 * 1000.0 ** _u(X[3])
        elif recipe == 5:
            T = np.array([1e-3, 0.05, 0.3, 1.0])
            ax, ay = T[(X[2] >> np.uint64(30)).astype(np.int64)], T[(X[3] >> np.uint64(30)).astype(np.int64)]
            b = Y[3]
            u1 = np.where((b & np.uint64(0x3F)) == 0, 0.0, u1)
            u2 = np.where(((b >> np.uint64(6)) & np.uint64(0x3F)) == 0, 0.0, u2)
            u2 = np.where(((b >> np.uint64(12)) & np.uint64(0x3F)) == 0, 1 - 2.0**-24, u2)
        else:
            raise ValueError(f"unknown recipe {recipe}")
    vals = (wx, wy, wz, ax, ay, u1, u2)
    return {k: np.ascontiguousarray(np.asarray(v, dtype=np.float32)) for k, v in zip(PLANES, vals)}
