"""Build libvndf.so in-tree with nvcc for sm_100a (no JIT cache, no torch ext).

The shared library carries its own static CUDA runtime; it takes plain device
pointers and a cudaStream_t, so it interoperates with torch's allocator and
streams through the driver's primary context.
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvndf.so")
SOURCES = [os.path.join(CSRC, "vndf.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")] + [
    os.path.join(ROOT, "include", "vndf.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xptxas", "-v",
    "-shared", "-Xcompiler", "-fPIC,-O2",
    "-cudart", "static",
]


STAMP = LIB + ".srchash"


def source_hash() -> str:
    """SHA-256 of every source the library is built from plus the nvcc command
    line: the build key (mtimes are unreliable across checkouts and copies)."""
    import hashlib
    h = hashlib.sha256()
    h.update(" ".join([NVCC, *NVCC_FLAGS]).encode())
    for p in sorted(DEPS):
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def stale() -> bool:
    if not (os.path.exists(LIB) and os.path.exists(STAMP)):
        return True
    with open(STAMP) as f:
        return f.read().strip() != source_hash()


class _FileLock:
    """Exclusive advisory lock: concurrent builders (e.g. every torchrun rank
    calling build()) compile once; the others wait and then see a fresh file."""

    def __init__(self, path: str):
        self.path = path

    def __enter__(self):
        import fcntl
        self.f = open(self.path, "w")
        fcntl.flock(self.f, fcntl.LOCK_EX)
        return self

    def __exit__(self, *exc):
        import fcntl
        fcntl.flock(self.f, fcntl.LOCK_UN)
        self.f.close()


def build(force: bool = False, verbose: bool = False) -> str:
    if not (force or stale()):
        return LIB
    with _FileLock(LIB + ".lock"):
        return _build_locked(force, verbose)


def _build_locked(force: bool, verbose: bool) -> str:
    if force or stale():
        cmd = [NVCC, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), *SOURCES, "-o", LIB + ".tmp"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
        os.replace(LIB + ".tmp", LIB)
        with open(STAMP, "w") as f:
            f.write(source_hash() + "\n")
        log = os.path.join(HERE, "csrc", "ptxas.log")
        with open(log, "w") as f:
            f.write(res.stderr)
        if verbose:
            print(res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
