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


BUILD_INFO = os.path.join(HERE, "build_info.json")


def _write_build_info() -> None:
    """Record the git commit the sources were built from (build_info.json,
    git-ignored, travels with the in-tree .so): the GPU box has no .git, so
    bench.py reads the commit from here when `git` cannot.  Written only where
    git answers, never overwritten with an unknown commit."""
    import json
    try:
        r = subprocess.run(["git", "-C", ROOT, "rev-parse", "HEAD"], capture_output=True, text=True, timeout=5)
        sha = r.stdout.strip()
        if r.returncode != 0 or not sha:
            return
        d = subprocess.run(["git", "-C", ROOT, "status", "--porcelain", "--untracked-files=no"],
                           capture_output=True, text=True, timeout=5).stdout.strip()
    except Exception:
        return
    with open(BUILD_INFO, "w") as f:
        json.dump({"git": sha, "git_dirty": bool(d), "libvndf_source_sha256": source_hash()}, f)


def build(force: bool = False, verbose: bool = False) -> str:
    _write_build_info()
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
