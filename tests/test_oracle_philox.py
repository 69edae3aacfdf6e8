"""Pins for the oracle's Philox4x32-10 and uniform conversion (not in the paper;
BASELINE.json config 4 names the generator; reading R11)."""
import os
import shutil
import subprocess

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def _kat_rows():
    rows = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        v = [int(t, 16) for t in line.split()]
        rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


def test_known_answer_vectors(orc):
    rows = _kat_rows()
    assert len(rows) == 3
    for ctr, key, out in rows:
        assert list(orc.philox4x32_10(ctr, key)) == out


CURAND_PROG = r"""
#include <cstdio>
#include <cstdint>
#include <vector_types.h>
#include <vector_functions.h>
#define QUALIFIERS static inline
#include <curand_philox4x32_x.h>
int main() {
  unsigned c0, c1, c2, c3, k0, k1;
  while (std::scanf("%x %x %x %x %x %x", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    uint4 c = make_uint4(c0, c1, c2, c3); uint2 k = make_uint2(k0, k1);
    uint4 r = curand_Philox4x32_10(c, k);
    std::printf("%08x %08x %08x %08x\n", r.x, r.y, r.z, r.w);
  }
}
"""


def test_matches_cuda_toolkit_curand_host_routine(orc, tmp_path):
    """A second, independent implementation: the CUDA toolkit's curand_Philox4x32_10."""
    inc = "/usr/local/cuda/include"
    if not (shutil.which("g++") and os.path.exists(os.path.join(inc, "curand_philox4x32_x.h"))):
        pytest.skip("CUDA toolkit headers or g++ not available")
    src = tmp_path / "cr.cpp"
    src.write_text(CURAND_PROG)
    exe = tmp_path / "cr"
    subprocess.run(["g++", "-O1", f"-I{inc}", str(src), "-o", str(exe)], check=True)
    rng = np.random.default_rng(123)
    inputs = rng.integers(0, 2**32, size=(2000, 6), dtype=np.uint64)
    inputs[:3] = np.array([r[0] + r[1] for r in _kat_rows()], dtype=np.uint64)
    # counters around the 32-bit carry and block ids used by the recipe
    inputs[3:8, 0] = 0xFFFFFFFF
    inputs[3:8, 2] = [0, 1, 2, 3, 4]
    text = "\n".join(" ".join(f"{int(x):08x}" for x in row) for row in inputs) + "\n"
    res = subprocess.run([str(exe)], input=text, capture_output=True, text=True, check=True)
    lines = res.stdout.strip().split("\n")
    assert len(lines) == len(inputs)
    for row, line in zip(inputs, lines):
        want = [int(t, 16) for t in line.split()]
        got = list(orc.philox4x32_10(row[:4], row[4:6]))
        assert got == want


def test_block_layout(orc):
    """counter = (i_lo, i_hi, block, 0), key = (seed_lo, seed_hi)  (DESIGN.md s.5)."""
    seed = 0x0123456789ABCDEF
    for idx in (0, 1, 2**32 - 1, 2**32, 2**32 + 5, 2**40 + 3):
        for b in (0, 1, 2):
            w = orc.philox_words(seed, [idx], b)[0]
            ref = orc.philox4x32_10([idx & 0xFFFFFFFF, idx >> 32, b, 0],
                                    [seed & 0xFFFFFFFF, seed >> 32])
            assert list(w) == list(ref)


def test_uniform_conversion_edges(orc):
    """u(w) = (w >> 8) 2^-24: exact, in [0, 1 - 2^-24]."""
    assert orc.u01(0) == 0.0
    assert orc.u01(0xFF) == 0.0
    assert orc.u01(0x100) == 2.0**-24
    assert orc.u01(0xFFFFFFFF) == 1.0 - 2.0**-24
    assert orc.u01(0x80000000) == 0.5
    # representable exactly in binary32
    for w in (0x12345678, 0xDEADBEEF, 0xFFFFFF00):
        v = orc.u01(w)
        assert float(np.float32(v)) == v


def test_c4_recipe_ranges(orc):
    """Config-4 inputs: unit upper-hemisphere wi, alpha in [0.01, 1], u in [0, 1)."""
    for i in list(range(200)) + [2**32 - 1, 2**32, 2**33 + 7]:
        v = orc.c4_inputs(3, i)
        assert abs(np.linalg.norm(v[:3]) - 1.0) < 1e-14
        assert v[2] > 0.0
        assert 0.01 <= v[3] <= 1.0 and 0.01 <= v[4] <= 1.0
        assert 0.0 <= v[5] < 1.0 and 0.0 <= v[6] < 1.0
