"""C-ABI checks that need no GPU: the library builds and loads, exports every
symbol include/vndf.h declares, and rejects bad arguments before touching CUDA."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vndf.h")


@pytest.fixture(scope="module")
def vndf():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2306_05044_b200 as v
    return v


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vndf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_survey_entry_points():
    syms = declared_symbols()
    for s in ("vndf_sample_cap", "vndf_sample_cap_pdf", "vndf_sample_heitz2018",
              "vndf_sample_cap_philox", "vndf_sample_heitz2018_philox", "vndf_philox4x32_10",
              "vndf_status_string", "vndf_last_cuda_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(vndf):
    out = subprocess.run(["nm", "-D", "--defined-only", vndf.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (vndf_[a-z0-9_]+)\b", out))
    for s in declared_symbols():
        assert s in exported, s
        getattr(vndf.lib(), s)
    assert set(vndf.SYMBOLS) == set(declared_symbols())


def test_header_compiles_as_c():
    src = f'#include "{HEADER}"\nint main(void) {{ return (int)VNDF_OK; }}\n'
    r = subprocess.run(["gcc", "-x", "c", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-"],
                       input=src, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_built_for_sm100a(vndf):
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", vndf.LIB_PATH],
                       capture_output=True, text=True)
    assert r.returncode == 0
    assert "sm_100a" in r.stdout


def test_status_strings_and_version(vndf):
    assert vndf.status_string(0) == "VNDF_OK"
    assert vndf.status_string(1) == "VNDF_ERR_INVALID_ARGUMENT"
    assert vndf.status_string(2) == "VNDF_ERR_CUDA"
    assert vndf.status_string(3) == "VNDF_ERR_NOT_IMPLEMENTED"
    assert vndf.version() == 100
    assert vndf.last_cuda_error() == 0


def test_argument_validation_without_gpu(vndf):
    """Bad arguments are rejected on the host, before any CUDA call."""
    L = vndf.lib()
    P = [ctypes.c_void_p(0x10000 * (k + 1)) for k in range(11)]  # fake, never dereferenced
    INV = vndf.VNDF_ERR_INVALID_ARGUMENT
    assert L.vndf_sample_cap_pdf(*P, -1, None) == INV
    assert L.vndf_sample_cap_pdf(*P, 0, None) == vndf.VNDF_OK  # n == 0: nothing enqueued
    assert L.vndf_sample_cap_pdf(*P[:3], None, *P[4:], 16, None) == INV
    assert L.vndf_sample_cap_pdf(*P[:10], None, 16, None) == INV  # pdf required
    assert L.vndf_sample_cap_pdf(*P[:7], P[0], *P[8:], 16, None) == INV  # output aliases input
    assert L.vndf_sample_cap_pdf(*P[:7], P[7], P[7], *P[9:], 16, None) == INV  # outputs alias
    # overlap (not equality) is also rejected: h_y starts inside h_x
    Q = P[:7] + [ctypes.c_void_p(0x80000), ctypes.c_void_p(0x80000 + 32)] + P[9:]
    assert L.vndf_sample_cap_pdf(*Q, 16, None) == INV
    odd = ctypes.c_void_p(0x10002)
    assert L.vndf_sample_cap_pdf(odd, *P[1:], 16, None) == INV
    assert L.vndf_sample_cap(*P[:10], -3, None) == INV
    assert L.vndf_sample_heitz2018(*P[:10], None, -3, None) == INV
    assert L.vndf_sample_cap_philox(1, 0, -1, *P[7:11], None) == INV
    assert L.vndf_sample_cap_philox(1, 0, 0, *P[7:11], None) == vndf.VNDF_OK
    assert L.vndf_sample_cap_philox(1, 0, 8, None, *P[8:11], None) == INV
    assert L.vndf_sample_heitz2018_philox(1, 0, 8, P[7], P[7], P[9], P[10], None) == INV
    assert L.vndf_philox4x32_10(1, 0, -1, 0, P[0], None) == INV
    assert L.vndf_philox4x32_10(1, 0, 4, 0, None, None) == INV
    assert L.vndf_count_fixups(*P[:7], -1, P[8], None) == INV
    assert L.vndf_count_fixups_philox(1, 0, 4, None, None) == INV
    assert L.vndf_sample_cap_pdf_host(*P, -1, None) == INV
    assert L.vndf_sample_cap_pdf_host(*P, 0, None) == vndf.VNDF_OK
    assert L.vndf_sample_cap_philox_host(1, 0, -1, *P[7:11], None) == INV
    assert L.vndf_sample_cap_philox_host(1, 0, 0, *P[7:11], None) == vndf.VNDF_OK
    assert L.vndf_sample_cap_philox_host(1, 0, 8, None, *P[8:11], None) == INV
    assert L.vndf_sample_cap_philox_host(1, 0, 8, P[7], P[7], P[9], P[10], None) == INV
    assert L.vndf_microbench_trace(0, 1, -1, 64, P[0], P[1], None) == INV
    assert L.vndf_microbench_trace(0, 1, 16, 64, P[0], None, None) == INV
    assert L.vndf_microbench_trace(3, 1, 16, 64, P[0], P[1], None) == INV
    assert L.vndf_microbench_trace(0, 1, 0, 64, P[0], P[1], None) == vndf.VNDF_OK
    # NEXT rows
    assert L.vndf_sample_cap_reflect(*P, P[0], -1, None) == INV
    assert L.vndf_sample_cap_reflect(*P[:11], None, 16, None) == INV          # weight required
    assert L.vndf_sample_cap_reflect(*P[:7], P[0], *P[8:11], P[0], 16, None) == INV  # aliasing
    for fn in (L.vndf_sample_cap_reflect_philox, L.vndf_sample_heitz2018_reflect_philox):
        assert fn(1, 0, -1, *P[:5], None) == INV
        assert fn(1, 0, 0, *P[:5], None) == vndf.VNDF_OK
        assert fn(1, 0, 16, *P[:4], None, None) == INV                     # weight required
        assert fn(1, 0, 16, P[0], P[0], *P[2:5], None) == INV                # outputs alias
        assert fn(1, 0, 16, odd, *P[1:5], None) == INV                       # misaligned
    assert L.vndf_pdf(*P[:8], None, 16, None) == INV
    assert L.vndf_pdf(*P[:8], P[0], 16, None) == INV                         # output aliases input
    assert L.vndf_sample_cap_pdf_native(*P, -1, None) == INV


def test_launch_config_validation(vndf):
    L = vndf.lib()
    assert L.vndf_set_launch_config(3, 0, 0) == vndf.VNDF_ERR_INVALID_ARGUMENT
    assert L.vndf_set_launch_config(0, 100, 0) == vndf.VNDF_ERR_INVALID_ARGUMENT
    assert L.vndf_set_launch_config(0, 0, -2) == vndf.VNDF_ERR_INVALID_ARGUMENT
    assert L.vndf_set_launch_config(0, 0, -1) == vndf.VNDF_OK
    assert L.vndf_set_launch_config(4, 128, 2) == vndf.VNDF_OK
    assert L.vndf_set_launch_config(0, 0, 0) == vndf.VNDF_OK


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    """No CPU fallback: a missing libvndf.so is an ImportError, not a silent path."""
    import paper_2306_05044_b200 as v
    monkeypatch.setattr(v, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(v, "_lib", None)
    with pytest.raises(ImportError):
        v.lib()


def test_product_path_does_not_reference_oracle():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2306_05044_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "oracle.c" not in text and "liboracle" not in text, f
