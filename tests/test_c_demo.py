"""The C ABI is usable from plain C: examples/c_demo.c compiles against
include/vndf.h and libvndf.so with gcc (CPU), and runs correctly on a B200 (GPU)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _compile(tmp_path):
    import __graft_entry__
    __graft_entry__.build()
    if not shutil.which("gcc") or not os.path.exists("/usr/local/cuda/include/cuda_runtime.h"):
        pytest.skip("gcc or CUDA headers missing")
    libdir = os.path.join(ROOT, "paper_2306_05044_b200")
    exe = tmp_path / "c_demo"
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Werror", os.path.join(ROOT, "examples", "c_demo.c"),
           "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(libdir, "libvndf.so"), "-L/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{libdir}", "-Wl,-rpath,/usr/local/cuda/lib64", "-o", str(exe), "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_demo_compiles(tmp_path):
    _compile(tmp_path)


@pytest.mark.gpu
def test_c_demo_runs(tmp_path):
    exe = _compile(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "vndf_sample_cap_pdf" in r.stdout
