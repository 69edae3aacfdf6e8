"""Build a variant of libvndf with extra preprocessor definitions, for the
side-by-side timings of tools/variants.py (fused kernels) and
tools/stream_variants.py (streamed kernels).  The build knobs are the
VNDF_* macros of paper_2306_05044_b200/csrc/ (block shapes, samples per
thread, launch bounds, VNDF_NO_FIXUP, ...).

python tools/build_variant.py NAME [-DMACRO=VALUE ...]   ->  paper_2306_05044_b200/var_NAME.so

e.g. the fused-kernel shape sweep of DESIGN.md s.6.4:
    python tools/build_variant.py b640 -DVNDF_PHILOX_BLOCK_CAP=640
    python tools/variants.py paper_2306_05044_b200/libvndf.so paper_2306_05044_b200/var_b640.so
Variant libraries are build products (git-ignored); delete them when done.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_05044_b200 import _build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "paper_2306_05044_b200", f"var_{name}.so")
cmd = [b.NVCC, *b.NVCC_FLAGS, *defs, "-I", os.path.join(ROOT, "include"), *b.SOURCES, "-o", out]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode != 0:
    sys.exit(r.stdout + r.stderr)
print(out)
