"""Mutation check of the GPU parity tests: plausible mistakes written into a
copy of the CUDA sources, each compiled into its own libvndf; on the GPU box
every mutant library runs the parity tests (against the float64 oracle) in a
copy of the repository.  A mutant is CAUGHT when a test fails; the unmutated
library must pass.

python tools/kernel_mutants.py build          # here: paper_2306_05044_b200/mut_<k>.so + mut_manifest.json
python tools/kernel_mutants.py run            # GPU box: report on stdout
"""
import json
import os
import shutil
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2306_05044_b200")
MANIFEST = os.path.join(PKG, "mut_manifest.json")

# (name, file under csrc/, old text (unique), new text)
MUTANTS = [
    ("cap: hs.z = a (q = 1 - u2 dropped)", "vndf_device.cuh", "    k.hz = q * k.a;", "    k.hz = k.a;"),
    ("cap: sin^2 = u2 (q a^2 - rs^2) (sign of rs^2)", "vndf_device.cuh",
     "const float sin2 = u2 * fmaf(k.hz, k.a, rs2);", "const float sin2 = u2 * fmaf(k.hz, k.a, -rs2);"),
    ("cap: hs.x = sin(theta) sin(phi) + ws.x (cos and sin swapped)", "vndf_device.cuh",
     "    k.hx = fmaf(st, cp, wsx);", "    k.hx = fmaf(st, sp, wsx);"),
    ("unstretch: m.x = alpha_y hs.x", "vndf_device.cuh", "    k.mx = ax * k.hx;", "    k.mx = ay * k.hx;"),
    ("pdf: (1 + ws.z) dropped from the denominator", "vndf_device.cuh",
     "const float den = (kPiF * ax * ay) * k.a * k.hs2;", "const float den = (kPiF * ax * ay) * k.hs2;"),
    ("conditioning test 100x looser (A <= 3000)", "vndf_device.cuh",
     "constexpr float kFlagA = 30.0f;", "constexpr float kFlagA = 3000.0f;"),
    ("flip: wi.z = +0 flipped too (reading R4: -0 and +0 are upper)", "vndf_device.cuh",
     "k.s = (FRAME == kFrameFlip && wz < 0.0f) ? -1.0f : 1.0f;", "k.s = (FRAME == kFrameFlip && wz <= 0.0f) ? -1.0f : 1.0f;"),
    ("float64 recomputation: hs.z = a", "vndf_device.cuh",
     "    const double hz = q * a;\n    const double st = sqrt(u2 * (hz * a + rs2));\n    double sp, cp;\n    sincospi(2.0 * u1, &sp, &cp);\n    const double hx = fma(st, cp, wsx), hy = fma(st, sp, wsy);\n    const double mx = ax * hx, my = ay * hy;\n    const double m2 = mx * mx + my * my + hz * hz;\n    const double hs2",
     "    const double hz = a;\n    const double st = sqrt(u2 * (hz * a + rs2));\n    double sp, cp;\n    sincospi(2.0 * u1, &sp, &cp);\n    const double hx = fma(st, cp, wsx), hy = fma(st, sp, wsy);\n    const double mx = ax * hx, my = ay * hy;\n    const double m2 = mx * mx + my * my + hz * hz;\n    const double hs2"),
    ("float64 recomputation: |hs|^2 scaled by 2^-k once", "vndf_device.cuh",
     "hs2s = (float)(hs2 * sc * sc);", "hs2s = (float)(hs2 * sc);"),
    ("Heitz: s = (1 - ws.z)/2", "vndf_device.cuh",
     "const float sh = (1.0f + wsz) * 0.5f;", "const float sh = (1.0f - wsz) * 0.5f;"),
    ("reflection: wo = (w.h) h - w", "vndf_device.cuh",
     "o.x = fmaf(d2, hx, -wx * inv_w);", "o.x = fmaf(dot, hx, -wx * inv_w);"),
    ("Philox: key schedule constant off by one", "vndf_device.cuh",
     "        a += 0x9E3779B9u;", "        a += 0x9E3779B8u;"),
    ("config-4 inputs: alpha_x from word X3", "vndf_device.cuh",
     "in.ax = ex2_approx(fmaf(fw_t<FW_HI>(X.z),", "in.ax = ex2_approx(fmaf(fw_t<FW_HI>(X.w),"),
    ("config-4 inputs: cos quadrant sign off", "vndf_device.cuh",
     "const uint32_t q1 = w + 0x60000000u;", "const uint32_t q1 = w + 0x20000000u;"),
    ("config-4 inputs: azimuth of the method mirrored", "vndf_device.cuh",
     "in.p1 = phi_reduced_w(f1);", "in.p1 = -phi_reduced_w(f1);"),
    ("streamed tail: h.x written from h.y", "kernels_stream.cuh",
     "            a.hx[i] = o.x;", "            a.hx[i] = o.y;"),
    ("standalone pdf: |h|^2 for |h|^3", "vndf_device.cuh",
     "const float h3 = h2 * (h2 * rsqrt_approx(h2));", "const float h3 = h2;"),
    ("native frame: 1 + ws.z below the horizon taken as 1 - ws.z", "vndf_device.cuh",
     "rs2 * rcp_approx(1.0f - wsz) : 1.0f + wsz;", "rs2 * rcp_approx(1.0f + wsz) : 1.0f + wsz;"),
    ("reflection weight: z_i dropped from G2/G1", "vndf_device.cuh",
     "    const float Lo = sqrt_approx(fmaf(ax * o.x, ax * o.x, fmaf(ay * o.y, ay * o.y, o.z * o.z)));\n    const float wgt = zo * (zi + L) * rcp_approx(fmaf(L, zo, Lo * zi));\n    o.weight = zo > 0.0f ? wgt : 0.0f;\n    return cap_flag",
     "    const float Lo = sqrt_approx(fmaf(ax * o.x, ax * o.x, fmaf(ay * o.y, ay * o.y, o.z * o.z)));\n    const float wgt = zo * L * rcp_approx(fmaf(L, zo, Lo * zi));\n    o.weight = zo > 0.0f ? wgt : 0.0f;\n    return cap_flag"),
    ("config-5 inputs: u2 = 0 injection lost", "vndf_device.cuh",
     "if (((Y.w >> 6) & 0x3Fu) == 0u) u2 = 0.0f;", "if (((Y.w >> 6) & 0x3Fu) == 0u) u2 = 0.5f;"),
    ("host path: every chunk from the call's first index", "vndf.cu",
     "result = launch_philox<kCap>(seed, first_index + (uint64_t)off, m,", "result = launch_philox<kCap>(seed, first_index, m,"),
]

TESTS = ["tests/test_parity_gpu.py", "tests/test_edge_gpu.py", "tests/test_edge_fused_gpu.py",
         "tests/test_reflect_gpu.py", "tests/test_pdf_gpu.py", "tests/test_microbench_gpu.py",
         "tests/test_native_gpu.py", "tests/test_host_paths_gpu.py"]


def build():
    sys.path.insert(0, ROOT)
    from paper_2306_05044_b200 import _build as b
    manifest = []
    for k, (name, fname, old, new) in enumerate(MUTANTS):
        tmp = tempfile.mkdtemp(prefix="kmut_")
        try:
            # same relative layout as the repository (vndf.cu includes ../../include/vndf.h)
            shutil.copytree(os.path.join(PKG, "csrc"), os.path.join(tmp, "pkg", "csrc"))
            shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
            p = os.path.join(tmp, "pkg", "csrc", fname)
            src = open(p).read()
            assert src.count(old) == 1, (name, src.count(old))
            open(p, "w").write(src.replace(old, new))
            out = os.path.join(PKG, f"mut_{k}.so")
            cmd = [b.NVCC, *b.NVCC_FLAGS, "-I", os.path.join(tmp, "include"), os.path.join(tmp, "pkg", "csrc", "vndf.cu"),
                   "-o", out]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.exit(f"{name}: build failed\n{r.stderr[-2000:]}")
            manifest.append({"k": k, "name": name, "file": fname, "lib": os.path.basename(out)})
            print(f"built mut_{k}.so  {name}", flush=True)
        finally:
            shutil.rmtree(tmp, ignore_errors=True)
    json.dump(manifest, open(MANIFEST, "w"), indent=1)


def run_in_copy(lib):
    tmp = tempfile.mkdtemp(prefix="kmut_run_")
    dst = os.path.join(tmp, "repo")
    try:
        shutil.copytree(ROOT, dst, symlinks=True, ignore=shutil.ignore_patterns(
            "gpurun_out", "profiles", ".git", "mut_*.so", "var_*.so", "*.ncu-rep", "__pycache__"))
        if lib:
            shutil.copy(os.path.join(PKG, lib), os.path.join(dst, "paper_2306_05044_b200", "libvndf.so"))
        t0 = time.time()
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", *TESTS, "-k",
                            "not beyond_2e31"], cwd=dst, capture_output=True, text=True, timeout=3600)
        failed = ""
        for line in r.stdout.splitlines():
            if line.startswith("FAILED") or line.startswith("ERROR"):
                failed = line.split(" - ")[0].replace("FAILED ", "").replace("ERROR ", "")
                break
        return r.returncode, failed, time.time() - t0, r.stdout[-300:]
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def run():
    manifest = json.load(open(MANIFEST))
    rc, failed, dt, tail = run_in_copy(None)
    print(f"# control (unmutated libvndf.so): rc={rc} ({dt:.0f} s) {failed}", flush=True)
    if rc != 0:
        print(tail)
        sys.exit(1)
    caught = 0
    for m in manifest:
        rc, failed, dt, _ = run_in_copy(m["lib"])
        ok = rc != 0
        caught += ok
        print(f"{'CAUGHT ' if ok else 'ESCAPED'}  {m['name']}  [{m['file']}]  -> {failed or 'all tests pass'}  ({dt:.0f} s)",
              flush=True)
    print(f"# {caught} of {len(manifest)} kernel mutants caught by the GPU parity tests")


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
