"""Mutation check of the oracle's pins: each plausible mistake below is written
into a copy of oracle/oracle.c, the copy is compiled, and the CPU pin suite
(tests/test_oracle_*.py, `-m "not gpu"`, stop at the first failure) runs
against it.  A mutant is CAUGHT when some pin fails; an unmutated copy must
pass.  No GPU, nothing under paper_2306_05044_b200/ is touched.

python tools/oracle_mutants.py [substring] > profiles/r2/oracle_mutants_r2.txt
(substring: only the mutants whose name contains it)
"""
import os
import shutil
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, paper passage, old text, new text): each old text occurs exactly once
MUTANTS = [
    ("cap: z = fma(1-u2, 1+ws.z, +ws.z) (sign of the cap's lower end)", "Listing 3, P:529",
     "double z = fma(1.0 - u2, 1.0 + wi.z, -wi.z);", "double z = fma(1.0 - u2, 1.0 + wi.z, wi.z);"),
    ("cap: phi = pi u1 (factor 2 dropped)", "Listing 3, P:528",
     "    double phi = 2.0 * ORC_PI * u1;\n    double z", "    double phi = ORC_PI * u1;\n    double z"),
    ("cap: c.x = sin(theta) sin(phi) (cos and sin swapped)", "Listing 3, P:531",
     "double x = sin_theta * cos(phi);", "double x = sin_theta * sin(phi);"),
    ("cap: h = c (ws not added)", "Listing 3, P:535",
     "v3 h = add(c, wi);", "v3 h = c;"),
    ("cap: sinTheta = sqrt(1 - z) (square dropped)", "Listing 3, P:530",
     "double sin_theta = sqrt(clampd(1.0 - z * z, 0.0, 1.0));", "double sin_theta = sqrt(clampd(1.0 - z, 0.0, 1.0));"),
    ("Listing 1: stretch by M instead of M^-1 (wi.xy / alpha)", "Listing 1, P:419",
     "v3 wi_std = normalize(mk(wi.x * ax, wi.y * ay, wi.z));\n    /* sample",
     "v3 wi_std = normalize(mk(wi.x / ax, wi.y / ay, wi.z));\n    /* sample"),
    ("Listing 1: unstretch by M^-1 instead of M^-T (h.xy / alpha)", "Listing 1, P:423",
     "v3 wm = normalize(mk(wm_std.x * ax, wm_std.y * ay, wm_std.z));\n    h_out[0] = s * wm.x;",
     "v3 wm = normalize(mk(wm_std.x / ax, wm_std.y / ay, wm_std.z));\n    h_out[0] = s * wm.x;"),
    ("Listing 1: alpha_x and alpha_y swapped in the stretch", "Listing 1, P:419",
     "v3 wi_std = normalize(mk(wi.x * ax, wi.y * ay, wi.z));\n    /* sample",
     "v3 wi_std = normalize(mk(wi.x * ay, wi.y * ax, wi.z));\n    /* sample"),
    ("flip: h not flipped back (reading R4)", "reading R4",
     "h_out[0] = s * wm.x; h_out[1] = s * wm.y; h_out[2] = s * wm.z;",
     "h_out[0] = wm.x; h_out[1] = wm.y; h_out[2] = wm.z;"),
    ("pdf: sigma_std = 1 + z_i (the 1/2 dropped)", "Eq. 4, P:497-500",
     "double orc_sigma_std(double zi) { return (1.0 + zi) / 2.0; }",
     "double orc_sigma_std(double zi) { return (1.0 + zi); }"),
    ("pdf: Jacobian |M^T wm|^-2 instead of ^-3", "Eq. 1, P:457-473",
     "return orc_Dvis_std(A, B) * fabs(detMT) / (nMT * nMT * nMT);",
     "return orc_Dvis_std(A, B) * fabs(detMT) / (nMT * nMT);"),
    ("pdf: |det M^T| = 1/alpha_x (alpha_y dropped)", "Eq. 1, P:457-473",
     "double detMT = 1.0 / (ax * ay);", "double detMT = 1.0 / ax;"),
    ("pdf: D_vis,std without max(wm.wi, 0)", "Eq. 2, P:478-484",
     "return fmax(dot(m, i), 0.0) * orc_D_std(m.z) / orc_sigma_std(i.z);",
     "return fabs(dot(m, i)) * orc_D_std(m.z) / orc_sigma_std(i.z);"),
    ("D_ggx: |M^T wm|^-3 instead of ^-4", "Eq. 12, P:961-971",
     "return orc_D_std(MTwm.z / n) * (1.0 / (ax * ay)) / (n * n * n * n);",
     "return orc_D_std(MTwm.z / n) * (1.0 / (ax * ay)) / (n * n * n);"),
    ("G1: z_i / sigma without chi+", "Eq. 16-17, P:998-1010",
     "double chi = dot(i, m) > 0.0 ? 1.0 : 0.0;", "double chi = 1.0;"),
    ("Heitz: s = (1 - wi.z)/2", "Listing 2, P:444",
     "double s = (1.0 + wi.z) / 2.0;                                /* P:444 */",
     "double s = (1.0 - wi.z) / 2.0;                                /* P:444 */"),
    ("Heitz: r = u2 (square root dropped)", "Listing 2, P:441",
     "double r = sqrt(u2);                                          /* P:441 */",
     "double r = u2;                                                /* P:441 */"),
    ("Heitz: w2 = w1 x wi (cross product order)", "Listing 2, P:438",
     "v3 w2 = cross(wi, w1);                                        /* P:438 */",
     "v3 w2 = cross(w1, wi);                                        /* P:438 */"),
    ("G2 separable Gi Go (the round-1 verdict's mutant)", "Eq. 13-14, P:977-985",
     "return den > 0.0 ? gi * go / den : 0.0;", "return gi * go;"),
    ("reflect: wo = (wm.wi) wm - wi (factor 2 dropped)", "Eq. 5, P:712-715",
     "for (int k = 0; k < 3; ++k) wo[k] = 2.0 * d * wm[k] - wi[k];",
     "for (int k = 0; k < 3; ++k) wo[k] = d * wm[k] - wi[k];"),
    ("Eq. 20: PDF / (2 cos theta_a)", "Eq. 20, P:1058-1066",
     "return orc_G1(wm, wa, ax, ay) * orc_D_ggx(wm, ax, ay) / (4.0 * wa[2]);",
     "return orc_G1(wm, wa, ax, ay) * orc_D_ggx(wm, ax, ay) / (2.0 * wa[2]);"),
    ("BRDF: f_r cos / (2 cos theta_i)", "Eq. 11, P:938-949",
     "return orc_G2(wh, wi, wo, ax, ay) * orc_D_ggx(wh, ax, ay) / (4.0 * wi[2]);",
     "return orc_G2(wh, wi, wo, ax, ay) * orc_D_ggx(wh, ax, ay) / (2.0 * wi[2]);"),
    ("config-4 inputs: cosine-weighted wi (the round-1 verdict's mutant)", "BJ config 4; SURVEY 8(d)",
     "    double z = 1.0 - ua;\n    double r = sqrt(ua * (2.0 - ua));",
     "    double z = sqrt(1.0 - ua);\n    double r = sqrt(ua);"),
    ("config-4 inputs: alpha log-uniform on [0.01, 10]", "BJ config 4",
     "out[3] = 0.01 * pow(100.0, orc_u01(X[2]));", "out[3] = 0.01 * pow(1000.0, orc_u01(X[2]));"),
    ("config-4 inputs: u2 from block X instead of Y", "DESIGN s.5 (R12)",
     "out[6] = orc_u01(Y[1]);", "out[6] = orc_u01(X[3]);"),
    ("Philox: key schedule constant W0 off by one", "Salmon et al. SC'11",
     "const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;", "const uint32_t W0 = 0x9E3779B8u, W1 = 0xBB67AE85u;"),
    ("Philox: 9 rounds", "Philox4x32-10",
     "for (int round = 0; round < 10; ++round) {", "for (int round = 0; round < 9; ++round) {"),
    ("native (binary128): z = fma(1-u2, 1+ws.z, +ws.z)", "Listing 3, P:529; Fig. 4",
     "q128 z = fmaq(1 - u2, 1 + wz, -wz);", "q128 z = fmaq(1 - u2, 1 + wz, wz);"),
    ("ray cast: surface normal (ax P.x, ay P.y, P.z) instead of (ax^2 P.x, ...)", "P:353-380",
     "v3 n = normalize(mk(ax * ax * P.x, ay * ay * P.y, P.z));", "v3 n = normalize(mk(ax * P.x, ay * P.y, P.z));"),
    ("Eq. 10: cap density 1/(2 pi (1 - z_i))", "Eq. 10, P:759-766",
     "return 1.0 / (2.0 * ORC_PI * (1.0 + wi[2]));", "return 1.0 / (2.0 * ORC_PI * (1.0 - wi[2]));"),
    ("Eq. 8: reflection Jacobian 1/(2 |wo.wh|)", "Eq. 8, P:744-748",
     "return 1.0 / (4.0 * fabs(wo[0] * wh[0] + wo[1] * wh[1] + wo[2] * wh[2]));",
     "return 1.0 / (2.0 * fabs(wo[0] * wh[0] + wo[1] * wh[1] + wo[2] * wh[2]));"),
    ("Eq. 6: half vector of wi - wo", "Eq. 6, P:720-723",
     "v3 h = normalize(mk(wi[0] + wo[0], wi[1] + wo[1], wi[2] + wo[2]));",
     "v3 h = normalize(mk(wi[0] - wo[0], wi[1] - wo[1], wi[2] - wo[2]));"),
    ("pdf: h not flipped with wi (reading R4)", "reading R4",
     "return vndf_pdf_upper(mk(s * h[0], s * h[1], s * h[2]),", "return vndf_pdf_upper(mk(h[0], h[1], h[2]),"),
    ("uniform: u(w) = (w >> 9) 2^-23 (23 bits)", "DESIGN s.5",
     "double orc_u01(uint32_t w) { return (double)(w >> 8) * (1.0 / 16777216.0); }",
     "double orc_u01(uint32_t w) { return (double)(w >> 9) * (1.0 / 8388608.0); }"),
]

PIN_TESTS = ["tests/test_oracle_closed_forms.py", "tests/test_oracle_distribution.py",
             "tests/test_oracle_inputs.py", "tests/test_oracle_native.py",
             "tests/test_oracle_philox.py", "tests/test_oracle_reflect.py"]


def run_copy(src_text):
    tmp = tempfile.mkdtemp(prefix="orc_mut_")
    try:
        for d in ("oracle", "tests", "synth"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("*.so", "*.lock", "__pycache__"))
        shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
        with open(os.path.join(tmp, "oracle", "oracle.c"), "w") as f:
            f.write(src_text)
        env = dict(os.environ, PYTHONPATH=tmp)
        t0 = time.time()
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", *PIN_TESTS],
                           cwd=tmp, env=env, capture_output=True, text=True, timeout=1800)
        failed = ""
        for line in r.stdout.splitlines():
            if line.startswith("FAILED") or line.startswith("ERROR"):
                failed = line.split(" - ")[0].replace("FAILED ", "").replace("ERROR ", "")
                break
        return r.returncode, failed, time.time() - t0
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def main():
    src = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    rc, _, dt = run_copy(src)
    print(f"# control (unmutated oracle.c): pin suite rc={rc} ({dt:.0f} s)")
    assert rc == 0, "the unmutated oracle must pass its pins"
    caught = 0
    sel = [m for m in MUTANTS if len(sys.argv) < 2 or sys.argv[1] in m[0]]
    for name, cite, old, new in sel:
        n = src.count(old)
        assert n == 1, (name, n)
        rc, failed, dt = run_copy(src.replace(old, new))
        ok = rc != 0
        caught += ok
        print(f"{'CAUGHT ' if ok else 'ESCAPED'}  {name}  [{cite}]  -> {failed or 'all pins pass'}  ({dt:.0f} s)",
              flush=True)
    print(f"# {caught} of {len(sel)} mutants caught by the CPU pins")


if __name__ == "__main__":
    main()
