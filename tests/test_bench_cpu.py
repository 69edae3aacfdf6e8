"""bench.py's host-side pieces on the CPU: the roofline objects (HBM and issue
bounds) carry the contract's keys and consistent arithmetic, and the CPU
baseline times the oracle as it stands (bounded samples) and checks GPU-side
outputs against it (here: the oracle's own outputs, so zero error)."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def bench():
    import bench as b
    return b


def test_hbm_roofline_keys_and_arithmetic(bench):
    r = bench.roofline(738197504, 0.1068, "cap_pdf_c2")
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert r["achieved"] == pytest.approx(738197504 / 0.1068e-3 / 1e9, rel=1e-3)
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-3)
    assert r["traffic"] is None or r["traffic"] > 0


def test_issue_roofline(bench):
    r = bench.issue_roofline(150.0, "cap_philox_c4_warp_inst_per_sample")
    assert r is not None
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r
    assert r["bound"] == "alu" and r["unit"] == "Gwarp-inst/s"
    assert r["peak"] == pytest.approx(148 * 4 * 1.965, rel=1e-4)
    assert r["achieved"] == pytest.approx(150.0 * r["warp_inst_per_sample"], rel=1e-3)
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-3)
    assert r["gsamples_s_bound"] == pytest.approx(r["peak"] / r["warp_inst_per_sample"], rel=1e-3)
    f = r["fma_pipe"]  # the FMA-datapath bound (measured per-instruction costs)
    assert f["gsamples_s_bound"] == pytest.approx(148 * 4 * 1.965e9 * 32 / f["cycles_per_warp_sample"] / 1e9,
                                                  rel=1e-3)
    assert f["frac"] == pytest.approx(150.0 / f["gsamples_s_bound"], rel=1e-3)
    assert f["gsamples_s_bound"] < r["gsamples_s_bound"]  # tighter than the issue bound


def test_cpu_baseline_is_the_oracle(bench, orc):
    import synth
    idx = np.arange(5, 5 + 512, dtype=np.uint64)
    h, p, _ = orc.batch_sample_philox(orc.CAP, bench.C4_SEED, idx)
    x1 = synth.fill_numpy(1, 0, 1 << 10)
    x3 = synth.fill_numpy(3, 2, 1 << 12)
    r = bench.cpu_baseline(check=(idx, h.astype(np.float32), p.astype(np.float32)),
                           c1_planes=[x1[k] for k in synth.PLANES], c3_planes=[x3[k] for k in synth.PLANES],
                           budget_s=0.3, log2_sub=12)
    assert r["kind"] == "oracle" and r["cores"] >= 1 and r["value"] > 0
    for k in ("c4_2e24", "c1_2e16", "c3_2e24"):
        assert r["subranges"][k]["T_threads"] > 0 and r["subranges"][k]["1_thread"] > 0
    pv = r["parity_vs_gpu"]
    assert pv["samples"] == 512 and pv["over_tol"] == 0 and pv["max_abs_dh"] < 1e-6


def test_line_order_and_summary(bench):
    """The contract keys lead the JSON line; the per-config objects and then the
    summary close it (the driver keeps the line's contract keys and the tail of stdout)."""
    r = {"value": 147.0, "metric": "m", "unit": "u", "roofline": {"frac": 0.65, "fma_pipe": {"frac": 0.74}},
         "c3": {"gb_s": 7200.0, "frac_hbm": 1.1, "t_heitz_over_t_cap": 1.0}, "c1": {"cap_us": 1.9},
         "parity": {"over_tol": 0}, "cpu_baseline": {"value": 0.08}, "extra": 1}
    o = bench.ordered(r)
    keys = list(o)
    assert keys[:4] == ["metric", "value", "unit", "roofline"] and keys[-1] == "summary"
    assert keys[-4:-1] == ["c1", "c3", "parity"] and keys.index("extra") < keys.index("c1")
    s = o["summary"]
    assert s["c4_gsamples_s"] == 147.0 and s["c4_frac_fma_pipe"] == 0.74 and s["c3_gb_s"] == 7200.0
    assert s["c1_cap_us"] == 1.9 and s["c5_t_heitz_over_t_cap"] is None and s["parity_over_tol"] == 0
    assert o["extra"] == 1


def test_c5_over_tolerance_counts(bench, orc):
    """The cpu leg's oracle half of the config-5 robustness object: outputs equal
    to the oracle's count zero, a perturbed sample counts one."""
    import synth
    x = synth.fill_numpy(5, 4, 256)
    ins = [x[k] for k in synth.PLANES]
    kept = {"inputs": ins}
    for name, method in (("cap", orc.CAP), ("heitz", orc.HEITZ)):
        h, p, _ = orc.batch_sample(method, *ins, pdf=True)
        kept[name] = [h[0].astype(np.float32), h[1].astype(np.float32), h[2].astype(np.float32),
                      p.astype(np.float32)]
    kept["heitz"][0][7] += 1e-3
    robust = {"cap": {}, "heitz": {}}
    bench.c5_over_tolerance(robust, kept)
    assert robust["cap"]["over_tolerance"] == 0 and robust["heitz"]["over_tolerance"] == 1
    assert robust["cap"]["of_sampled"] == 256
