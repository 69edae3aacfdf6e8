"""bench.py's host-side pieces on the CPU: the roofline objects (HBM, issue and
instruction-mix bounds) carry the contract's keys and consistent arithmetic,
and the CPU baseline times the oracle as it stands (bounded sample)."""
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


def test_issue_and_mix_rooflines(bench):
    r = bench.issue_roofline(200.0, "cap_philox_c4_warp_inst_per_sample")
    assert r["bound"] == "alu" and r["unit"] == "Gsamples/s"
    ipc = float(r["model"].split("/ ")[1].split()[0])
    assert r["peak"] == pytest.approx(148 * 4 * 1.965e9 / ipc / 1e9, rel=1e-3)
    m = bench.mix_roofline(200.0)
    assert m["peak"] < r["peak"]  # the measured-rate bound is tighter than 1 inst/clk
    assert m["frac"] == pytest.approx(200.0 / m["peak"], rel=1e-3)


def test_cpu_baseline_is_the_oracle(bench, orc):
    import synth
    x = synth.fill_numpy(2, 1, 1 << 12)
    r = bench.cpu_baseline([x[k] for k in synth.PLANES], 1 << 12, budget_s=0.3)
    assert r["kind"] == "oracle" and r["cores"] >= 1 and r["value"] > 0
    assert r["value_1_thread"] > 0 and "samples" in r["sample"]
