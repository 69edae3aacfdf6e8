"""bench.py's contract on a B200 (short run): one JSON line on stdout with the
driver's keys, the contract keys first and the per-config summary last,
a roofline object whose fraction follows from its own numbers, and an e2e
object measured through the host entry point."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                        "--no-variants", "--no-cpu"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    keys = list(d)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches"):
        assert k in d, k
    assert keys[-1] == "summary" and keys.index("gpu_launches") < keys.index("fixups")
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 50.0  # Gsamples/s; config 4 runs at ~150 on a B200
    assert abs(d["value"] - (1 << 30) / (d["ms_per_step"] * 1e6)) / d["value"] < 2e-3
    rl = d["roofline"]
    assert rl["frac"] == pytest.approx(rl["achieved"] / rl["peak"], rel=1e-3) and 0.0 < rl["frac"] < 1.0
    assert 0.0 < rl["fma_pipe"]["frac"] < 1.0
    e = d["e2e"]
    assert e["value"] > 0 and e["d2h_bytes_per_step"] == 16 * e["samples_per_rank_per_step"]
    assert e["bit_identical_to_device"] is True
    assert d["gpu_launches"] == 2 * d["steps"] and d["fixups"]["count"] > 0
