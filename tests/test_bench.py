"""bench.py's output contract: one JSON line on stdout with the keys the driver
reads (the reference arm on CPU; our arm on a B200)."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    p = subprocess.run([sys.executable, os.path.join(REPO, "bench.py")] + args, cwd=REPO, capture_output=True,
                       text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, p.stdout  # nothing else on stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    import reforacle
    if not reforacle.available():
        pytest.skip("oracle/_ref not built")
    d = _run(["--impl", "reference", "--workload", "c1_single", "--steps", "1", "--warmup", "3"], 300)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "events/s"
    assert d["e2e"] == {"value": d["value"], "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] == 1
    assert d["warmup"] >= 3 and d["higher_is_better"] is True


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--steps", "3", "--warmup", "3", "--no-cpu-baseline"], 900)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["metric"] == "simulated_events_per_sec" and d["n_gpus"] == 1 and d["steps"] == 3
    assert d["config"]["replicas"] == 65536 and d["config"]["events_per_step"] == 880021538
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert d["clocks"]["samples"] > 0 and d["clocks"]["sm_mhz"] > 0
