"""bench.py keeps the driver's JSON contract (one line on stdout).

CPU: the reference arm (`--impl reference`: the oracle port of the
reference engine on host cores) on C1.  GPU: the device arm's line carries
every key the contract names -- value / e2e / roofline / superstep
aggregate / cpu_baseline-free variant / clocks / gpu_launches."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _line(["--impl", "reference", "--config", "C1", "--steps", "3", "--warmup", "3"], 600)
    assert d["impl"] == "reference"
    assert d["unit"] == "GTEPS" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["steps"] == 3 and d["warmup"] == 3  # exactly K timed steps after W
    assert d["e2e"] == {"value": d["value"], "unit": "GTEPS", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["config"]["workload"].startswith("C1")


@pytest.mark.gpu
def test_device_arm_line():
    d = _line(["--steps", "3", "--warmup", "3", "--no-per-config", "--no-cpu-baseline"], 900)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "e2e", "gpu_launches", "roofline", "clocks", "superstep_aggregate"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3
    assert d["gpu_launches"] == 3 and d["value"] > 0
    assert d["config"]["workload"].startswith("C2")
    e = d["e2e"]
    assert e["unit"] == d["unit"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    agg = d["superstep_aggregate"]
    assert len(agg["per_superstep"]) == d["config"]["supersteps"]
