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
    assert d["config"]["workload"].startswith("C5")  # the headline at every N
    e = d["e2e"]
    assert e["unit"] == d["unit"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    agg = d["superstep_aggregate"]
    assert len(agg["per_superstep"]) == d["config"]["supersteps"]


def test_workload_strings_match_between_arms():
    """Both arms print the same config.workload for the same config (the
    driver's same_config check)."""
    sys.path.insert(0, ROOT)
    import bench
    from oracle import oracle as O
    n, off, tgt = O.rmat_csr(O.CONFIGS["C1"])
    ref = _line(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "3"], 600)
    assert ref["config"]["workload"] == bench.workload("C1", "pagerank", n, int(tgt.size))
    assert ref["config"]["workload"].startswith("C1: PageRank")


def test_reference_arm_caps_steps_to_its_budget():
    d = _line(["--impl", "reference", "--config", "C1", "--steps", "1000", "--warmup", "50",
               "--ref-budget", "0.5"], 600)
    assert d["steps_requested"] == 1000 and d["warmup_requested"] == 50
    assert 1 <= d["steps"] < 1000 and 1 <= d["warmup"] < 50
    assert f"{d['steps']} full C1" in d["cpu_baseline"]["sample"]


@pytest.mark.gpu
def test_device_arm_two_ranks_gloo():
    """torchrun --nproc-per-node 2 bench.py over gloo (functional: both
    ranks share the one GPU of the test box) on a C5-shaped small graph:
    the partitioned path's line, with the exchange of every superstep."""
    import socket

    def free_port():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            return s.getsockname()[1]
    env = dict(os.environ, PGX_DIST_BACKEND="gloo")
    for exchange, allowed in (("hybrid", {"dense", "sparse"}), ("dense", {"dense"}),
                              ("auto", {"dense", "sparse", "peer"})):
        out = subprocess.run(
            [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
             "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
             os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
             "--config", "C5S", "--exchange", exchange],
            capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
        assert out.returncode == 0, out.stderr[-3000:]
        lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
        assert len(lines) == 1, out.stdout
        d = json.loads(lines[0])
        assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0
        assert d["config"]["workload"].startswith("C5S")
        ex = d["config"]["exchange_per_superstep"]
        assert len(ex) == d["config"]["supersteps"] and set(ex) <= allowed, ex
        assert d["gpu_launches"] >= 2 * 3 * d["config"]["supersteps"]
        assert d["e2e"]["value"] > 0 and d["roofline"]["frac"] > 0
