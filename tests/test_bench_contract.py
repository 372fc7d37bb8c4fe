"""bench.py's output contract (the driver parses ONE JSON line): the CPU
reference arm (the oracle, this tier's reference) here, and a short GPU run of
our arm with every key the contract names (metric / unit from BASELINE.json,
roofline, e2e with the copied bytes, gpu_launches, clocks, cpu_baseline)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))


def run_bench(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def check_common(d, steps):
    assert d["metric"] == BASELINE["metric"]
    assert d["unit"] == "GDOF*it/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["steps"] == steps and d["warmup"] >= 3
    assert d["n_gpus"] == 1 and d["scaling"] == "weak" and d["vs_baseline"] is None
    assert d["dtype"] == "f64" and d["data"] == "synthetic"
    assert "200x200x25" in d["config"]["workload"]


def test_reference_arm_line():
    """`bench.py --impl reference`: the oracle on the host cores, same metric and
    config as our arm, with its own cpu_baseline and a zero-copy e2e."""
    d = run_bench("--impl", "reference", "--steps", "2", "--warmup", "3", timeout=600)
    check_common(d, 2)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_line():
    """A short run of our arm (no sweep, no CPU leg): every contract key."""
    d = run_bench("--steps", "3", "--warmup", "3", "--no-sweep", "--no-cpu", "--e2e-reps", "1",
                  "--e2e-iters", "5", "--apply-reps", "5")
    check_common(d, 3)
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["launches_timed"] >= 3 and r["launch_ms"] > 0
    e = d["e2e"]
    n = d["config"]["dofs_per_gpu_local"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 8 * n == e["d2h_bytes_per_step"]
    assert d["gpu_launches"] > 0
    c = d["clocks"]
    assert c["sm_max_mhz"] > 0 and isinstance(c["reasons"], list)
    assert d["cpu_baseline"] is None  # --no-cpu
