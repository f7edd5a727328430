"""bench.py's JSON-line contract (the driver parses these lines): the reference
arm on CPU, the N=1 arm on a GPU. Each runs bench.py as the driver does and
checks the keys and units of the one line it prints."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COMMON = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
          "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config")


def run_bench(*argv, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    """`bench.py --impl reference`: the reference's CPU engine (oracle/_ref, or
    the C port when it was not built) on the GPU arm's config and metric."""
    d = run_bench("--impl", "reference", "--steps", "2", "--warmup", "3")
    for k in COMMON:
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["unit"] == "us" and d["higher_is_better"] is False and d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == d["value"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_n1_line():
    """The default N=1 line: device-timed value, roofline against the measured
    HBM peak, CPU baseline, e2e through the C ABI with the bytes it moves, the
    launch count and clocks (bench.py asserts parity with the oracle itself)."""
    d = run_bench("--steps", "3", "--warmup", "3", "--no-sweep")
    for k in COMMON:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["unit"] == "us" and d["higher_is_better"] is False
    assert 0 < d["value"] < 100
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert r["algorithmic_bytes"] == 2 * 8 * (1 << 20)
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("reference", "port")
    e = d["e2e"]
    assert e["unit"] == "us" and e["value"] > d["value"]
    assert e["h2d_bytes_per_step"] == 8 * (1 << 20) and e["d2h_bytes_per_step"] == 8 * (1 << 20)
    assert e["python_api_us"] > 0
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
