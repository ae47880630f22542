"""GPU: bench.py keeps the driver's JSON-line contract (a short run).

One line on stdout with the metric/value/unit/... keys, a roofline object for
the dominant kernel, clocks sampled in the timed region, an e2e object with
the bytes copied each step, and gpu_launches counted from the kernels the
step launches.  The reference arm prints the same shape with impl=reference.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches")


def _run(*args: str) -> dict:
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract(cuda):
    d = _run("--steps", "3", "--warmup", "3", "--no-cpu", "--no-configs", "--no-fcn")
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 1e9 and d["unit"] == "events/s" and d["dtype"] == "f64"
    assert d["config"]["workload"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0.2 < r["frac"] <= 1.0
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert d["gpu_launches"] == 3 * d["steps"]
    e = d["e2e"]
    assert e["value"] > 0 and e["d2h_bytes_per_step"] >= 104 * 10**8 and e["h2d_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_reference_arm_contract(cuda):
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "events/s"
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
