"""The device math (csrc/hk_math.cuh: sincospi, exp) is __host__ __device__;
compile it for the CPU and check it against long double references."""

from __future__ import annotations

import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_device_math_accuracy(tmp_path):
    exe = tmp_path / "math_harness"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-std=c++17",
                    "-I", os.path.join(ROOT, "paper_1711_05683_b200", "csrc"),
                    os.path.join(ROOT, "tests", "math_harness.cpp"), "-o", str(exe)], check=True)
    out = json.loads(subprocess.run([str(exe), str(1 << 22)], capture_output=True, text=True,
                                    check=True).stdout)
    assert out["special_ok"], out
    assert out["sincospi_max_abs_err_ulp1"] <= 2.0, out   # absolute, in ulp(1) = 2.2e-16
    assert out["sincospi_gen_max_abs_err_ulp1"] <= 2.0, out
    assert out["exp_max_rel_err_ulp"] <= 2.0, out
