"""The C ABI from a plain C host (examples/c_host.c): compiled with gcc against
libhepkit_cuda.so and cudart, no Python in the process -- what a cgo / JNI /
N-API binding of include/hepkit_cuda.h does.  Its results equal the Python
API's on the same rows."""

from __future__ import annotations

import json
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_host_generates_the_same_rows(cuda, hk, tmp_path):
    lib_dir = os.path.join(ROOT, "paper_1711_05683_b200")
    exe = str(tmp_path / "c_host")
    subprocess.run(["gcc", "-std=c99", "-O2", "-Wall", "-Werror", os.path.join(ROOT, "examples", "c_host.c"),
                    "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include", "-L" + lib_dir,
                    "-lhepkit_cuda", "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib_dir}", "-o", exe],
                   check=True, capture_output=True)
    n = 1_000_003
    out = subprocess.run([exe, str(n)], check=True, capture_output=True, text=True, timeout=300)
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["abi"] == hk._lib.lib().hk_abi_version() and r["n"] == n
    spec = hk.DecaySpec(5.27966, (3.0969, 0.493677, 0.13957039))
    blk = hk.phsp_generate(spec, hk.FourVector.at_rest(5.27966), n, hk.RngKey(1, 1))
    w = np.asarray(blk.column("weight"))
    assert [r["w0"], r["w1"], r["w2"]] == [float(v) for v in w[:3]]
    moments = hk.phsp_weight_moments(blk)
    assert abs(r["sum_w"] - moments.sum_w) <= 1e-12 * moments.sum_w
    assert abs(r["sum_w2"] - float(np.sum(w * w))) <= 1e-12 * r["sum_w2"]
    assert abs(r["host_sum_w"] - r["sum_w"]) <= 1e-12 * r["sum_w"]
    assert r["host_equals_device"] == 1
    assert r["bad_rc"] != 0 and "daughter" in r["bad_msg"]
