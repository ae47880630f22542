"""Shared fixtures.  `-m gpu` tests need a CUDA device and the built
libhepkit_cuda.so; everything else runs on the CPU (oracle, host logic,
ABI surface, gloo multi-process sharding)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libhepkit_cuda.so")


@pytest.fixture(scope="session")
def golden():
    arrays = np.load(os.path.join(GOLDEN, "golden.npz"))
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        scalars = json.load(fh)
    return arrays, scalars


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.lib()
    return O


@pytest.fixture(scope="session")
def hk():
    import paper_1711_05683_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def cuda(hk):
    """Fail loudly (not skip) when a gpu test runs without a device."""
    import torch
    assert torch.cuda.is_available(), "gpu test run without a CUDA device"
    from paper_1711_05683_b200 import _lib
    _lib.lib()
    return torch


B0 = (5.27966, (3.0969, 0.493677, 0.13957039))
M_MU = 0.1056583755
