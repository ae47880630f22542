"""GPU CSV writer (csrc/hk_csv.cu, ColumnStore.write_csv for device stores):
byte-identical to the reference's Python formatting (store.py:181-204,
f"{v:.17g}" per value) on random bit patterns of every magnitude, on the
awkward cases of the 'g' layout and on a generated phase-space block."""

from __future__ import annotations

import io

import numpy as np
import pytest

from tests.common import B0_DAUGHTERS, B0_MASS

pytestmark = pytest.mark.gpu


def _py_csv(names, cols) -> str:
    """The reference body (store.py:181-204) for real64 columns."""
    lines = [",".join(names)]
    for i in range(len(cols[0])):
        lines.append(",".join(f"{c[i]:.17g}" for c in cols))
    return "\n".join(lines) + "\n"


def _device_store(hk, names, cols):
    import torch
    return hk.ColumnStore.from_columns(hk.ColumnSchema.real64(*names),
                                       [torch.tensor(np.asarray(c, dtype=np.float64), device="cuda") for c in cols])


SPECIAL = [0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 2.0 / 3.0, 1e16, 1e17, 9.999999999999999e16, 1e-4, 1e-5,
           9.9999999999999995e-5, 0.00099999999999999998, 0.001, 123456789012345678.0, 2.0 ** 53,
           2.0 ** 53 + 2, 2.0 ** 63, 2.0 ** 64, 5e-324, 2.2250738585072014e-308, 2.225073858507201e-308,
           1.7976931348623157e308, 1e308, 1e-308, 1e22, 1e23, 9007199254740993.0, 0.3, 1.5, 2.5,
           float("inf"), float("-inf"), float("nan"), -float("nan"), 100.0, 1234.5, 5.27966,
           3.0969, 0.493677, 0.13957039, 0.1056583755, 1e-300, 4.9406564584124654e-324 * 3]


def test_special_values(hk, cuda):
    got = _device_store(hk, ["v"], [SPECIAL]).to_csv()
    assert got == _py_csv(["v"], [SPECIAL])


@pytest.mark.parametrize("seed", [1, 2])
def test_random_bit_patterns(hk, cuda, seed):
    """Every exponent, subnormals, NaN payloads: uniform random 64-bit patterns,
    plus values drawn log-uniformly over the normal range."""
    rs = np.random.default_rng(seed)
    bits = rs.integers(0, 2 ** 64, size=200_000, dtype=np.uint64).view(np.float64)
    logu = (10.0 ** rs.uniform(-310, 308, 200_000)) * rs.choice([-1.0, 1.0], 200_000)
    near = rs.uniform(-20, 20, 200_000)            # the fast (128-bit) path's range
    cols = [bits, logu, near]
    got = _device_store(hk, ["a", "b", "c"], cols).to_csv()
    want = _py_csv(["a", "b", "c"], cols)
    if got != want:
        g, w = got.splitlines(), want.splitlines()
        bad = [(i, g[i], w[i]) for i in range(min(len(g), len(w))) if g[i] != w[i]][:5]
        raise AssertionError(f"{len(g)} vs {len(w)} lines; first differences: {bad}")


def test_phase_space_block_and_roundtrip(hk, cuda):
    spec = hk.DecaySpec(B0_MASS, B0_DAUGHTERS)
    blk = hk.phsp_generate(spec, hk.FourVector.at_rest(B0_MASS), 50_000, hk.RngKey(1, 1))
    assert blk.on_device
    text = blk.to_csv()
    host = blk.to_host()
    assert not host.on_device
    assert text == host.to_csv()                    # GPU formatter == the Python body
    back = hk.read_csv(io.StringIO(text))
    for name in blk.schema.names:
        assert np.array_equal(back.column(name).view(np.int64), blk.column(name).view(np.int64))


def test_chunked_stream_and_files(hk, cuda, tmp_path):
    rs = np.random.default_rng(9)
    cols = [rs.normal(size=30_011), rs.exponential(size=30_011)]
    store = _device_store(hk, ["x", "y"], cols)
    want = _py_csv(["x", "y"], cols)
    buf = io.StringIO()
    store._write_csv_device(buf, chunk_bytes=4096)   # ~80 rows per chunk: many chunks, ragged tail
    assert buf.getvalue() == want
    path = tmp_path / "s.csv"
    store.write_csv(str(path))
    assert path.read_text() == want
    bio = io.BytesIO()
    store.write_csv(bio)
    assert bio.getvalue().decode() == want
    empty = _device_store(hk, ["x"], [np.zeros(0)])
    assert empty.to_csv() == "x\n"
