"""GPU: specialised functor kernels (csrc/hk_jit.cu) are bit-identical to the
interpreter (hk::run_program) -- chunk moments, per-row values and the
first-bad-row domain reporting -- so the policy switch never changes a result."""

from __future__ import annotations

import numpy as np
import pytest

from tests.common import B0_DAUGHTERS, B0_MASS, jit_cases, m12sq_builder

pytestmark = pytest.mark.gpu


def _bits(t):
    import torch
    return t.contiguous().view(torch.int64).cpu().numpy()


@pytest.fixture(scope="module")
def block(hk, cuda):
    spec = hk.DecaySpec(B0_MASS, B0_DAUGHTERS)
    return hk.phsp_generate(spec, hk.FourVector.at_rest(B0_MASS), 5 * 4096 + 517, hk.RngKey(11, 3))


def _moments(hk, block, prog):
    from paper_1711_05683_b200 import _lib
    from paper_1711_05683_b200.phasespace import _moment_partials
    bad = _lib.bad_cells(2)
    parts = _moment_partials(block, prog, bad)
    return _bits(parts), _lib.read_bad(bad)


def test_moments_and_map_bitwise(hk, block):
    from paper_1711_05683_b200 import _lib
    from paper_1711_05683_b200.functors import lower_average
    from paper_1711_05683_b200.phasespace import _map_program
    names = block.schema.names
    cols = block.device_columns()
    for name, expr, builder in jit_cases(hk):
        prog, _ = lower_average(expr, builder, names)
        with _lib.jit_mode(_lib.JIT_OFF):
            ref = _moments(hk, block, prog)
            ref_map = _map_program(prog, cols, len(block))
        with _lib.jit_mode(_lib.JIT_ALWAYS):
            got = _moments(hk, block, prog)
            got_map = _map_program(prog, cols, len(block))
        assert np.array_equal(got[0], ref[0]), name
        assert got[1] == ref[1], name
        assert np.array_equal(got_map.view(np.int64), ref_map.view(np.int64)), name


def test_domain_rows_match(hk, cuda):
    """Zero divisors and non-finite values report the same first rows.  A
    division in the expression tree (_BinaryOp "/") is checked
    (functors.py:200-207); numpy division inside an arg_builder is not -- it
    gives inf, which the average reports as non-finite (phasespace.py:314-316)."""
    from paper_1711_05683_b200 import _lib
    from paper_1711_05683_b200.functors import lower_average
    n = 3 * 4096 + 77
    rng = np.random.default_rng(5)
    a, b, w = rng.normal(size=n), rng.normal(size=n), rng.uniform(size=n)
    b[[9000, 400, 12000]] = 0.0
    a[[7000, 300]] = np.inf
    store = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("weight", "a", "b"), [w, a, b])
    ratio = hk.combine("/", hk.coordinate(0, 2), hk.coordinate(1, 2))
    for expr, builder, want in ((ratio, lambda c: (c["a"], c["b"]), [400, 300]),
                                (hk.identity(), lambda c: (c["a"] / c["b"],), [_lib.HK_NO_BAD_ROW, 300])):
        prog, _ = lower_average(expr, builder, store.schema.names)
        with _lib.jit_mode(_lib.JIT_OFF):
            ref = _moments(hk, store, prog)
        with _lib.jit_mode(_lib.JIT_ALWAYS):
            got = _moments(hk, store, prog)
        assert ref[1] == want
        assert got[1] == ref[1]
        assert np.array_equal(got[0], ref[0])
    with _lib.jit_mode(_lib.JIT_ALWAYS), pytest.raises(hk.EvaluationError, match="division by zero"):
        hk.phsp_average(ratio, store, lambda c: (c["a"], c["b"]))
    with _lib.jit_mode(_lib.JIT_ALWAYS), pytest.raises(hk.EvaluationError, match="non-finite model value at event 300"):
        hk.phsp_average(hk.identity(), store, lambda c: (c["a"] / c["b"],))


def test_auto_policy(hk, cuda):
    """auto: small blocks stay on the interpreter, >= HK_JIT_MIN_ROWS compiles
    once and the cached kernel then serves every size."""
    from paper_1711_05683_b200 import _lib
    L = _lib.lib()
    spec = hk.DecaySpec(B0_MASS, B0_DAUGHTERS)
    big = hk.phsp_generate(spec, hk.FourVector.at_rest(B0_MASS), _lib.HK_JIT_MIN_ROWS, hk.RngKey(2, 2))
    small = hk.phsp_generate(spec, hk.FourVector.at_rest(B0_MASS), 10_000, hk.RngKey(2, 2))
    unique = hk.constant(0.123456789012345)       # a program no other test compiles
    expr = hk.identity() * unique
    with _lib.jit_mode(_lib.JIT_AUTO):
        c0 = L.hk_jit_count()
        r_small = hk.phsp_average(expr, small, m12sq_builder)
        assert L.hk_jit_count() == c0
        r_big = hk.phsp_average(expr, big, m12sq_builder)
        assert L.hk_jit_count() == c0 + 1
        r_small2 = hk.phsp_average(expr, small, m12sq_builder)
        assert L.hk_jit_count() == c0 + 1
    assert r_small2.value == r_small.value and r_small2.error == r_small.error
    with _lib.jit_mode(_lib.JIT_OFF):
        r_big_interp = hk.phsp_average(expr, big, m12sq_builder)
    assert r_big.value == r_big_interp.value and r_big.error == r_big_interp.error


@pytest.mark.parametrize("n_daughters,rng,moving", [(3, "reference", False), (3, "philox", False),
                                                    (3, "reference", True), (5, "reference", False)])
def test_fused_integrate_bitwise(hk, cuda, n_daughters, rng, moving):
    """phsp_integrate: specialised generator+integrand == interpreter, chunk
    moments bit for bit (ragged tail chunk included)."""
    import torch
    from paper_1711_05683_b200 import _lib
    masses = (0.5, 0.3, 0.2, 0.1, 0.15)[:n_daughters]
    spec = hk.DecaySpec(B0_MASS, masses)
    mother = (hk.FourVector(float(np.hypot(B0_MASS, 3.0)), 1.0, -2.0, 2.0) if moving
              else hk.FourVector.at_rest(B0_MASS))
    n = 7 * 4096 + 1234
    for name, expr, builder in jit_cases(hk):
        def run():
            return hk.phsp_integrate(expr, spec, mother, n, hk.RngKey(4, 9), builder, rng=rng,
                                     return_partials=True)
        with _lib.jit_mode(_lib.JIT_OFF):
            ref = _bits(run())
        with _lib.jit_mode(_lib.JIT_ALWAYS):
            got = _bits(run())
        assert np.array_equal(got, ref), (name, n_daughters, rng, moving)
        torch.cuda.synchronize()
