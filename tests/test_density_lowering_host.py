"""Host-side checks of the FCN's density lowering (no GPU): the model traced
once with symbolic parameters (fitting._SymbolicDensity) gives the same
per-event densities as tracing at the current values, across parameter
points; closures that read state outside (x, p) keep the per-call trace."""

from __future__ import annotations

import numpy as np
import pytest

from tests.common import run_program_numpy
from tests.golden.generic_models import GENERIC_POINTS, generic_models


@pytest.fixture(scope="module")
def hk():
    import paper_1711_05683_b200 as hk
    return hk


def _numeric_density(fitting, model):
    """The per-call path: trace at the current values (no symbolic cache)."""
    dens, pdfs = fitting.density_nodes(model)
    roots, values = fitting.parametrize([dens, *pdfs])
    plan = fitting._DensityPlan(roots, len(values), model.arity, len(model.components))
    return plan.fill(values, [float(y.value) for y, _ in model.components])


def _points(model, rs, n=2000):
    lo_hi = [(0.6, 1.2)] if model.arity == 1 and "m0" in model.param_set() else [(0.0, 10.0)] * model.arity
    return [rs.uniform(lo, hi, n) for lo, hi in lo_hi]


@pytest.mark.parametrize("name,symbolic", [("g1", True), ("g2", True), ("g6", False)])
def test_symbolic_density_equals_per_call_trace(hk, name, symbolic):
    from paper_1711_05683_b200 import fitting
    rs = np.random.default_rng(3)
    model = generic_models(hk, np, GENERIC_POINTS[0])[name]
    cols = _points(model, rs)
    ps = model.param_set()
    for point in GENERIC_POINTS:
        for p in ps:
            if p.name in point:
                p.set(point[p.name])
        got = fitting.lower_density(model)
        assert bool(model._hk_sym) is symbolic
        want = _numeric_density(fitting, model)
        a, _ = run_program_numpy(got.program, cols)
        b, _ = run_program_numpy(want.program, cols)
        assert np.allclose(a, b, rtol=1e-14, atol=0.0)
        assert np.all(np.isfinite(a)) and np.all(a > 0)


def test_closure_reading_captured_state_is_retraced(hk):
    """A closure that reads a captured value is traced at every call, so a
    change of that value reaches the device program (the reference evaluates
    the closure on every call)."""
    from paper_1711_05683_b200 import fitting
    P = hk.Parameter
    scale = {"k": 2.0}
    a = P("a", 1.0)
    shape = hk.wrap_closure(lambda x, p: p["a"].value + scale["k"] * x[0], [a])
    model = hk.add_pdfs([P("n", 100.0)], [hk.make_pdf(shape, lambda r: 1.0, hk.BoundedRegion(((0.0, 1.0),)))])
    x = [np.linspace(0.1, 0.9, 9)]
    v1, _ = run_program_numpy(fitting.lower_density(model).program, x)
    assert model._hk_sym is False
    scale["k"] = 3.0
    v2, _ = run_program_numpy(fitting.lower_density(model).program, x)
    assert np.allclose(v2, 100.0 * (1.0 + 3.0 * x[0]), rtol=1e-15)
    assert not np.allclose(v1, v2)


def test_symbolic_path_raises_the_shape_errors(hk):
    """Value checks of the builtin shapes (sigma > 0) still run per call on
    the symbolic path, with the reference's exception and message."""
    from paper_1711_05683_b200 import fitting
    from paper_1711_05683_b200.functors import EvaluationError
    P = hk.Parameter
    mu, s = P("mu", 1.0), P("s", 0.5)
    g = hk.shape_gaussian(mu, s)
    bw = hk.wrap_closure(lambda x, p: 1.0 / ((x[0] - p["mu"].value) ** 2 + 1.0), [mu])
    region = hk.BoundedRegion(((0.0, 2.0),))
    model = hk.add_pdfs([P("n1", 10.0), P("n2", 5.0)],
                        [hk.make_pdf(g, lambda r: 1.0, region), hk.make_pdf(bw, lambda r: 1.0, region)])
    fitting.lower_density(model)
    assert model._hk_sym
    s.value = -1.0
    with pytest.raises(EvaluationError, match="sigma must be positive, got -1.0"):
        fitting.lower_density(model)


def test_many_components_lowering(hk):
    """Twelve components (above HK_MAX_COMPONENTS): the FCN's density has one
    pinned slot, the density itself with yield 1; a ratio / sWeight pass
    (_lower_pass) pins the density (yield 1) and the picked expressions
    (yield 0), so the kernels' d = sum_k N_k p_k is the density."""
    from paper_1711_05683_b200 import _lib, fitting
    rs = np.random.default_rng(5)
    model = generic_models(hk, np, GENERIC_POINTS[0])["g12"]
    K = len(model.components)
    assert K > _lib.HK_MAX_COMPONENTS
    x = [rs.uniform(0.0, 10.0, 3000)]
    dm = fitting.lower_density(model)
    assert dm.n_comp == 1 and dm.yield_[0] == 1.0
    dens, _, slots = run_program_numpy(dm.program, x, want_slots=True)
    assert np.array_equal(slots[dm.pdf_slot[0]], dens)
    sel = [0, 5, 11]
    pm = fitting._lower_pass(model, lambda pdfs: [pdfs[k] for k in sel])
    assert pm.n_comp == 1 + len(sel)
    assert list(pm.yield_[:pm.n_comp]) == [1.0, 0.0, 0.0, 0.0]
    d2, _, s2 = run_program_numpy(pm.program, x, want_slots=True)
    assert np.array_equal(d2, dens) and np.array_equal(s2[pm.pdf_slot[0]], dens)
    with np.errstate(all="ignore"):
        total = sum(float(y.value) * s2[pm.pdf_slot[1 + sel.index(k)]] for k, (y, _) in
                    enumerate(model.components) if k in sel)
    assert np.all(total < dens)
    with pytest.raises(ValueError):
        fitting._lower_pass(model, lambda pdfs: pdfs[:_lib.HK_MAX_COMPONENTS])
