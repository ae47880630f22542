"""GPU: the FCN and its companion passes for ANY model the reference's nll
accepts (VERDICT r01 "what's missing" 1, 2, 5): closures, compositions,
observable arity 2, six and twelve components -- through the parametric functor program
(interpreter and NVRTC-specialised), against the reference's own values
frozen in tests/golden (make_golden.py add_generic_models), 1e-10.  Plus the
reference's error precedence (zero divisor vs non-positive density) and the
row-sharded FCN's NCCL path (one-rank group) against the one-pass value."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from tests.golden.generic_models import GENERIC_POINTS, generic_models

pytestmark = pytest.mark.gpu


def _stores(hk, arrays):
    s1 = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [arrays["g1_x"]])
    s2 = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0", "x1"), [arrays["g2_x"], arrays["g2_y"]])
    s6 = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [arrays["g6_x"]])
    s12 = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [arrays["g12_x"]])
    return {"g1": (s1, ["x0"]), "g2": (s2, ["x0", "x1"]), "g6": (s6, ["x0"]), "g12": (s12, ["x0"])}


@pytest.mark.parametrize("jit", ["interpreter", "specialised"])
def test_generic_models_nll_vs_reference(cuda, hk, golden, jit):
    from paper_1711_05683_b200 import _lib
    arrays, scalars = golden
    gen = scalars["generic"]
    stores = _stores(hk, arrays)
    mode = _lib.JIT_OFF if jit == "interpreter" else _lib.JIT_ALWAYS
    with _lib.jit_mode(mode):
        for i, pt in enumerate(GENERIC_POINTS):
            models = generic_models(hk, np, pt)
            for name in ("g1", "g2", "g6", "g12"):
                store, cols = stores[name]
                got = hk.nll(models[name], store, cols)
                assert got == pytest.approx(gen[name][i], rel=1e-10), (name, i)


def test_generic_program_compiles_once_per_structure(cuda, hk, golden):
    """Parameter changes reuse the specialised FCN module: the constants are
    kernel arguments, only a new op structure compiles."""
    from paper_1711_05683_b200 import _lib
    arrays, scalars = golden
    store, cols = _stores(hk, arrays)["g1"]
    L = _lib.lib()
    with _lib.jit_mode(_lib.JIT_ALWAYS):
        models = generic_models(hk, np, GENERIC_POINTS[0])
        m = models["g1"]
        hk.nll(m, store, cols)
        c0 = L.hk_jit_count()
        ps = m.param_set()
        vals = []
        for k in range(6):
            ps["m0"].set(0.89 + 0.002 * k)
            ps["g"].set(0.045 + 0.001 * k)
            ps["n_bw"].set(3000.0 + 10 * k)
            vals.append(hk.nll(m, store, cols))
        assert L.hk_jit_count() == c0
    assert len(set(vals)) == len(vals)
    with _lib.jit_mode(_lib.JIT_OFF):
        assert hk.nll(m, store, cols) == pytest.approx(vals[-1], rel=1e-14)


def test_generic_yield_sums_vs_reference(cuda, hk, golden):
    """Yield stationarity (fitting.py:401-434) for the six-component model
    (above the old four-component device limit) against the reference."""
    from paper_1711_05683_b200.fitting import _yield_stationarity
    arrays, scalars = golden
    store, cols = _stores(hk, arrays)["g6"]
    for i, pt in enumerate(GENERIC_POINTS):
        model = generic_models(hk, np, pt)["g6"]
        g, A = _yield_stationarity(model, store, cols)
        want = scalars["generic"]["g6_yields"][i]
        np.testing.assert_allclose(g + 1.0, np.asarray(want["g"]) + 1.0, rtol=1e-10, atol=0)
        np.testing.assert_allclose(A, np.asarray(want["A"]), rtol=1e-10, atol=0)


def test_many_components_vs_reference(cuda, hk, golden):
    """Twelve components, above the HK_MAX_COMPONENTS = 8 slots one pass
    pins: the FCN (one slot, the density), the yield sums (passes over
    pairs of component blocks) and the sWeights (passes over species
    blocks) against the reference's own values, 1e-10; the batched FCN
    against the single-point values."""
    from paper_1711_05683_b200.fitting import _yield_stationarity
    arrays, scalars = golden
    store, cols = _stores(hk, arrays)["g12"]
    for i, pt in enumerate(GENERIC_POINTS):
        model = generic_models(hk, np, pt)["g12"]
        assert len(model.components) == 12
        g, A = _yield_stationarity(model, store, cols)
        want = scalars["generic"]["g12_yields"][i]
        np.testing.assert_allclose(g + 1.0, np.asarray(want["g"]) + 1.0, rtol=1e-10, atol=0)
        np.testing.assert_allclose(A, np.asarray(want["A"]), rtol=1e-10, atol=0)
    model = generic_models(hk, np, GENERIC_POINTS[0])["g12"]
    sw = hk.splot_weights(model, store, cols, arrays["g12_V"])
    assert list(sw.schema.names) == [f"sw_z{k}" for k in range(12)]
    got = np.stack([np.asarray(sw.column(c)) for c in sw.schema.names])
    want = arrays["g12_sw"]
    assert np.max(np.abs(got - want)) <= 1e-10 * np.max(np.abs(want))
    one = hk.nll(model, store, cols)
    assert one == pytest.approx(scalars["generic"]["g12"][0], rel=1e-10)
    from paper_1711_05683_b200.fitting import nll_many
    ps = model.param_set()
    base = ps.values()
    iz = ps.names.index("z3")
    points = []
    for k in range(5):
        pt = list(base)
        pt[iz] = 900.0 + 7.0 * k
        points.append(pt)
    many = nll_many(model, store, cols, points)
    serial = []
    for pt in points:
        ps.set_values(pt)
        serial.append(hk.nll(model, store, cols))
    assert many == serial


def test_generic_splot_identities(cuda, hk, golden):
    """sPlot on a generic model: after the yield polish the species weights
    of each event sum to one and each species' weights sum to its yield
    (splot.py:1-15), through the program-driven kernels."""
    from paper_1711_05683_b200.fitting import _polish_yields
    arrays, _ = golden
    store, cols = _stores(hk, arrays)["g1"]
    model = generic_models(hk, np, dict(GENERIC_POINTS[0], n_bw=11500.0, n_poly=800.0))["g1"]
    for y in model.yields():
        y.lower = 0.0
    _polish_yields(model, store, cols, 1)
    g, _ = __import__("paper_1711_05683_b200.fitting", fromlist=["x"])._yield_stationarity(model, store, cols)
    assert np.max(np.abs(g)) < 1e-9
    V = hk.splot_matrix(model, store, cols)
    sw = hk.splot_weights(model, store, cols, V)
    w = np.stack([np.asarray(sw.column(c)) for c in sw.schema.names])
    np.testing.assert_allclose(w.sum(axis=0), 1.0, rtol=0, atol=1e-9)
    yields = [y.value for y in model.yields()]
    np.testing.assert_allclose(w.sum(axis=1), yields, rtol=1e-8)


def test_generic_error_precedence(cuda, hk):
    """A zero divisor in an expression-tree division raises EvaluationError
    with the point (functors.py:200-207); a closure's numpy division does
    not raise -- its inf density is reported as not positive
    (fitting.py:200-205); the earliest 65536-row batch wins."""
    P = hk.Parameter
    region = hk.BoundedRegion(((0.0, 10.0),))
    x = np.linspace(0.5, 9.5, 200_000)
    x[150_000] = 3.0                                   # batch 2
    x[70_000] = 7.0                                    # batch 1
    store = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
    c = P("c", 3.0)
    tree = hk.combine("/", hk.constant(1.0), hk.combine("-", hk.identity(), hk.wrap_closure(lambda v, p: p["c"].value + 0.0 * v[0], [c])))
    m1 = hk.add_pdfs([P("n", 1.0)], [hk.make_pdf(tree * tree, lambda r: 1.0, region)])
    with pytest.raises(hk.EvaluationError, match=r"division by zero at point \(np.float64\(3.0\),\)"):
        hk.nll(m1, store, ["x0"])
    clos = hk.wrap_closure(lambda v, p: 1.0 / (v[0] - 7.0) ** 2, [])
    m2 = hk.add_pdfs([P("n2", 1.0)], [hk.make_pdf(clos, lambda r: 1.0, region)])
    with pytest.raises(ValueError, match=r"model density np.float64\(inf\) is not positive at event 70000"):
        hk.nll(m2, store, ["x0"])
    both = hk.add_pdfs([P("a", 1.0), P("b", 1.0)], [hk.make_pdf(tree * tree, lambda r: 1.0, region),
                                                    hk.make_pdf(clos, lambda r: 1.0, region)])
    with pytest.raises(ValueError, match="is not positive at event 70000"):   # batch 1 before batch 2
        hk.nll(both, store, ["x0"])


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_nll_nccl_path_one_rank(cuda, hk, golden):
    """parallel.sharded_nll's device path -- asynchronous FCN pass, NCCL
    all-gather of the 8-double record, hk_nll_combine publishing into the
    mapped mailbox -- on a one-rank NCCL group equals nll(), for the closed
    form and a generic model, and reports a bad event by its global row."""
    import torch
    import torch.distributed as dist
    from paper_1711_05683_b200 import parallel
    arrays, _ = golden
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        x = arrays["nll_x"]
        P = hk.Parameter
        region = hk.BoundedRegion(((0.0, 10.0),))
        g, e = hk.shape_gaussian(P("mean", 5.0), P("sigma", 0.5)), hk.shape_exponential(P("tau", 3.0))
        toy = hk.add_pdfs([P("n_sig", 4000.0), P("n_bkg", 6000.0)],
                          [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])
        data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
        assert parallel.sharded_nll(toy, data, ["x0"], 0, _force_collective=True) == hk.nll(toy, data, ["x0"])
        store, cols = _stores(hk, arrays)["g2"]
        g2 = generic_models(hk, np, GENERIC_POINTS[1])["g2"]
        assert parallel.sharded_nll(g2, store, cols, 0, _force_collective=True) == hk.nll(g2, store, cols)
        bad = x.copy()
        bad[[2500, 700]] = np.nan
        bstore = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [bad])
        with pytest.raises(ValueError, match=r"not positive at event 1000700"):
            parallel.sharded_nll(toy, bstore, ["x0"], 1_000_000, _force_collective=True)
    finally:
        dist.destroy_process_group()


def _toy_model(hk, n_sig=4000.0, n_bkg=6000.0):
    P = hk.Parameter
    region = hk.BoundedRegion(((0.0, 10.0),))
    g = hk.shape_gaussian(P("mean", 5.0, step=0.1), P("sigma", 0.5, step=0.05, lower=1e-4))
    e = hk.shape_exponential(P("tau", 3.0, step=0.2, lower=1e-4))
    return hk.add_pdfs([P("n_sig", n_sig, step=60.0, lower=0.0), P("n_bkg", n_bkg, step=80.0, lower=0.0)],
                       [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])


@pytest.mark.parametrize("k", [1, 3, 4, 51, 70])
def test_nll_many_bitwise_equals_serial(cuda, hk, golden, k):
    """fitting.nll_many (hk_nll_eval_many: one data pass for all points) is
    bit-identical to k serial nll() calls, ragged tile included, and a bad
    point raises the serial path's error for the first such point."""
    from paper_1711_05683_b200.fitting import nll_many
    arrays, _ = golden
    x = np.concatenate([arrays["nll_x"], arrays["nll_x"][:777]])
    data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
    model = _toy_model(hk)
    ps = model.param_set()
    rs = np.random.default_rng(k)
    base = np.array(ps.values())
    pts = [tuple(base * (1.0 + 0.02 * rs.standard_normal(len(base)))) for _ in range(k)]
    got = nll_many(model, data, ["x0"], pts)
    assert ps.values() == tuple(base)
    want = []
    for pt in pts:
        ps.set_values(pt)
        want.append(hk.nll(model, data, ["x0"]))
    ps.set_values(tuple(base))
    assert np.array_equal(np.array(got), np.array(want))
    # generic model: per-point device passes, same values as serial
    g1 = generic_models(hk, np, GENERIC_POINTS[0])["g1"]
    s1 = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [arrays["g1_x"]])
    p1 = g1.param_set()
    b1 = p1.values()
    gp = [b1, tuple(v * 1.01 for v in b1)]
    gv = nll_many(g1, s1, ["x0"], gp)
    p1.set_values(gp[1])
    assert gv[1] == hk.nll(g1, s1, ["x0"])
    p1.set_values(b1)
    # a NaN observable: every point's density fails there; the first point's
    # error is raised, as by the serial evaluation
    xb = x.copy()
    xb[9000] = np.nan
    bdata = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [xb])
    with pytest.raises(ValueError) as want:
        ps.set_values(pts[0])
        hk.nll(model, bdata, ["x0"])
    ps.set_values(tuple(base))
    with pytest.raises(ValueError) as got_exc:
        nll_many(model, bdata, ["x0"], pts)
    assert str(got_exc.value) == str(want.value) == "model density np.float64(nan) is not positive at event 9000"
    assert ps.values() == tuple(base)


def test_fit_batched_objective_identical_to_serial(cuda, hk, golden):
    """fit() through NllObjective (batched simplex vertices and Hessian) ends
    at exactly the parameters, errors and call count of the serial objective
    (fitting.py:477-513), and numeric_errors gives the same errors bitwise."""
    from paper_1711_05683_b200.fitting import NllObjective, minimize, numeric_errors
    arrays, _ = golden
    data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [arrays["nll_x"]])
    m1, m2 = _toy_model(hk), _toy_model(hk)
    for m in (m1, m2):
        ps = m.param_set()
        ps["mean"].set(4.8)
        ps["sigma"].set(0.6)
        ps["tau"].set(2.5)
    r1 = minimize(NllObjective(m1, data, ["x0"]), m1.param_set())
    r2 = minimize(lambda _p: hk.nll(m2, data, ["x0"]), m2.param_set())
    assert r1.status == r2.status and r1.n_calls == r2.n_calls and r1.nll_min == r2.nll_min
    assert m1.param_set().values() == m2.param_set().values()
    assert r1.errors == r2.errors
    e1 = numeric_errors(NllObjective(m1, data, ["x0"]), m1.param_set())
    e2 = numeric_errors(lambda _p: hk.nll(m2, data, ["x0"]), m2.param_set())
    assert e1 == e2
    res = hk.fit(m1, data, ["x0"])
    assert res.status is hk.FitStatus.CONVERGED


def test_fcn_session_bitwise_and_lifecycle(cuda, hk, golden):
    """fcn_session: nll() through the resident CTAs equals the launched path
    bit for bit across changing parameters; the CTAs leave on idle and come
    back on the next call; a bad event stops the session and raises the
    reference error; other GPU work runs after the block."""
    import time
    from paper_1711_05683_b200 import _lib
    arrays, _ = golden
    x = np.concatenate([arrays["nll_x"]] * 3)[:29_999]
    data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
    model = _toy_model(hk, 12000.0, 18000.0)
    ps = model.param_set()
    pts = [(4000.0 * 3, 5.0, 0.5, 18000.0, 3.0), (12100.0, 4.9, 0.55, 17900.0, 2.8)]
    want = []
    for pt in pts:
        ps.set_values(pt)
        want.append(hk.nll(model, data, ["x0"]))
    with hk.fcn_session(model, data, ["x0"], idle_ms=20.0) as s:
        assert s.on
        got = []
        for i in range(10):
            ps.set_values(pts[i % 2])
            got.append(hk.nll(model, data, ["x0"]))
        assert got == [want[i % 2] for i in range(10)]
        time.sleep(0.1)                      # the CTAs leave on their idle timeout ...
        ps.set_values(pts[1])
        assert hk.nll(model, data, ["x0"]) == want[1]   # ... and come back
    assert not s.on
    t = cuda.ones(10, device="cuda")
    assert float(t.sum()) == 10.0
    bad = x.copy()
    bad[777] = np.nan
    bdata = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [bad])
    with pytest.raises(ValueError) as want_exc:
        hk.nll(model, bdata, ["x0"])
    with hk.fcn_session(model, bdata, ["x0"]) as s2:
        with pytest.raises(ValueError) as got_exc:
            hk.nll(model, bdata, ["x0"])
        assert not s2.on
    assert str(got_exc.value) == str(want_exc.value)
    # a generic model opens no session and keeps the launched path
    g1 = generic_models(hk, np, GENERIC_POINTS[0])["g1"]
    s1 = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [arrays["g1_x"]])
    with hk.fcn_session(g1, s1, ["x0"]) as s3:
        assert not s3.on
        assert hk.nll(g1, s1, ["x0"]) == pytest.approx(-116014.30412842518, rel=1e-10)
    assert _lib.lib().hk_fcn_session_stop() == 0


def test_nll_large_column_tma_path(cuda, hk):
    """Columns of >= 4096 x 4096 rows take the persistent TMA-pipelined FCN
    (k_nll_fast_tma); its value equals the single-pass nll_many evaluation
    (k_nll_many: same tiles, rows and fold) bit for bit, repeats bitwise, and
    matches the oracle within the FCN's 1e-10 budget, ragged tail included."""
    from oracle import oracle as O  # checker only
    from paper_1711_05683_b200.fitting import nll_many
    rs = np.random.default_rng(11)
    n = 4096 * 4096 + 4096 * 333 + 777
    x = np.clip(np.concatenate([rs.normal(5, 0.5, n // 2), rs.exponential(3.0, n - n // 2)]), 1e-3, 9.999)
    rs.shuffle(x)
    data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
    model = _toy_model(hk, 0.4 * n, 0.6 * n)
    ps = model.param_set()
    base = ps.values()
    pts = [base, (0.41 * n, 4.9, 0.55, 0.59 * n, 2.8)]
    got = []
    for pt in pts:
        ps.set_values(pt)
        got.append(hk.nll(model, data, ["x0"]))
        assert hk.nll(model, data, ["x0"]) == got[-1]
        want = O.nll(x, O.gauss_exp_components(pt[1], pt[2], pt[4], pt[0], pt[3]))
        assert abs(got[-1] - want) <= 1e-10 * abs(want)
    ps.set_values(base)
    assert nll_many(model, data, ["x0"], pts) == got


@pytest.mark.parametrize("mu,sigma,tau", [(5.0, 0.5, 3.0),      # the check-free kFcnFast path
                                          (9.0, 0.3, 0.2),      # q reaches ~65 > 59: kFcnFactored
                                          (1.0, 0.05, 50.0),    # q down to ~-23000: kFcnFactored
                                          (0.0, 2.0, 1e6)])     # nearly flat background
def test_nll_regimes_vs_oracle(cuda, hk, mu, sigma, tau):
    """The Gaussian + exponential FCN against the oracle at 1e-10 in each
    regime of the host proof (fast_coeffs): inside it the check-free kernel
    runs, outside it the factored kernel with its per-event fallback; the
    single-point, batched and repeated evaluations agree bit for bit."""
    from oracle import oracle as O  # checker only
    from paper_1711_05683_b200.fitting import nll_many
    rs = np.random.default_rng(5)
    n = 4096 * 300 + 123
    x = rs.uniform(1e-3, 9.999, n)
    data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
    P = hk.Parameter
    region = hk.BoundedRegion(((0.0, 10.0),))
    g = hk.shape_gaussian(P("mean", mu), P("sigma", sigma))
    e = hk.shape_exponential(P("tau", tau))
    model = hk.add_pdfs([P("n_sig", 0.3 * n), P("n_bkg", 0.7 * n)],
                        [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])
    got = hk.nll(model, data, ["x0"])
    want = O.nll(x, O.gauss_exp_components(mu, sigma, tau, 0.3 * n, 0.7 * n))
    assert abs(got - want) <= 1e-10 * abs(want)
    assert hk.nll(model, data, ["x0"]) == got
    assert nll_many(model, data, ["x0"], [model.param_set().values()] * 3) == [got] * 3


_SCAN_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1711_05683_b200 as hk
from paper_1711_05683_b200.fitting import nll_many
rs = np.random.default_rng(21)
x = np.clip(np.concatenate([rs.normal(5, 0.5, 400_000), rs.exponential(3.0, 600_123)]), 1e-3, 9.999)
data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
P = hk.Parameter
region = hk.BoundedRegion(((0.0, 10.0),))
g = hk.shape_gaussian(P("mean", 5.0), P("sigma", 0.5))
e = hk.shape_exponential(P("tau", 3.0))
m = hk.add_pdfs([P("n_sig", 4e5), P("n_bkg", 6e5)],
                [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])
vals = [hk.nll(m, data, ["x0"]) for _ in range(3)] + nll_many(m, data, ["x0"], [m.param_set().values()] * 5)
print(repr([float(v).hex() for v in vals]))
"""


def test_fcn_scan_direction_does_not_change_values(cuda):
    """The FCN's tile scan order is an L2 hint (csrc/hk_fcn.cu fcn_flip): last
    to first for columns within 0.85 of L2, alternating per call beyond
    (HK_FCN_REV_MAX_BYTES=0 forces alternation here).  Every order gives the
    same bits, single-point and batched."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = _SCAN_SCRIPT.format(root=root)
    outs = []
    for thr in ("0", str(1 << 40)):
        env = dict(os.environ, HK_FCN_REV_MAX_BYTES=thr)
        r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(eval(r.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1]
    assert len(set(outs[0])) == 1


def test_nll_random_models_vs_oracle(cuda, hk):
    """Randomised Gaussian + exponential models and data shapes against the
    oracle: whichever kernel the host proof (fast_coeffs) picks, the value
    matches at 1e-10, and a non-positive density raises the reference's
    message for the same event."""
    from oracle import oracle as O  # checker only
    rs = np.random.default_rng(2024)
    P = hk.Parameter
    region = hk.BoundedRegion(((0.0, 10.0),))
    import os
    checked = raised = 0
    cases = int(os.environ.get("HK_TEST_RANDOM_CASES", "40"))
    for case in range(cases):
        n = int(rs.integers(1, 200_000))
        kind = case % 3
        if kind == 0:
            x = rs.uniform(0.0, 10.0, n)
        elif kind == 1:
            x = np.clip(rs.normal(rs.uniform(0, 10), rs.uniform(0.05, 3), n), 1e-6, 10.0)
        else:
            x = np.clip(rs.exponential(rs.uniform(0.2, 20), n), 0.0, 10.0)
        mu, sigma = rs.uniform(-5, 15), 10 ** rs.uniform(-2, 0.7)
        tau = (10 ** rs.uniform(-1.3, 1.7)) * (1 if rs.random() < 0.85 else -1)
        n_sig, n_bkg = 10 ** rs.uniform(0, 6), 10 ** rs.uniform(0, 6)
        g = hk.shape_gaussian(P("mean", mu), P("sigma", sigma))
        e = hk.shape_exponential(P("tau", tau))
        model = hk.add_pdfs([P("n_sig", n_sig), P("n_bkg", n_bkg)],
                            [hk.make_pdf(g, hk.gaussian_norm(g), region),
                             hk.make_pdf(e, hk.exponential_norm(e), region)])
        data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
        norms = (O.gaussian_norm(mu, sigma, 0.0, 10.0), O.exponential_norm(tau, 0.0, 10.0))
        if not all(np.isfinite(v) and v > 0 for v in norms):
            # Pdf.norm's check comes first, as in the reference (fitting.py:80-89)
            with pytest.raises(ValueError, match="normalization must be positive and finite"):
                hk.nll(model, data, ["x0"])
            continue
        try:
            want = O.nll(x, O.gauss_exp_components(mu, sigma, tau, n_sig, n_bkg))
        except ValueError as exc:
            with pytest.raises(ValueError) as got:
                hk.nll(model, data, ["x0"])
            assert str(got.value) == str(exc)
            raised += 1
            continue
        got = hk.nll(model, data, ["x0"])
        assert abs(got - want) <= 1e-10 * max(abs(want), 1.0), (case, mu, sigma, tau, got, want)
        checked += 1
    assert checked >= cases // 2


def test_nll_random_closure_models_vs_numpy(cuda, hk):
    """Randomised Breit-Wigner + polynomial closure models (the density-program
    path, lowered once with symbolic parameters) against the reference
    semantics evaluated with numpy on the same closures, at 1e-10, through
    the interpreter and the NVRTC module alternately."""
    import math
    import os
    from paper_1711_05683_b200 import _lib
    rs = np.random.default_rng(77)
    P = hk.Parameter
    lo, hi = 0.6, 1.2
    cases = int(os.environ.get("HK_TEST_RANDOM_CASES", "30"))
    m0, g, c0, c1 = P("m0", 0.9), P("g", 0.05), P("c0", 1.0), P("c1", 0.5)
    bw = hk.wrap_closure(lambda x, p: 1.0 / ((x[0] - p["m0"].value) ** 2 + (0.5 * p["g"].value) ** 2), [m0, g])
    poly = hk.wrap_closure(lambda x, p: p["c0"].value + p["c1"].value * x[0], [c0, c1])
    region = hk.BoundedRegion(((lo, hi),))

    def bw_norm(r):
        h = 0.5 * g.value
        return (math.atan((hi - m0.value) / h) - math.atan((lo - m0.value) / h)) / h

    def poly_norm(r):
        return c0.value * (hi - lo) + 0.5 * c1.value * (hi * hi - lo * lo)

    n_bw, n_poly = P("n_bw", 1.0), P("n_poly", 1.0)
    model = hk.add_pdfs([n_bw, n_poly], [hk.make_pdf(bw, bw_norm, region), hk.make_pdf(poly, poly_norm, region)])
    for case in range(cases):
        n = int(rs.integers(1, 100_000))
        x = rs.uniform(lo, hi, n)
        data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
        m0.set(rs.uniform(0.7, 1.1)); g.set(10 ** rs.uniform(-2.5, -0.5))
        c0.set(rs.uniform(0.1, 2.0)); c1.set(rs.uniform(-0.1, 1.0))
        n_bw.set(10 ** rs.uniform(0, 5)); n_poly.set(10 ** rs.uniform(0, 5))
        d = (n_bw.value * (bw.eval((x,)) / bw_norm(region)) + n_poly.value * (poly.eval((x,)) / poly_norm(region)))
        want = n_bw.value + n_poly.value - float(np.sum(np.log(d)))
        with _lib.jit_mode(_lib.JIT_ALWAYS if case % 2 else _lib.JIT_OFF):   # NVRTC module / interpreter
            got = hk.nll(model, data, ["x0"])
        assert abs(got - want) <= 1e-10 * max(abs(want), 1.0), (case, got, want)
    assert model._hk_sym          # the symbolic lowering served every call


def test_many_components_first_bad_event(cuda, hk, golden):
    """Twelve components with a negative yield: nll, the yield sums (the
    density-only flag pass) and sWeights name the first event whose density
    is not positive -- the row a numpy restatement of the density finds
    (fitting.py:200-205, :416-418, splot.py:114)."""
    import math

    from paper_1711_05683_b200.fitting import _yield_stationarity
    from tests.golden.generic_models import G12_MEANS
    arrays, _ = golden
    store, cols = _stores(hk, arrays)["g12"]
    x = arrays["g12_x"]
    model = generic_models(hk, np, dict(GENERIC_POINTS[0], z5=-2.0e5))["g12"]
    # numpy restatement of sum_k N_k shape_k(x) / norm_k on [0, 10]
    dens = np.zeros_like(x)
    for i in range(10):
        mu, s, y = G12_MEANS[i], 0.2 + 0.03 * i, (-2.0e5 if i == 5 else 800.0 + 40.0 * i)
        nm = s * math.sqrt(2.0 * math.pi) * 0.5 * (math.erf((10.0 - mu) / (s * math.sqrt(2.0)))
                                                   - math.erf((0.0 - mu) / (s * math.sqrt(2.0))))
        dens += y * np.exp(-0.5 * ((x - mu) / s) ** 2) / nm
    tau = 2.5
    dens += 2000.0 * np.exp(-x / tau) / (tau * (1.0 - math.exp(-10.0 / tau)))
    dens += 1200.0 * np.ones_like(x) / 10.0
    bad = np.flatnonzero(~(dens > 0))
    assert bad.size and bad[0] > 0
    j = int(bad[0])
    assert abs(dens[j]) > 1e-6 * np.max(np.abs(dens))     # not a rounding-level crossing
    with pytest.raises(ValueError, match=rf"is not positive at event {j}$"):
        hk.nll(model, store, cols)
    with pytest.raises(ValueError, match=rf"model density is not positive at event {j}$"):
        _yield_stationarity(model, store, cols)
    with pytest.raises(ValueError, match=rf"is not positive at event {j}$"):
        hk.splot_weights(model, store, cols, np.eye(12))
