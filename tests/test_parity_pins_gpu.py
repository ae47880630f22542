"""GPU parity pins added in round 2 (VERDICT r01 "what's weak" 1-4): every
check here compares the CUDA path against the reference's own frozen outputs
(tests/golden, written by make_golden.py from the reference) or against the
CPU oracle pinned to them -- never CUDA against CUDA.

* the C4 FCN data set: generate_model_sample vs the reference sample (bits)
  and its 1e7-event fingerprints, nll at two points;
* weight sum / mean / variance vs golden and vs numpy on oracle windows;
* every functor-program opcode through phsp_average, map_evaluate and
  phsp_integrate vs numpy evaluation of the same expression;
* the Philox4x32-10 production stream: Random123 known answers on the
  device round function, the stream mapping, and generation/chains bit-exact
  against the oracle's Philox mode;
* yield-stationarity sums and sPlot V / sWeights vs the reference.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from tests.common import B0_DAUGHTERS, B0_MASS, M_JPSI, M_MU, assert_block_parity, jit_cases
from tests.test_oracle_golden import PHILOX_KAT

pytestmark = pytest.mark.gpu


def _toy(hk, scale: float, **values):
    """tests/toymodel.py build_model (the reference's toy) on the drop-in."""
    v = {"mean": 5.0, "sigma": 0.5, "tau": 3.0, "n_sig": 20000.0 * scale, "n_bkg": 30000.0 * scale}
    v.update(values)
    P = hk.Parameter
    region = hk.BoundedRegion(((0.0, 10.0),))
    mean = P("mean", v["mean"], step=0.1)
    sigma = P("sigma", v["sigma"], step=0.05, lower=1e-4)
    tau = P("tau", v["tau"], step=0.2, lower=1e-4)
    g, e = hk.shape_gaussian(mean, sigma), hk.shape_exponential(tau)
    n_sig = P("n_sig", v["n_sig"], step=max(v["n_sig"] ** 0.5, 1.0), lower=0.0)
    n_bkg = P("n_bkg", v["n_bkg"], step=max(v["n_bkg"] ** 0.5, 1.0), lower=0.0)
    return hk.add_pdfs([n_sig, n_bkg], [hk.make_pdf(g, hk.gaussian_norm(g), region),
                                        hk.make_pdf(e, hk.exponential_norm(e), region)])


def _set(model, values: dict) -> None:
    ps = model.param_set()
    for k, v in values.items():
        ps[k].set(v)


# ------------------------------------------------------------ C4 data set --
def test_model_sample_small_equals_reference_bits(cuda, hk, golden):
    """generate_model_sample(build_model(0.2), RngKey(7, 2), poisson=False) is
    the reference's sample bit for bit (golden nll_x, fitting.py:526-552)."""
    arrays, _ = golden
    got = np.asarray(hk.generate_model_sample(_toy(hk, 0.2), hk.RngKey(7, 2), poisson=False).column("x0"))
    want = arrays["nll_x"]
    assert got.shape == want.shape
    mism = int(np.count_nonzero(got.view(np.int64) != want.view(np.int64)))
    assert mism == 0, f"{mism} of {len(want)} samples differ from the reference"


def test_model_sample_poisson_equals_reference(cuda, hk, golden):
    """poisson=True: the component counts come from the same counter-based
    Poisson draw (fitting.py:516-523) and the rows are the reference's."""
    arrays, scalars = golden
    got = np.asarray(hk.generate_model_sample(_toy(hk, 0.2), hk.RngKey(7, 2), poisson=True).column("x0"))
    assert len(got) == scalars["c4"]["poisson_small_n"]
    assert np.array_equal(got.view(np.int64), arrays["c4_poisson_small_x"].view(np.int64))


def test_c4_dataset_fingerprints_and_nll(cuda, hk, golden):
    """The bench's 1e7-event FCN input: head, sum,
    SHA-256 of the bytes and a strided sample equal the reference's; nll at
    the truth and at (4.9, 0.55, 2.8) within 1e-10."""
    arrays, scalars = golden
    c4 = scalars["c4"]
    model = _toy(hk, 200)
    data = hk.generate_model_sample(model, hk.RngKey(7, 2), poisson=False)
    x = np.asarray(data.column("x0"))
    assert len(x) == c4["n"] == 10_000_000
    assert x[:8].tolist() == c4["head"]
    assert np.array_equal(x[arrays["c4_strided_idx"]], arrays["c4_strided_x"])
    assert hashlib.sha256(x.tobytes()).hexdigest() == c4["sha256"]
    assert float(np.sum(x)) == c4["xsum"]
    assert hk.nll(model, data, ["x0"]) == pytest.approx(c4["nll_truth"], rel=1e-10)
    _set(model, c4["alt_point"])
    assert hk.nll(model, data, ["x0"]) == pytest.approx(c4["nll_alt"], rel=1e-10)


# ------------------------------------------------------- weight moments ----
def test_weight_moments_vs_golden_and_numpy(cuda, hk, golden, oracle):
    """phsp_weight_moments: sum / mean / np.var(ddof=0) of the weights
    (test_phasespace.py:41) against the reference's C1 values and against
    numpy on oracle windows of the C2 run, both the fused-generation path and
    the standalone pass over a stored weight column."""
    _, scalars = golden
    c1 = scalars["c1"]
    spec, mother = hk.DecaySpec(B0_MASS, B0_DAUGHTERS), hk.FourVector.at_rest(B0_MASS)
    blk = hk.phsp_generate(spec, mother, c1["n"], hk.RngKey(1, 1))
    wm = hk.phsp_weight_moments(blk)
    assert wm.sum_w == pytest.approx(c1["wsum"], rel=1e-12)
    assert wm.mean == pytest.approx(c1["wmean"], rel=1e-12)
    assert wm.variance == pytest.approx(c1["wvar"], rel=1e-10)
    store = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("weight"), [np.asarray(blk.column("weight"))])
    alone = hk.phsp_weight_moments(store)
    assert alone.variance == pytest.approx(c1["wvar"], rel=1e-10)
    for start, n in ((0, 1_000_000), (50_000_000, 1_000_003), (99_000_000, 1_000_000)):
        w = oracle.generate(B0_DAUGHTERS, B0_MASS, n, 1, 1, ev_begin=start, threads=8)["weight"]
        got = hk.phsp_weight_moments(hk.phsp_generate(spec, mother, n, hk.RngKey(1, 1), row_offset=start))
        assert got.sum_w == pytest.approx(float(np.sum(w)), rel=1e-12), start
        assert got.mean == pytest.approx(float(np.mean(w)), rel=1e-12), start
        assert got.variance == pytest.approx(float(np.var(w)), rel=1e-10), start


# --------------------------------------------- functor programs vs numpy ---
def _numpy_f(expr, builder, cols: dict) -> np.ndarray:
    with np.errstate(all="ignore"):
        return np.asarray(expr.eval(tuple(np.asarray(a, dtype=float) for a in builder(cols))), dtype=float)


def _error_floor(value: float, sums) -> float:
    """Rounding floor of phsp_average's error (phasespace.py:341-349): the
    spread sum w^2 f^2 - 2 mu sum w^2 f + mu^2 sum w^2 cancels to ~0 for a
    near-constant f, leaving ~eps * mu^2 sum w^2 of noise, so error values
    below ~|mu| sqrt(eps sum w^2) / sum w are rounding, in the reference too."""
    sw, _, sw2, _, _ = sums
    return 10.0 * abs(value) * float(np.sqrt(np.finfo(float).eps * sw2)) / sw


@pytest.mark.parametrize("jit", ["interpreter", "specialised"])
def test_programs_vs_numpy(cuda, hk, oracle, jit):
    """Every opcode (jit_cases) through phsp_average (1e-10), map values
    (<= 4 ulp: exp/log/sqrt/div round like numpy up to libm ulps) and the
    fused phsp_integrate (1e-10 against oracle-generated events)."""
    from paper_1711_05683_b200 import _lib
    from paper_1711_05683_b200.functors import lower_average
    from paper_1711_05683_b200.phasespace import _map_program
    mode = _lib.JIT_OFF if jit == "interpreter" else _lib.JIT_ALWAYS
    spec, mother = hk.DecaySpec(B0_MASS, B0_DAUGHTERS), hk.FourVector.at_rest(B0_MASS)
    n = 5 * 4096 + 517
    blk = hk.phsp_generate(spec, mother, n, hk.RngKey(11, 3))
    host = {name: np.asarray(blk.column(name)) for name in blk.schema.names}
    ref_blk = oracle.generate(B0_DAUGHTERS, B0_MASS, n, 11, 3)
    for name, expr, builder in jit_cases(hk):
        f = _numpy_f(expr, builder, host)
        with _lib.jit_mode(mode):
            r = hk.phsp_average(expr, blk, builder)
            prog, _ = lower_average(expr, builder, blk.schema.names)
            got = _map_program(prog, blk.device_columns(), n)
            fused = hk.phsp_integrate(expr, spec, mother, n, hk.RngKey(11, 3), builder)
        v, e, sums = oracle.average(host["weight"], f)
        assert r.value == pytest.approx(v, rel=1e-10), name
        assert r.error == pytest.approx(e, rel=1e-10, abs=_error_floor(v, sums)), name
        np.testing.assert_array_max_ulp(got, f, maxulp=4)
        fr = _numpy_f(expr, builder, ref_blk)
        vr, er, sums_r = oracle.average(ref_blk["weight"], fr)
        # the fused path regenerates the events (|dp| <= 1e-12 E vs the
        # oracle); p1_e / p2_pz near pz = 0 amplifies that, hence 1e-9 there
        tol = 1e-9 if name == "ratio" else 1e-10
        assert fused.value == pytest.approx(vr, rel=tol), name
        assert fused.error == pytest.approx(er, rel=tol, abs=_error_floor(vr, sums_r)), name


# ------------------------------------------------ Philox production stream -
def test_philox_device_known_answers(cuda, hk, oracle):
    """The device Philox4x32-10 round function against the Random123 KATs and
    against the oracle on 2^16 random (ctr, key) rows."""
    torch = cuda
    from paper_1711_05683_b200 import _lib
    rs = np.random.default_rng(123)
    rows = np.concatenate([np.array([[*c, *k] for c, k, _ in PHILOX_KAT], dtype=np.uint32),
                           rs.integers(0, 2 ** 32, size=(1 << 16, 6), dtype=np.uint32)])
    d_in = torch.from_numpy(rows.view(np.int32)).cuda()
    d_out = torch.empty((rows.shape[0], 4), dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().hk_philox4x32_10(d_in.data_ptr(), rows.shape[0], d_out.data_ptr(),
                                           _lib.stream_ptr()), "hk_philox4x32_10")
    got = d_out.cpu().numpy().view(np.uint32)
    assert got[:3].tolist() == [list(o) for _, _, o in PHILOX_KAT]
    assert np.array_equal(got, oracle.philox4x32_10(rows[:, :4], rows[:, 4:]))


def test_philox_stream_and_generation_bit_exact(cuda, hk, oracle):
    """raw64 in Philox mode and phsp_generate(rng="philox") -- weights bit for
    bit, momenta <= 1e-12 E -- against the oracle's Philox mode, for 2- to
    8-body decays, a window at a far offset and a moving mother."""
    from paper_1711_05683_b200.rng import raw64
    ctr = np.array([0, 1, 2, 2 ** 40 + 7, 2 ** 64 - 1], dtype=np.uint64)
    assert np.array_equal(raw64(hk.RngKey(7, 1, 5), ctr, rng="philox"), oracle.philox_raw64(7, 1, 5, ctr))
    cases = [((0.3, 0.3), 1.0, 0), (B0_DAUGHTERS, B0_MASS, 0), (B0_DAUGHTERS, B0_MASS, 987_654_321_000),
             ((0.3, 0.1, 0.4, 0.2), 2.0, 0), ((0.1,) * 8, 2.0, 12345)]
    for masses, M, start in cases:
        n = 3 * 4096 + 77
        got = hk.phsp_generate(hk.DecaySpec(M, masses), hk.FourVector.at_rest(M), n, hk.RngKey(3, 1),
                               rng="philox", row_offset=start)
        ref = oracle.generate(masses, M, n, 3, 1, ev_begin=start, rng="philox")
        assert_block_parity(np.stack([np.asarray(got.column(c)) for c in got.schema.names]),
                            np.stack(list(ref.values())), len(masses), f"philox {len(masses)}-body @{start}")
        assert np.array_equal(np.asarray(got.column("weight")), ref["weight"])
    mom = (6.0, 1.3, -0.7, 2.9)
    m_m = float(np.sqrt(mom[0] ** 2 - mom[1] ** 2 - mom[2] ** 2 - mom[3] ** 2))
    spec = hk.DecaySpec(m_m, B0_DAUGHTERS)
    got = hk.phsp_generate(spec, hk.FourVector(*mom), 5000, hk.RngKey(9, 1), rng="philox")
    ref = oracle.generate(B0_DAUGHTERS, m_m, 5000, 9, 1, mother=mom, rng="philox")
    assert_block_parity(np.stack([np.asarray(got.column(c)) for c in got.schema.names]),
                        np.stack(list(ref.values())), 3, "philox moving")


def test_philox_chains_bit_exact(cuda, hk, oracle):
    """Decay chains in Philox mode (standalone and the fused C3 kernel) against
    the oracle's Philox-mode chain."""
    spec, mother = hk.DecaySpec(B0_MASS, B0_DAUGHTERS), hk.FourVector.at_rest(B0_MASS)
    sub = hk.DecaySpec(M_JPSI, (M_MU, M_MU))
    n = 2 * 4096 + 333
    parent = oracle.generate(B0_DAUGHTERS, B0_MASS, n, 1, 1, rng="philox")
    ref = oracle.decay_chain(parent, 1, (M_MU, M_MU), M_JPSI, 2, 1, rng="philox")
    ref_arr = np.stack(list(ref.values()))
    blk = hk.phsp_generate(spec, mother, n, hk.RngKey(1, 1), rng="philox")
    two = hk.phsp_decay_chain(blk, 1, sub, hk.RngKey(2, 1), rng="philox")
    fused = hk.phsp_generate_chain(spec, mother, n, hk.RngKey(1, 1), 1, sub, hk.RngKey(2, 1), rng="philox")
    for got, what in ((two, "two-step"), (fused, "fused")):
        arr = np.stack([np.asarray(got.column(c)) for c in got.schema.names])
        assert_block_parity(arr, ref_arr, 4, f"philox chain {what}")
        assert np.array_equal(arr[0], ref_arr[0])


# ------------------------------------------------- yield sums and sPlot ----
def test_yield_stationarity_vs_reference(cuda, hk, golden):
    """g_k and A_kj (fitting.py:401-434) at the truth and off the optimum,
    against the reference's own sums on the same data, 1e-10."""
    from paper_1711_05683_b200.fitting import _yield_stationarity
    arrays, scalars = golden
    data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [arrays["nll_x"]])
    for pt in scalars["yields_splot"]["points"]:
        model = _toy(hk, 0.2)
        _set(model, pt["values"])
        g, A = _yield_stationarity(model, data, ["x0"])
        np.testing.assert_allclose(g + 1.0, np.asarray(pt["g"]) + 1.0, rtol=1e-10, atol=0)
        np.testing.assert_allclose(g, np.asarray(pt["g"]), rtol=1e-6, atol=1e-10)
        np.testing.assert_allclose(A, np.asarray(pt["A"]), rtol=1e-10, atol=0)


def test_splot_vs_reference(cuda, hk, golden):
    """sPlot at the reference fit's parameters: V (splot.py:45-87) within
    1e-10, every sWeight (splot.py:90-117) within 1e-10 of the reference
    value (relative to the largest weight)."""
    arrays, scalars = golden
    ys = scalars["yields_splot"]
    data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [arrays["nll_x"]])
    model = _toy(hk, 0.2)
    _set(model, ys["fit_values"])
    V = hk.splot_matrix(model, data, ["x0"])
    np.testing.assert_allclose(V, np.asarray(ys["V"]), rtol=1e-10, atol=0)
    sw = hk.splot_weights(model, data, ["x0"], np.asarray(ys["V"]))
    got = np.stack([np.asarray(sw.column(n)) for n in sw.schema.names])
    want = arrays["splot_sw"]
    assert np.max(np.abs(got - want)) <= 1e-10 * np.max(np.abs(want))
