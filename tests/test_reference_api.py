"""The reference's own behavioural contracts (pkg/tests/test_phasespace.py,
test_fitting.py, test_rng.py, test_acceptance.py criterion 2), exercised
against the drop-in package on the GPU.  Written independently; each test
names the reference test it mirrors."""

from __future__ import annotations

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _p4(block, k):
    return [np.asarray(block.column(f"p{k}_{c}")) for c in ("e", "px", "py", "pz")]


def _inv_mass(e, x, y, z):
    return np.sqrt(np.maximum(e * e - x * x - y * y - z * z, 0.0))


# --- test_phasespace.py::TestGenerate ---------------------------------------
def test_two_body_weight_constant_and_equal_to_breakup(cuda, hk):
    blk = hk.phsp_generate(hk.DecaySpec(1.0, (0.3, 0.3)), hk.FourVector.at_rest(1.0), 5000, hk.RngKey(1, 1))
    w = np.asarray(blk.column("weight"))
    ref = hk.breakup_momentum(1.0, 0.3, 0.3)
    assert np.max(np.abs(w - ref)) <= 1e-12 * ref
    assert np.var(w) <= 1e-12 * ref * ref


def test_pair_mass_inside_dalitz_bounds(cuda, hk):
    M, (m1, m2, m3) = 1.0, (0.15, 0.2, 0.25)
    blk = hk.phsp_generate(hk.DecaySpec(M, (m1, m2, m3)), hk.FourVector.at_rest(M), 20_000, hk.RngKey(2, 1))
    a, b = _p4(blk, 1), _p4(blk, 2)
    m12 = _inv_mass(*(u + v for u, v in zip(a, b)))
    assert m12.min() >= m1 + m2 - 1e-9 and m12.max() <= M - m3 + 1e-9


def test_four_momentum_conservation(cuda, hk):
    blk = hk.phsp_generate(hk.DecaySpec(2.0, (0.3, 0.1, 0.4, 0.2)), hk.FourVector.at_rest(2.0), 10_000,
                           hk.RngKey(3, 1))
    tot = [sum(_p4(blk, k)[c] for k in range(1, 5)) for c in range(4)]
    assert np.max(np.abs(tot[0] - 2.0)) <= 2e-9
    for c in (1, 2, 3):
        assert np.max(np.abs(tot[c])) <= 2e-9


def test_daughters_on_their_mass_shell(cuda, hk):
    ms = (0.3, 0.1, 0.4)
    blk = hk.phsp_generate(hk.DecaySpec(1.5, ms), hk.FourVector.at_rest(1.5), 10_000, hk.RngKey(4, 1))
    for k, m in enumerate(ms, start=1):
        assert np.max(np.abs(_inv_mass(*_p4(blk, k)) - m)) <= 1e-9 * max(m, 1e-6)


def test_boosted_mother_conservation(cuda, hk):
    beta = 0.8
    g = 1.0 / math.sqrt(1.0 - beta * beta)
    mother = hk.FourVector(g, 0.0, 0.0, g * beta)
    blk = hk.phsp_generate(hk.DecaySpec(1.0, (0.2, 0.2)), mother, 5000, hk.RngKey(5, 1))
    e = _p4(blk, 1)[0] + _p4(blk, 2)[0]
    pz = _p4(blk, 1)[3] + _p4(blk, 2)[3]
    assert np.max(np.abs(e - mother.e)) <= 1e-9 * mother.e
    assert np.max(np.abs(pz - mother.pz)) <= 1e-9 * mother.e


def test_worker_knob_has_no_effect(cuda, hk):
    spec, mother = hk.DecaySpec(1.0, (0.1, 0.1, 0.1)), hk.FourVector.at_rest(1.0)
    a = hk.phsp_generate(spec, mother, 150_000, hk.RngKey(7, 1), workers=1)
    b = hk.phsp_generate(spec, mother, 150_000, hk.RngKey(7, 1), workers=8)
    for name in a.schema.names:
        assert np.array_equal(a.column(name), b.column(name))


def test_two_body_direction_isotropic(cuda, hk):
    blk = hk.phsp_generate(hk.DecaySpec(1.0, (0.2, 0.3)), hk.FourVector.at_rest(1.0), 200_000, hk.RngKey(8, 1))
    e, x, y, z = _p4(blk, 1)
    cos = z / np.sqrt(x * x + y * y + z * z)
    assert abs(float(np.mean(cos))) < 5.0 / math.sqrt(3 * len(blk))


# --- TestMaxWeight / TestUnweight -------------------------------------------
def test_max_weight_bounds_a_million_events(cuda, hk):
    spec = hk.DecaySpec(1.0, (0.1, 0.1, 0.1))
    blk = hk.phsp_generate(spec, hk.FourVector.at_rest(1.0), 1_000_000, hk.RngKey(9, 1), workers=2)
    assert float(np.max(blk.column("weight"))) <= hk.phsp_max_weight(spec)


def test_unweight_contracts(cuda, hk):
    spec = hk.DecaySpec(1.0, (0.3, 0.3))
    blk = hk.phsp_generate(spec, hk.FourVector.at_rest(1.0), 2000, hk.RngKey(10, 1))
    out = hk.phsp_unweight(blk, float(blk.column("weight")[0]), hk.RngKey(10, 4))
    assert len(out) == len(blk) and np.all(out.column("weight") == 1.0)
    spec3 = hk.DecaySpec(1.0, (0.1, 0.1, 0.1))
    three = hk.phsp_generate(spec3, hk.FourVector.at_rest(1.0), 20_000, hk.RngKey(13, 1))
    kept = hk.phsp_unweight(three, hk.phsp_max_weight(spec3), hk.RngKey(13, 4))
    assert 0 < len(kept) < len(three)
    e_in, e_out = np.asarray(three.column("p1_e")), np.asarray(kept.column("p1_e"))
    assert np.array_equal(e_in[np.isin(e_in, e_out)], e_out)


# --- TestDecayChain ------------------------------------------------------------
def test_chain_schema_conservation_and_weights(cuda, hk):
    spec, sub = hk.DecaySpec(2.0, (0.9, 0.3)), hk.DecaySpec(0.9, (0.2, 0.3))
    blk = hk.phsp_generate(spec, hk.FourVector.at_rest(2.0), 5000, hk.RngKey(14, 1))
    ch = hk.phsp_decay_chain(blk, 1, sub, hk.RngKey(15, 1))
    assert ch.schema.names[1:5] == ("p1_e", "p1_px", "p1_py", "p1_pz")
    tot = [sum(_p4(ch, k)[c] for k in (1, 2, 3)) for c in range(4)]
    assert np.max(np.abs(tot[0] - 2.0)) <= 2e-9 and np.max(np.abs(tot[1])) <= 2e-9
    expected = hk.breakup_momentum(2.0, 0.9, 0.3) * hk.breakup_momentum(0.9, 0.2, 0.3)
    assert np.max(np.abs(np.asarray(ch.column("weight")) - expected)) <= 1e-12 * expected
    for k, m in ((1, 0.2), (2, 0.3), (3, 0.3)):
        assert np.max(np.abs(_inv_mass(*_p4(ch, k)) - m)) <= 1e-8 * max(m, 1e-6)


# --- TestAverage ------------------------------------------------------------------
def _m12sq(cols):
    e = cols["p1_e"] + cols["p2_e"]
    px = cols["p1_px"] + cols["p2_px"]
    py = cols["p1_py"] + cols["p2_py"]
    pz = cols["p1_pz"] + cols["p2_pz"]
    return (e * e - px * px - py * py - pz * pz,)


def test_weighted_and_unweighted_averages_agree(cuda, hk):
    spec = hk.DecaySpec(1.0, (0.1, 0.1, 0.1))
    blk = hk.phsp_generate(spec, hk.FourVector.at_rest(1.0), 400_000, hk.RngKey(23, 1))
    flat = hk.phsp_unweight(blk, hk.phsp_max_weight(spec), hk.RngKey(23, 4))
    rw = hk.phsp_average(hk.identity(), blk, _m12sq)
    ru = hk.phsp_average(hk.identity(), flat, _m12sq)
    assert abs(rw.value - ru.value) < 3 * math.hypot(rw.error, ru.error)


def test_average_worker_invariance(cuda, hk):
    blk = hk.phsp_generate(hk.DecaySpec(1.0, (0.1, 0.1, 0.1)), hk.FourVector.at_rest(1.0), 100_000,
                           hk.RngKey(24, 1))
    a = hk.phsp_average(hk.identity(), blk, _m12sq, workers=1)
    b = hk.phsp_average(hk.identity(), blk, _m12sq, workers=8)
    assert a.value == b.value and a.error == b.error


# --- test_acceptance.py criterion 2: Dalitz flatness of an unweighted sample ---
def test_unweighted_dalitz_plot_is_flat(cuda, hk):
    scipy_stats = pytest.importorskip("scipy.stats")
    M, ms = 1.0, (0.1, 0.1, 0.1)
    spec = hk.DecaySpec(M, ms)
    blk = hk.phsp_generate(spec, hk.FourVector.at_rest(M), 1_000_000, hk.RngKey(2, 1))
    flat = hk.phsp_unweight(blk, hk.phsp_max_weight(spec), hk.RngKey(2, 4))
    d1, d2, d3 = _p4(flat, 1), _p4(flat, 2), _p4(flat, 3)
    s12 = _inv_mass(*(a + b for a, b in zip(d1, d2))) ** 2
    s23 = _inv_mass(*(a + b for a, b in zip(d2, d3))) ** 2
    nb = 20
    e12 = np.linspace((ms[0] + ms[1]) ** 2, (M - ms[2]) ** 2, nb + 1)
    e23 = np.linspace((ms[1] + ms[2]) ** 2, (M - ms[0]) ** 2, nb + 1)
    counts, _, _ = np.histogram2d(s12, s23, bins=[e12, e23])

    def s23_range(s12v):
        m1, m2, m3 = ms
        E2 = (s12v - m1 * m1 + m2 * m2) / (2 * np.sqrt(s12v))
        E3 = (M * M - s12v - m3 * m3) / (2 * np.sqrt(s12v))
        p2 = np.sqrt(np.maximum(E2 * E2 - m2 * m2, 0))
        p3 = np.sqrt(np.maximum(E3 * E3 - m3 * m3, 0))
        return (E2 + E3) ** 2 - (p2 + p3) ** 2, (E2 + E3) ** 2 - (p2 - p3) ** 2

    inside = []
    for i in range(nb):
        lo, hi = s23_range(np.linspace(e12[i], e12[i + 1], 33))
        for j in range(nb):
            if np.max(lo) <= e23[j] and np.min(hi) >= e23[j + 1]:
                inside.append(counts[i, j])
    inside = np.asarray(inside)
    expect = inside.sum() / inside.size
    chi2 = float(np.sum((inside - expect) ** 2 / expect))
    assert scipy_stats.chi2.sf(chi2, inside.size - 1) > 0.001


# --- test_fitting.py ---------------------------------------------------------
def _toy(hk, scale=1.0, **over):
    v = {"mean": 5.0, "sigma": 0.5, "tau": 3.0, "n_sig": 20000.0 * scale, "n_bkg": 30000.0 * scale}
    v.update(over)
    region = hk.BoundedRegion(((0.0, 10.0),))
    mean = hk.Parameter("mean", v["mean"], step=0.1)
    sigma = hk.Parameter("sigma", v["sigma"], step=0.05, lower=1e-4)
    tau = hk.Parameter("tau", v["tau"], step=0.2, lower=1e-4)
    g, e = hk.shape_gaussian(mean, sigma), hk.shape_exponential(tau)
    ns = hk.Parameter("n_sig", v["n_sig"], step=max(v["n_sig"] ** 0.5, 1.0), lower=0.0)
    nb = hk.Parameter("n_bkg", v["n_bkg"], step=max(v["n_bkg"] ** 0.5, 1.0), lower=0.0)
    return hk.add_pdfs([ns, nb], [hk.make_pdf(g, hk.gaussian_norm(g), region),
                                  hk.make_pdf(e, hk.exponential_norm(e), region)])


def _store(hk, x):
    return hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [np.asarray(x, dtype=float)])


def test_nll_duplicate_events_double_the_event_sum(cuda, hk):
    model = _toy(hk)
    x = np.linspace(1.0, 9.0, 101)
    base = hk.nll(model, _store(hk, x), ["x0"])
    doubled = hk.nll(model, _store(hk, np.concatenate([x, x])), ["x0"])
    total = model.expected_total()
    assert doubled - total == pytest.approx(2.0 * (base - total), rel=1e-12)


def test_nll_worker_invariance_and_cache_equivalence(cuda, hk):
    model = _toy(hk)
    data = hk.generate_model_sample(model, hk.RngKey(51, 2))
    vals = {w: hk.nll(model, data, ["x0"], workers=w) for w in (1, 2, 8)}
    assert vals[1] == vals[2] == vals[8]
    seq = [{"mean": 5.1, "sigma": 0.52}, {"mean": 5.1, "sigma": 0.52}, {"mean": 4.9, "sigma": 0.48}]
    got = []
    for upd in seq:
        ps = model.param_set()
        for k, v in upd.items():
            ps[k].set(v)
        got.append(hk.nll(model, data, ["x0"]))
    fresh = [hk.nll(_toy(hk, **upd), data, ["x0"]) for upd in seq]
    assert got == fresh


def test_fit_recovers_truth_and_yield_sum(cuda, hk):
    model = _toy(hk, scale=0.2)
    data = hk.generate_model_sample(model, hk.RngKey(61, 2), workers=2)
    n = len(data)
    ps = model.param_set()
    ps["mean"].set(4.7)
    ps["sigma"].set(0.6)
    ps["tau"].set(2.6)
    res = hk.fit(model, data, ["x0"], workers=2)
    assert res.status is hk.FitStatus.CONVERGED
    total = ps["n_sig"].value + ps["n_bkg"].value
    assert total == pytest.approx(n, rel=1e-6)
    assert abs(total - n) < 3 * math.sqrt(n)
    truth = {"mean": 5.0, "sigma": 0.5, "tau": 3.0}
    for name in truth:
        assert abs((ps[name].value - truth[name]) / res.errors[name]) < 5


def test_pull_calibration_200_toys(cuda, hk):
    """test_acceptance.py criterion 3 (pull calibration): 200 toys of ~1e4
    events, each sampled on the GPU and fitted with the GPU FCN; pulls of all
    five parameters have |mean| < 0.15 and width in [0.85, 1.15], at most 2
    failed fits."""
    truth = {"mean": 5.0, "sigma": 0.5, "tau": 3.0, "n_sig": 4000.0, "n_bkg": 6000.0}
    pulls = {name: [] for name in truth}
    failed = 0
    for t in range(200):
        model = _toy(hk, scale=0.2)
        sample = hk.generate_model_sample(model, hk.RngKey(6, 2, counter=t << 40))
        res = hk.fit(model, sample, ["x0"])
        if res.status is not hk.FitStatus.CONVERGED:
            failed += 1
            continue
        ps = model.param_set()
        for name in pulls:
            pulls[name].append((ps[name].value - truth[name]) / res.errors[name])
    assert failed <= 2
    for name, vals in pulls.items():
        arr = np.asarray(vals)
        assert abs(float(np.mean(arr))) < 0.15, (name, float(np.mean(arr)))
        assert 0.85 <= float(np.std(arr, ddof=1)) <= 1.15, (name, float(np.std(arr, ddof=1)))


def test_fit_with_everything_fixed(cuda, hk):
    model = _toy(hk, scale=0.01)
    data = hk.generate_model_sample(model, hk.RngKey(62, 2))
    for p in model.param_set():
        p.fixed = True
    res = hk.fit(model, data, ["x0"])
    assert res.status is hk.FitStatus.CONVERGED and res.errors == {}
    assert res.nll_min == pytest.approx(hk.nll(model, data, ["x0"]), rel=1e-12)


def test_model_sample_sizes(cuda, hk):
    model = _toy(hk, scale=0.02)
    sizes = {len(hk.generate_model_sample(model, hk.RngKey(seed, 2))) for seed in range(5)}
    assert len(sizes) > 1
    assert len(hk.generate_model_sample(model, hk.RngKey(65, 2), poisson=False)) == 1000
    a = hk.generate_model_sample(model, hk.RngKey(66, 2), workers=1)
    b = hk.generate_model_sample(model, hk.RngKey(66, 2), workers=8)
    assert np.array_equal(a.column("x0"), b.column("x0"))


# --- test_rng.py ------------------------------------------------------------------
def test_uniform_contracts(cuda, hk):
    key = hk.RngKey(123, stream=0, counter=42)
    assert hk.uniform(key) == hk.uniform(key)
    assert hk.uniform(hk.RngKey(123).at(0)) != hk.uniform(hk.RngKey(123).at(1))
    idx = np.arange(1000, dtype=np.uint64)
    a = hk.uniform_array(hk.RngKey(5, stream=0), idx)
    b = hk.uniform_array(hk.RngKey(5, stream=1), idx)
    assert np.mean(a != b) > 0.99
    u = hk.uniform_array(hk.RngKey(2024), np.arange(1_000_000, dtype=np.uint64))
    assert abs(float(np.mean(u)) - 0.5) < 0.002 and u.min() >= 0.0 and u.max() < 1.0
    k2 = hk.RngKey(9, stream=2)
    assert hk.uniform(k2.at(1000)) == hk.uniform_array(k2.at(990), np.array([10], dtype=np.uint64))[0]


def test_sample_pdf_contracts(cuda, hk):
    flat = hk.constant(1.0)
    out = hk.sample_pdf(flat, hk.BoundedRegion(((0.0, 1.0),)), 10_000, hk.RngKey(3, 0), ceiling=1.0)
    assert len(out) == 10_000 and abs(float(np.mean(out.column("x0"))) - 0.5) < 0.012
    g = hk.shape_gaussian(hk.Parameter("mean", 0.5), hk.Parameter("sigma", 0.3))
    a = hk.sample_pdf(g, hk.BoundedRegion(((-2.0, 3.0),)), 150_000, hk.RngKey(6, 0), workers=1)
    b = hk.sample_pdf(g, hk.BoundedRegion(((-2.0, 3.0),)), 150_000, hk.RngKey(6, 0), workers=8)
    assert np.array_equal(a.column("x0"), b.column("x0"))
    with pytest.raises(ValueError):
        hk.sample_pdf(g, hk.BoundedRegion.cube(0, 1, 2), 10, hk.RngKey(1, 0))


# --- cli.py:193-204 (cmd_phsp) and cli.py:311-343 (cmd_bench): host callers -
def test_cli_phsp_sequence_on_the_drop_in(cuda, hk, oracle, tmp_path):
    """cmd_phsp's body, run against the drop-in: generate with the CLI's
    phase-space stream, unweight against phsp_max_weight with its unweight
    stream, write CSV.  The file parses back to the oracle's accepted events:
    same rows and count, weights 1.0, momenta within 1e-12 * E."""
    from tests.common import B0_DAUGHTERS, B0_MASS, assert_block_parity
    stream_phasespace, stream_unweight = 1, 4      # cli.py:50, :53
    seed, n = 2024, 50_000
    spec = hk.DecaySpec(B0_MASS, B0_DAUGHTERS)
    block = hk.phsp_generate(spec, hk.FourVector.at_rest(B0_MASS), n, hk.RngKey(seed, stream=stream_phasespace))
    w_max = hk.phsp_max_weight(spec)
    block = hk.phsp_unweight(block, w_max, hk.RngKey(seed, stream=stream_unweight))
    path = tmp_path / "phsp.csv"
    path.write_text(block.to_csv())
    back = hk.read_csv(str(path))
    ref = oracle.generate(B0_DAUGHTERS, B0_MASS, n, seed, stream_phasespace, threads=4)
    acc = oracle.unweight_accept(ref["weight"], w_max, seed, stream_unweight)
    want = np.stack([v[acc] for v in ref.values()])
    want[0] = 1.0
    got = np.stack([np.asarray(back.column(c)) for c in back.schema.names])
    assert back.schema.names == tuple(ref.keys()) and got.shape == want.shape
    assert np.all(got[0] == 1.0)
    assert_block_parity(got, want, 3, "cmd_phsp")


def test_cli_bench_sequence_on_the_drop_in(cuda, hk):
    """cmd_bench's body: a toy sample with poisson=False and workers=0, then
    nll timed at several worker counts -- every worker count returns the same
    value on the drop-in (workers is accepted and has no effect)."""
    region = hk.BoundedRegion(((0.0, 10.0),))
    g = hk.shape_gaussian(hk.Parameter("mean", 5.0), hk.Parameter("sigma", 1.0))
    e = hk.shape_exponential(hk.Parameter("tau", 4.0))
    model = hk.add_pdfs([hk.Parameter("n_gauss", 5e4), hk.Parameter("n_exp", 5e4)],
                        [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])
    sample = hk.generate_model_sample(model, hk.RngKey(7, stream=2), poisson=False, workers=0)
    assert len(sample) == 100_000
    values = {w: hk.nll(model, sample, ["x0"], workers=w) for w in (1, 2, 4, 8)}
    assert len(set(values.values())) == 1


# --- TestUnweight / TestAverage / TestMaxWeight: the remaining contracts --------
def test_unweight_two_body_accepts_all_and_names_a_violation(cuda, hk):
    """A 2-body decay's weight is its maximum (acceptance one); a ceiling below
    the block's largest weight raises the reference's "exceeds w_max"."""
    spec = hk.DecaySpec(1.0, (0.2, 0.25))
    blk = hk.phsp_generate(spec, hk.FourVector.at_rest(1.0), 5000, hk.RngKey(11, 1))
    assert len(hk.phsp_unweight(blk, hk.phsp_max_weight(spec), hk.RngKey(11, 4))) == len(blk)
    spec3 = hk.DecaySpec(1.0, (0.1, 0.1, 0.1))
    three = hk.phsp_generate(spec3, hk.FourVector.at_rest(1.0), 1000, hk.RngKey(12, 1))
    with pytest.raises(ValueError, match="exceeds w_max"):
        hk.phsp_unweight(three, float(np.max(three.column("weight"))) * 0.5, hk.RngKey(12, 4))


def test_average_of_one_and_the_empty_block(cuda, hk):
    blk = hk.phsp_generate(hk.DecaySpec(1.0, (0.1, 0.1, 0.1)), hk.FourVector.at_rest(1.0), 1000,
                           hk.RngKey(22, 1))
    r = hk.phsp_average(hk.constant(1.0), blk, lambda cols: (cols["weight"] * 0 + 1,))
    assert abs(r.value - 1.0) <= 1e-12 and abs(r.error) <= 1e-12
    with pytest.raises(ValueError, match="empty"):
        hk.phsp_average(hk.identity(), hk.ColumnStore(hk.phsp_schema(2)), lambda cols: (cols["weight"],))


def test_max_weight_two_body_and_threshold(cuda, hk):
    assert hk.phsp_max_weight(hk.DecaySpec(1.0, (0.3, 0.2))) == pytest.approx(
        hk.breakup_momentum(1.0, 0.3, 0.2), rel=1e-15)
    with pytest.raises(hk.BelowThreshold):
        hk.phsp_max_weight(hk.DecaySpec(1.0, (0.6, 0.5)))


@pytest.mark.parametrize("n", [1, 4095, 4097, 300_001])
@pytest.mark.parametrize("density", [0.0, 0.01, 0.5, 1.0])
def test_device_selection_equals_numpy(cuda, hk, n, density):
    """where_mask of a device store (the order-preserving compaction kernel
    behind phsp_unweight) equals numpy boolean indexing, column by column."""
    rs = np.random.default_rng(n + int(density * 100))
    blk = hk.phsp_generate(hk.DecaySpec(1.0, (0.1, 0.1, 0.1)), hk.FourVector.at_rest(1.0), n,
                           hk.RngKey(5, 1))
    mask = rs.random(n) < density
    sel = blk.where_mask(mask)
    assert len(sel) == int(mask.sum())
    for name in blk.schema.names:
        assert np.array_equal(np.asarray(sel.column(name)), np.asarray(blk.column(name))[mask])
