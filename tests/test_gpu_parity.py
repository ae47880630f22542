"""GPU parity: the sm_100a kernels (through the C ABI, via the package)
against the golden vectors frozen from the reference and against the CPU
oracle on the same seeded inputs.  Tolerances (north_star):

* RNG (reference stream), weights, counts, row order: bit-exact;
* four-momenta: |d| <= 1e-12 * E_daughter;
* integrals / averages / NLL: <= 1e-10 relative.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from tests.common import (B0_DAUGHTERS, B0_MASS, M_JPSI, M_MU, assert_block_parity, m12sq_builder,
                          m23sq_builder)

pytestmark = pytest.mark.gpu


def _arr(store) -> np.ndarray:
    return np.stack([np.asarray(store.column(n)) for n in store.schema.names])


def _b0(hk):
    return hk.DecaySpec(B0_MASS, B0_DAUGHTERS), hk.FourVector.at_rest(B0_MASS)


# --------------------------------------------------------------------- RNG --
def test_rng_known_answers(cuda, hk, golden):
    arrays, _ = golden
    ctr = arrays["rng_counters"]
    for i, k in enumerate(arrays["rng_keys"]):
        key = hk.RngKey(int(k[0]), int(k[1]), int(k[2]))
        assert np.array_equal(hk.rng.raw64(key, ctr), arrays["rng_raw64"][i])
        assert np.array_equal(hk.uniform_array(key, ctr), arrays["rng_uniform"][i])
    u = hk.uniform_array(hk.RngKey(7, 1), np.arange(4096, dtype=np.uint64))
    assert np.array_equal(u, arrays["rng_uniform_seq_7_1"])


def test_rng_large_counters_vs_oracle(cuda, hk, oracle):
    rs = np.random.default_rng(0)
    ctr = rs.integers(0, 2**63, size=1_000_000, dtype=np.int64).astype(np.uint64) * np.uint64(2)
    key = hk.RngKey(2**64 - 5, 3, 2**63 + 11)
    assert np.array_equal(hk.rng.raw64(key, ctr), oracle.raw64(key.seed, key.stream, key.counter, ctr))


def test_philox_stream_statistics(cuda, hk):
    u = hk.uniform_array(hk.RngKey(2024), np.arange(1_000_000, dtype=np.uint64), rng="philox")
    assert np.all((u >= 0) & (u < 1))
    assert abs(float(np.mean(u)) - 0.5) < 0.002
    assert abs(float(np.var(u)) - 1 / 12) < 0.001
    ref = hk.uniform_array(hk.RngKey(2024), np.arange(1000, dtype=np.uint64))
    assert np.mean(u[:1000] != ref) > 0.99


def test_philox_uniform_contracts(cuda, hk):
    """The reference's TestUniform contracts (test_rng.py:10-40), re-run on the
    Philox stream: deterministic, distinct counters differ, streams separate,
    key.counter offsets compose with array counters, range and 1e6-draw mean."""
    key = hk.RngKey(123, stream=0, counter=42)
    assert hk.uniform(key, rng="philox") == hk.uniform(key, rng="philox")
    k = hk.RngKey(123)
    assert hk.uniform(k.at(0), rng="philox") != hk.uniform(k.at(1), rng="philox")
    idx = np.arange(1000, dtype=np.uint64)
    a = hk.uniform_array(hk.RngKey(5, stream=0), idx, rng="philox")
    b = hk.uniform_array(hk.RngKey(5, stream=1), idx, rng="philox")
    assert np.mean(a != b) > 0.99
    k = hk.RngKey(9, stream=2)
    direct = hk.uniform(k.at(1000), rng="philox")
    shifted = hk.uniform_array(k.at(990), np.array([10], dtype=np.uint64), rng="philox")[0]
    assert direct == shifted
    u = hk.uniform_array(hk.RngKey(1), np.arange(100_000, dtype=np.uint64), rng="philox")
    assert np.all(u >= 0.0) and np.all(u < 1.0)
    u = hk.uniform_array(hk.RngKey(2024), np.arange(1_000_000, dtype=np.uint64), rng="philox")
    assert abs(float(np.mean(u)) - 0.5) < 0.002


# -------------------------------------------------------------- generation --
def test_generated_blocks_vs_golden(cuda, hk, golden):
    arrays, scalars = golden
    for b in scalars["gen_blocks"]:
        spec = hk.DecaySpec(b["M"], tuple(b["masses"]))
        blk = hk.phsp_generate(spec, hk.FourVector(*b["mother"]), b["rows"], hk.RngKey(*b["key"]))
        assert blk.schema.names == hk.phsp_schema(spec.n).names
        got = _arr(blk)
        ref = arrays["gen_" + b["name"]]
        assert_block_parity(got, ref, spec.n, b["name"])
        ok = ~np.isnan(ref[0])
        assert np.array_equal(got[0][ok], ref[0][ok]), f"{b['name']}: weights not bit-exact"


@pytest.mark.parametrize("n_daughters", [2, 3, 4, 5, 6, 7, 8, 9, 12])
def test_generate_vs_oracle_all_arities(cuda, hk, oracle, n_daughters):
    masses = tuple(0.05 + 0.031 * k for k in range(n_daughters))
    M = sum(masses) + 1.7
    n = 50_000 if n_daughters <= 8 else 8_000
    for rng_key in [(11, 1, 0), (12, 1, 777)]:
        blk = hk.phsp_generate(hk.DecaySpec(M, masses), hk.FourVector.at_rest(M), n, hk.RngKey(*rng_key))
        ref = oracle.generate(masses, M, n, *rng_key, threads=4)
        assert_block_parity(_arr(blk), np.stack(list(ref.values())), n_daughters, f"n={n_daughters}")
        assert np.array_equal(np.asarray(blk.column("weight")), ref["weight"])


def test_c1_full_size_vs_oracle_and_golden(cuda, hk, oracle, golden):
    _, scalars = golden
    spec, mother = _b0(hk)
    blk = hk.phsp_generate(spec, mother, 100_000, hk.RngKey(1, 1))
    ref = oracle.generate(B0_DAUGHTERS, B0_MASS, 100_000, 1, 1, threads=8)
    got = _arr(blk)
    assert_block_parity(got, np.stack(list(ref.values())), 3, "C1")
    assert np.array_equal(got[0], ref["weight"])
    assert float(np.sum(got[0])) == scalars["c1"]["wsum"]       # bit-exact weights -> same numpy sum
    for i, s in enumerate(scalars["c1"]["colsum"]):
        scale = np.sum(np.abs(got[1 + 4 * ((i - 1) // 4)])) if i else abs(s)
        assert abs(float(np.sum(got[i])) - s) <= 1e-12 * scale, i


def test_moving_mother_conservation(cuda, hk):
    spec = hk.DecaySpec(B0_MASS, B0_DAUGHTERS)
    p = (1.3, -0.7, 4.1)
    e = math.sqrt(B0_MASS ** 2 + sum(c * c for c in p))
    mother = hk.FourVector(e, *p)
    blk = hk.phsp_generate(spec, mother, 200_000, hk.RngKey(3, 1))
    tot = [sum(np.asarray(blk.column(f"p{k}_{c}")) for k in (1, 2, 3)) for c in ("e", "px", "py", "pz")]
    for got, want in zip(tot, (e, *p)):
        assert np.max(np.abs(got - want)) <= 1e-9 * e


def test_mother_mass_mismatch(cuda, hk):
    with pytest.raises(ValueError, match="does not match"):
        hk.phsp_generate(hk.DecaySpec(1.0, (0.2, 0.2)), hk.FourVector.at_rest(1.1), 10, hk.RngKey(6, 1))


def test_empty_and_ragged_sizes(cuda, hk, oracle):
    spec, mother = _b0(hk)
    assert len(hk.phsp_generate(spec, mother, 0, hk.RngKey(1, 1))) == 0
    for n in (1, 255, 4095, 4097, 12_289):
        blk = hk.phsp_generate(spec, mother, n, hk.RngKey(9, 1, 5))
        ref = oracle.generate(B0_DAUGHTERS, B0_MASS, n, 9, 1, 5)
        assert_block_parity(_arr(blk), np.stack(list(ref.values())), 3, f"n={n}")
        wm = hk.phsp_weight_moments(blk)
        assert wm.sum_w == pytest.approx(float(np.sum(ref["weight"])), rel=1e-13)


@pytest.mark.parametrize("masses,excess", [((0.13957039, 0.13957039, 0.493677), 1e-12),
                                           ((0.13957039, 0.13957039, 0.493677), 1e-9),
                                           ((3.0969, 0.493677), 1e-13),
                                           ((0.0, 0.0, 0.0), 1.0),
                                           ((0.0, 0.0), 1.0),
                                           ((0.0, 0.2, 0.0, 0.1), 0.5)])
def test_threshold_and_massless_edges_vs_oracle(cuda, hk, oracle, masses, excess):
    """Edges of the branch-free kernels: breakup lambda tiny or rounded
    negative just above threshold (np.maximum(lam, 0) as a sign mask, sqrt(+0)
    through the clamped seed), massless daughters (zero energies and frame
    masses), and the seed = stream = 0 key whose first uniform is exactly 0
    (cos theta = -1, sqrt(1 - cz^2) = sqrt(0))."""
    M = sum(masses) + excess
    spec, mother = hk.DecaySpec(M, masses), hk.FourVector.at_rest(M)
    n = 20_000
    for key in ((0, 0, 0), (5, 3, 0), (0, 0, 12_345)):
        blk = hk.phsp_generate(spec, mother, n, hk.RngKey(*key))
        ref = oracle.generate(masses, M, n, *key, threads=4)
        got = _arr(blk)
        assert_block_parity(got, np.stack(list(ref.values())), len(masses), f"{masses} +{excess} key {key}")
        assert np.array_equal(got[0], ref["weight"], equal_nan=True), "weights not bit-exact"
        # massless + u = 0 gives the reference's 0/0 NaNs (phasespace.py:67-71): same pattern
        assert np.array_equal(np.isnan(got), np.isnan(np.stack(list(ref.values())))), "NaN pattern"
    blk = hk.phsp_generate(spec, mother, 1, hk.RngKey(0, 0))
    assert np.array_equal(np.asarray(blk.column("weight")), oracle.generate(masses, M, 1, 0, 0)["weight"],
                          equal_nan=True)


def test_windows_equal_full_run_rows(cuda, hk):
    """Row offsets (GPU shards) and key.counter windows reproduce rows of a
    one-shot run bit for bit (phasespace.py:106)."""
    spec, mother = _b0(hk)
    full = _arr(hk.phsp_generate(spec, mother, 300_000, hk.RngKey(4, 1)))
    for s, n in ((123_457, 50_000), (4096 * 7, 4096 * 3), (299_999, 1)):
        by_key = _arr(hk.phsp_generate(spec, mother, n, hk.RngKey(4, 1, s)))
        by_off = _arr(hk.phsp_generate(spec, mother, n, hk.RngKey(4, 1), row_offset=s))
        assert np.array_equal(by_key, full[:, s:s + n], equal_nan=True)
        assert np.array_equal(by_off, full[:, s:s + n], equal_nan=True)


def test_large_window_vs_oracle(cuda, hk, oracle):
    """Config C2 size (1e8 events) generated in one launch; windows of it are
    checked against the oracle at far offsets (size-independent property)."""
    spec, mother = _b0(hk)
    n = 100_000_000
    blk = hk.phsp_generate(spec, mother, n, hk.RngKey(1, 1))
    w = blk.device_column("weight")
    for s in (0, 4096 * 9_999, 77_777_777, n - 1000):
        ref = oracle.generate(B0_DAUGHTERS, B0_MASS, 1000, 1, 1, ev_begin=s)
        got = np.stack([blk.device_column(c)[s:s + 1000].cpu().numpy() for c in blk.schema.names])
        assert_block_parity(got, np.stack(list(ref.values())), 3, f"window {s}")
    # weight integration over the full 1e8 block: fused moments == separate pass
    wm = hk.phsp_weight_moments(blk)
    blk.meta.pop("weight_partials")
    wm2 = hk.phsp_weight_moments(blk)
    assert wm.sum_w == pytest.approx(wm2.sum_w, rel=1e-12)
    assert wm.variance == pytest.approx(wm2.variance, rel=1e-10)
    torch = cuda
    assert wm.sum_w == pytest.approx(float(torch.sum(w)), rel=1e-10)
    assert float(torch.max(w)) <= hk.phsp_max_weight(spec)
    # conservation over the whole block (acceptance criterion 2, 1e-9 relative)
    for c, target in (("e", B0_MASS), ("px", 0.0), ("py", 0.0), ("pz", 0.0)):
        tot = sum(blk.device_column(f"p{k}_{c}") for k in (1, 2, 3))
        assert float(torch.max(torch.abs(tot - target))) <= 1e-9 * B0_MASS
    del blk, w


def test_host_buffer_generation_equals_device(cuda, hk):
    spec, mother = _b0(hk)
    n = 3 * 4096 * 100 + 17
    dev = _arr(hk.phsp_generate(spec, mother, n, hk.RngKey(8, 1)))
    host, sums = hk.phsp_generate_to_host(spec, mother, n, hk.RngKey(8, 1), stage_bytes=64 << 20)
    assert np.array_equal(_arr(host), dev, equal_nan=True)
    assert sums[0] == pytest.approx(float(np.sum(dev[0])), rel=1e-13)
    assert sums[1] == pytest.approx(float(np.sum(dev[0] ** 2)), rel=1e-13)


def test_philox_generation_physics(cuda, hk):
    spec, mother = _b0(hk)
    blk = hk.phsp_generate(spec, mother, 1_000_000, hk.RngKey(1, 1), rng="philox")
    w = np.asarray(blk.column("weight"))
    ref = hk.phsp_generate(spec, mother, 1_000_000, hk.RngKey(1, 1))
    wr = np.asarray(ref.column("weight"))
    assert not np.array_equal(w, wr)
    assert abs(w.mean() - wr.mean()) < 5 * math.sqrt(w.var() / len(w) + wr.var() / len(wr))
    assert w.max() <= hk.phsp_max_weight(spec)
    e = sum(np.asarray(blk.column(f"p{k}_e")) for k in (1, 2, 3))
    assert np.max(np.abs(e - B0_MASS)) <= 1e-9 * B0_MASS


# ------------------------------------------------------------------ chains --
def test_chain_vs_golden(cuda, hk, golden):
    arrays, _ = golden
    spec, mother = _b0(hk)
    sub = hk.DecaySpec(M_JPSI, (M_MU, M_MU))
    ch = hk.phsp_decay_chain(hk.phsp_generate(spec, mother, 256, hk.RngKey(1, 1)), 1, sub, hk.RngKey(2, 1))
    assert_block_parity(_arr(ch), arrays["chain_c3"], 4, "chain_c3")
    par = hk.phsp_generate(hk.DecaySpec(3.0, (0.3, 1.2)), hk.FourVector.at_rest(3.0), 128, hk.RngKey(21, 1))
    ch = hk.phsp_decay_chain(par, 2, hk.DecaySpec(1.2, (0.2, 0.3, 0.4)), hk.RngKey(22, 1))
    assert_block_parity(_arr(ch), arrays["chain_three_sub"], 4, "chain_three_sub")
    par = hk.phsp_generate(spec, mother, 64, hk.RngKey(1, 1, 5000))
    ch = hk.phsp_decay_chain(par, 1, sub, hk.RngKey(2, 1, 5000))
    assert_block_parity(_arr(ch), arrays["chain_c3_window_5000"], 4, "window")


def _fused_vs_two_step(fused, two, k: int, n_sub: int):
    """The fused chain against generate + decay_chain: weights and every
    parent-daughter column bit-identical; the sub-decay columns (the fixed-frame
    boost path, hk_phsp_generate_chain) within the parity budget |dc| <= 1e-12 E."""
    sub_rows = set(range(1 + 4 * (k - 1), 1 + 4 * (k - 1 + n_sub)))
    for r in range(fused.shape[0]):
        if r not in sub_rows:
            assert np.array_equal(fused[r], two[r], equal_nan=True), f"column {r} differs"
    assert_block_parity(fused, two, fused.shape[0] // 4, "fused vs two-step")


def test_fused_chain_equals_two_step(cuda, hk, oracle):
    spec, mother = _b0(hk)
    sub = hk.DecaySpec(M_JPSI, (M_MU, M_MU))
    n = 200_000
    two = _arr(hk.phsp_decay_chain(hk.phsp_generate(spec, mother, n, hk.RngKey(1, 1)), 1, sub,
                                   hk.RngKey(2, 1)))
    fused = hk.phsp_generate_chain(spec, mother, n, hk.RngKey(1, 1), 1, sub, hk.RngKey(2, 1))
    assert fused.schema.names == hk.phsp_schema(4).names
    _fused_vs_two_step(_arr(fused), two, 1, 2)
    ref = oracle.decay_chain(oracle.generate(B0_DAUGHTERS, B0_MASS, n, 1, 1, threads=8), 1,
                             (M_MU, M_MU), M_JPSI, 2, 1, threads=8)
    assert_block_parity(two, np.stack(list(ref.values())), 4, "C3")
    assert_block_parity(_arr(fused), np.stack(list(ref.values())), 4, "C3 fused")
    # sub-decay on daughter 3 (pion -> two photons-like massless pair): gamma
    # up to ~16 fails the fixed-frame bound, so this runs the per-event frame
    # mass path, bit-identical to the two-step chain
    sub3 = hk.DecaySpec(B0_DAUGHTERS[2], (0.0, 0.0))
    a = _arr(hk.phsp_generate_chain(spec, mother, 5000, hk.RngKey(5, 1), 3, sub3, hk.RngKey(6, 1)))
    b = _arr(hk.phsp_decay_chain(hk.phsp_generate(spec, mother, 5000, hk.RngKey(5, 1)), 3, sub3,
                                 hk.RngKey(6, 1)))
    assert np.array_equal(a, b, equal_nan=True)


def test_fused_chain_moving_mother_and_ragged(cuda, hk, oracle):
    """The fused chain with a boosted parent (the generator's non-ILP boost
    path) and a ragged size: against generate + decay_chain (parent columns
    and weights bit-identical) and within the parity budget of the oracle's
    generate + decay_chain."""
    spec = hk.DecaySpec(B0_MASS, B0_DAUGHTERS)
    p = (0.7, -1.9, 3.3)
    e = math.sqrt(B0_MASS ** 2 + sum(c * c for c in p))
    mother = hk.FourVector(e, *p)
    sub = hk.DecaySpec(M_JPSI, (M_MU, M_MU))
    n = 3 * 4096 + 1001
    fused = _arr(hk.phsp_generate_chain(spec, mother, n, hk.RngKey(8, 1), 1, sub, hk.RngKey(9, 1)))
    two = _arr(hk.phsp_decay_chain(hk.phsp_generate(spec, mother, n, hk.RngKey(8, 1)), 1, sub,
                                   hk.RngKey(9, 1)))
    _fused_vs_two_step(fused, two, 1, 2)
    par = oracle.generate(B0_DAUGHTERS, B0_MASS, n, 8, 1, mother=(e, *p), threads=4)
    ref = oracle.decay_chain(par, 1, (M_MU, M_MU), M_JPSI, 9, 1, threads=4)
    assert_block_parity(fused, np.stack(list(ref.values())), 4, "moving-mother chain")
    tot = [sum(fused[1 + 4 * k + c] for k in range(4)) for c in range(4)]
    for got, want in zip(tot, (e, *p)):
        assert np.max(np.abs(got - want)) <= 1e-9 * e


def test_fused_chain_fixed_frame_paths(cuda, hk, oracle):
    """The fixed-frame fused chain (frame mass = m_k, host-proved) with a
    three-body sub-decay (boost_m per daughter) against the two-step chain and
    the oracle; a sub-decay whose mother mass is off by 0.5 of the mismatch
    tolerance takes the per-event path (bit-identical to two-step, no error);
    one off by 2x the tolerance raises the reference's error at event 0."""
    spec, mother = _b0(hk)
    n = 3 * 4096 + 77
    sub = hk.DecaySpec(M_JPSI, (M_MU, M_MU, 0.0))
    fused = _arr(hk.phsp_generate_chain(spec, mother, n, hk.RngKey(3, 1), 1, sub, hk.RngKey(4, 1)))
    two = _arr(hk.phsp_decay_chain(hk.phsp_generate(spec, mother, n, hk.RngKey(3, 1)), 1, sub,
                                   hk.RngKey(4, 1)))
    _fused_vs_two_step(fused, two, 1, 3)
    ref = oracle.decay_chain(oracle.generate(B0_DAUGHTERS, B0_MASS, n, 3, 1, threads=4), 1,
                             (M_MU, M_MU, 0.0), M_JPSI, 4, 1, threads=4)
    assert_block_parity(fused, np.stack(list(ref.values())), 5, "fixed-frame 3-body sub")
    near = hk.DecaySpec(M_JPSI * (1 + 0.5e-9), (M_MU, M_MU))
    a = _arr(hk.phsp_generate_chain(spec, mother, 5000, hk.RngKey(3, 1), 1, near, hk.RngKey(4, 1)))
    b = _arr(hk.phsp_decay_chain(hk.phsp_generate(spec, mother, 5000, hk.RngKey(3, 1)), 1, near,
                                 hk.RngKey(4, 1)))
    assert np.array_equal(a, b, equal_nan=True)
    far = hk.DecaySpec(M_JPSI * (1 + 2e-9), (M_MU, M_MU))
    with pytest.raises(ValueError, match=r"event 0: daughter 1 mass .* does not match"):
        hk.phsp_generate_chain(spec, mother, 5000, hk.RngKey(3, 1), 1, far, hk.RngKey(4, 1))


def test_chain_mass_mismatch_names_event(cuda, hk):
    spec = hk.DecaySpec(2.0, (0.9, 0.3))
    blk = hk.phsp_generate(spec, hk.FourVector.at_rest(2.0), 100, hk.RngKey(20, 1))
    with pytest.raises(ValueError, match=r"event 0: daughter 1 mass .* does not match"):
        hk.phsp_decay_chain(blk, 1, hk.DecaySpec(0.8, (0.2, 0.3)), hk.RngKey(21, 1))
    with pytest.raises(ValueError, match="out of range"):
        hk.phsp_decay_chain(blk, 3, hk.DecaySpec(0.8, (0.2, 0.3)), hk.RngKey(21, 1))


# ---------------------------------------------------------------- averages --
def test_average_vs_golden(cuda, hk, golden):
    _, scalars = golden
    spec, mother = _b0(hk)
    blk = hk.phsp_generate(spec, mother, 100_000, hk.RngKey(1, 1))
    r = hk.phsp_average(hk.identity(), blk, m12sq_builder)
    v, e = scalars["c1"]["avg_m12sq"]
    assert r.value == pytest.approx(v, rel=1e-10) and r.error == pytest.approx(e, rel=1e-10)
    assert r.calls_used == 100_000 and r.iterations == 1
    mbw, gbw = scalars["c1"]["avg_bw_kstar"][2:]
    rb = hk.phsp_average(hk.breit_wigner(mbw, gbw), blk, m23sq_builder)
    assert rb.value == pytest.approx(scalars["c1"]["avg_bw_kstar"][0], rel=1e-10)
    assert rb.error == pytest.approx(scalars["c1"]["avg_bw_kstar"][1], rel=1e-10)
    r1 = hk.phsp_average(hk.constant(1.0), blk, lambda cols: (cols["weight"] * 0 + 1,))
    assert r1.value == pytest.approx(1.0, abs=1e-12) and r1.error == pytest.approx(0.0, abs=1e-12)


def test_fused_integrate_equals_stored_average(cuda, hk):
    spec, mother = _b0(hk)
    n = 1_000_000
    blk = hk.phsp_generate(spec, mother, n, hk.RngKey(1, 1))
    for expr, builder in ((hk.identity(), m12sq_builder),                     # pair fast path
                          (hk.breit_wigner(0.89555, 0.0473), m23sq_builder),  # pair fast path
                          (hk.identity() * hk.identity(), m12sq_builder)):    # interpreter
        a = hk.phsp_average(expr, blk, builder)
        b = hk.phsp_integrate(expr, spec, mother, n, hk.RngKey(1, 1), builder)
        assert b.value == pytest.approx(a.value, rel=1e-10)
        assert b.error == pytest.approx(a.error, rel=1e-10)


def test_survey_appendix_1e6_values(cuda, hk):
    spec, mother = _b0(hk)
    n = 1_000_000
    r = hk.phsp_integrate(hk.identity(), spec, mother, n, hk.RngKey(1, 1), m12sq_builder)
    assert r.value == pytest.approx(18.920064852245346, rel=1e-10)
    assert r.error == pytest.approx(0.0030180565813491982, rel=1e-10)
    wm = hk.phsp_weight_moments(hk.phsp_generate(spec, mother, n, hk.RngKey(1, 1)))
    assert wm.sum_w == pytest.approx(616817.9666723448, rel=1e-10)


def test_c5_full_size_chunk_partials(cuda, hk, oracle):
    """Config C5 at full size (1e10 events, fused, nothing stored) in one
    launch.  Size-independent properties: each 4096-row chunk's five moments
    depend only on that chunk's rows, so windows regenerated at far offsets
    give bit-identical partials -- including the ragged last chunk (1e10 is
    not a multiple of 4096) -- and match the oracle's chunk sums there."""
    spec, mother = _b0(hk)
    n = 10_000_000_000
    parts = hk.phsp_integrate(hk.identity(), spec, mother, n, hk.RngKey(1, 1), m12sq_builder,
                              return_partials=True)
    n_chunks = (n + 4095) // 4096
    assert parts.numel() == 5 * n_chunks
    for c0 in (0, 1_234_567, 2_000_000, n_chunks - 7):
        s = c0 * 4096
        m = min(7 * 4096, n - s)
        win = hk.phsp_integrate(hk.identity(), spec, mother, m, hk.RngKey(1, 1), m12sq_builder,
                                row_offset=s, return_partials=True)
        k = win.numel() // 5
        assert cuda.equal(win, parts[5 * c0:5 * (c0 + k)]), f"chunks {c0}..{c0 + k}"
        ref = oracle.generate(B0_DAUGHTERS, B0_MASS, m, 1, 1, ev_begin=s, threads=4)
        f = oracle.pair_mass2(ref, 1, 2) + 0.0
        got = win.view(k, 5).cpu().numpy()
        for j, (a, b) in enumerate(oracle.chunk_windows(m)):
            want = oracle.average(ref["weight"][a:b], f[a:b])[2]
            np.testing.assert_allclose(got[j], want, rtol=1e-12, err_msg=f"chunk {c0 + j}")
    tot = parts.view(n_chunks, 5).sum(0).cpu().numpy()
    mu = tot[1] / tot[0]
    assert mu == pytest.approx(18.920064852245346, rel=2e-4)   # the 1e6-event value, within MC error


def test_c3_full_size_chain_windows(cuda, hk, oracle):
    """Config C3's per-GPU shard (1.25e8 chained events = 1e9 / 8, 17 columns,
    17 GB) in one fused launch.  Windows at far offsets are regenerated by the
    oracle's generate + decay_chain, and four-momentum conservation holds over
    the whole block."""
    spec, mother = _b0(hk)
    sub = hk.DecaySpec(M_JPSI, (M_MU, M_MU))
    n = 125_000_000
    ch = hk.phsp_generate_chain(spec, mother, n, hk.RngKey(1, 1), 1, sub, hk.RngKey(2, 1))
    assert len(ch) == n
    for s in (0, 4096 * 12_345 + 17, 99_999_999, n - 1000):
        par = oracle.generate(B0_DAUGHTERS, B0_MASS, 1000, 1, 1, ev_begin=s)
        ref = oracle.decay_chain(par, 1, (M_MU, M_MU), M_JPSI, 2, 1, ev_begin=s)
        got = np.stack([ch.device_column(c)[s:s + 1000].cpu().numpy() for c in ch.schema.names])
        assert_block_parity(got, np.stack(list(ref.values())), 4, f"C3 window {s}")
    torch = cuda
    for c, target in (("e", B0_MASS), ("px", 0.0), ("py", 0.0), ("pz", 0.0)):
        tot = sum(ch.device_column(f"p{k}_{c}") for k in (1, 2, 3, 4))
        assert float(torch.max(torch.abs(tot - target))) <= 1e-9 * B0_MASS, c
    del ch


def test_average_errors(cuda, hk):
    spec, mother = _b0(hk)
    blk = hk.phsp_generate(spec, mother, 70_000, hk.RngKey(3, 1))
    with pytest.raises(ValueError, match="empty"):
        hk.phsp_average(hk.identity(), hk.ColumnStore(hk.phsp_schema(2)), lambda c: (c["weight"],))
    # log of a negative component -> non-finite at the first event
    with pytest.raises(hk.EvaluationError, match="non-finite model value at event"):
        hk.phsp_average(hk.wrap_closure(lambda x, p: np.log(x[0])), blk, lambda c: (c["p1_px"],))
    # division by zero inside the expression tree
    zero = hk.combine("/", hk.identity(), hk.constant(0.0))
    with pytest.raises(hk.EvaluationError, match="division by zero"):
        hk.phsp_average(zero, blk, m12sq_builder)


# --------------------------------------------------------------- unweight --
def test_unweight_vs_golden(cuda, hk, golden):
    arrays, scalars = golden
    spec, mother = _b0(hk)
    blk = hk.phsp_generate(spec, mother, 100_000, hk.RngKey(1, 1))
    out = hk.phsp_unweight(blk, hk.phsp_max_weight(spec), hk.RngKey(1, 4))
    assert len(out) == scalars["c1"]["unweight_count"]
    acc = np.unpackbits(arrays["c1_unweight_accept_bits"])[:100_000].astype(bool)
    src = np.asarray(blk.column("p1_e"))
    assert np.array_equal(np.asarray(out.column("p1_e")), src[acc])
    assert np.all(np.asarray(out.column("weight")) == 1.0)
    with pytest.raises(ValueError, match="exceeds w_max"):
        hk.phsp_unweight(blk, 0.5 * float(np.max(np.asarray(blk.column("weight")))), hk.RngKey(1, 4))


@pytest.mark.parametrize("n,offset", [(1, 0), (4095, 0), (4097, 0), (12_289, 7), (50_000, 1_234_567)])
def test_unweight_ragged_and_offset_vs_oracle(cuda, hk, oracle, n, offset):
    """Accept masks at ragged sizes and row offsets (the scan/compaction tail
    and the counter of a shard) equal the oracle's; order is preserved."""
    spec, mother = _b0(hk)
    w_max = hk.phsp_max_weight(spec)
    blk = hk.phsp_generate(spec, mother, n, hk.RngKey(6, 1), row_offset=offset)
    out = hk.phsp_unweight(blk, w_max, hk.RngKey(6, 4), row_offset=offset)
    w = np.asarray(blk.column("weight"))
    acc = oracle.unweight_accept(w, w_max, 6, 4, ev_begin=offset)
    assert len(out) == int(acc.sum())
    for c in ("p1_e", "p2_px", "p3_pz"):
        assert np.array_equal(np.asarray(out.column(c)), np.asarray(blk.column(c))[acc])
    assert np.all(np.asarray(out.column("weight")) == 1.0)


def test_where_mask_on_device(cuda, hk):
    spec, mother = _b0(hk)
    blk = hk.phsp_generate(spec, mother, 20_000, hk.RngKey(2, 1))
    mask = np.asarray(blk.column("weight")) > 0.6
    sel = blk.where_mask(mask)
    assert np.array_equal(np.asarray(sel.column("p2_pz")), np.asarray(blk.column("p2_pz"))[mask])


# -------------------------------------------------------------------- FCN --
def _model(hk, mean, sigma, tau, n_sig, n_bkg, lo=0.0, hi=10.0):
    region = hk.BoundedRegion(((lo, hi),))
    g = hk.shape_gaussian(hk.Parameter("mean", mean), hk.Parameter("sigma", sigma))
    e = hk.shape_exponential(hk.Parameter("tau", tau))
    return hk.add_pdfs([hk.Parameter("n_sig", n_sig), hk.Parameter("n_bkg", n_bkg)],
                       [hk.make_pdf(g, hk.gaussian_norm(g), region),
                        hk.make_pdf(e, hk.exponential_norm(e), region)])


def _store(hk, x):
    return hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [np.asarray(x, dtype=float)])


def test_nll_vs_golden(cuda, hk, golden):
    arrays, scalars = golden
    data = _store(hk, arrays["nll_x"])
    for pt, val in zip(scalars["nll"]["points"], scalars["nll"]["values"]):
        m = _model(hk, pt["mean"], pt["sigma"], pt["tau"], pt["n_sig"], pt["n_bkg"])
        assert hk.nll(m, data, ["x0"]) == pytest.approx(val, rel=1e-10)
    g = hk.shape_gaussian(hk.Parameter("mean", 0.0), hk.Parameter("sigma", 1.0))
    m1 = hk.add_pdfs([hk.Parameter("n", 1.0)], [hk.make_pdf(g, hk.gaussian_norm(g),
                                                             hk.BoundedRegion(((-10.0, 10.0),)))])
    assert hk.nll(m1, _store(hk, [0.0]), ["x0"]) == pytest.approx(1.9189385332046727, rel=1e-14)


def test_nll_large_vs_oracle(cuda, hk, oracle):
    rs = np.random.default_rng(7)
    n = 10_000_000
    x = np.concatenate([rs.normal(5.0, 0.5, 4 * n // 10), rs.exponential(3.0, 6 * n // 10)])
    x = x[(x > 0) & (x < 10)]
    data = _store(hk, x)
    for pt in ((5.0, 0.5, 3.0, 4e6, 6e6), (4.9, 0.55, 2.8, 4e6, 6e6), (5.2, 0.45, 3.3, 3.9e6, 6.1e6)):
        got = hk.nll(_model(hk, *pt), data, ["x0"])
        want = oracle.nll(x, oracle.gauss_exp_components(*pt))
        assert got == pytest.approx(want, rel=1e-10), pt


def test_nll_first_bad_event(cuda, hk, golden):
    arrays, scalars = golden
    x = arrays["nll_x"].copy()
    for j in (2500, 700, 2000):
        x[j] = np.nan
    with pytest.raises(ValueError) as exc:
        hk.nll(_model(hk, 5.0, 0.5, 3.0, 4000.0, 6000.0), _store(hk, x), ["x0"])
    assert str(exc.value) == scalars["nll"]["bad_message"]
    e = hk.shape_exponential(hk.Parameter("tau", 1.0))
    pdf = hk.make_pdf(e, hk.exponential_norm(e), hk.BoundedRegion(((0.0, 10.0),)))
    with pytest.raises(ValueError, match="event 0"):
        hk.nll(hk.add_pdfs([hk.Parameter("n", 0.0)], [pdf]), _store(hk, [1.0]), ["x0"])
    with pytest.raises(ValueError):
        hk.nll(_model(hk, 5.0, 0.5, 3.0, 1.0, 1.0), _store(hk, []), ["x0"])


def test_nll_extreme_tails_match_reference_semantics(cuda, hk, oracle):
    """The one-exp factored FCN path hands events whose exponents leave its
    safe window back to the reference-order density: tiny-but-positive
    densities still sum like the oracle, underflow to 0 and overflow to inf
    raise the reference's message at the same event."""
    rs = np.random.default_rng(3)
    base = np.concatenate([rs.normal(5.0, 0.5, 40_000), rs.exponential(3.0, 60_000)])
    pt = (5.0, 0.5, 3.0, 4e4, 6e4)
    comps = oracle.gauss_exp_components(*pt)
    # far tail, still positive and normal: exp(-x/tau) ~ e^-690 .. e^-708, below the
    # factored window (M < -700 here), so these take the reference-order density.
    # (Deeper tails make exp(-x/tau) subnormal, where the reference itself keeps
    # only a few significant bits and no evaluation order can agree to 1e-10.)
    tail = base.copy()
    tail[[17, 50_000, 99_999, 123]] = [2070.0, 2105.0, 2115.0, 2124.0]
    got = hk.nll(_model(hk, *pt), _store(hk, tail), ["x0"])
    assert got == pytest.approx(oracle.nll(tail, comps), rel=1e-10)
    # both terms underflow to 0 -> not positive, first such event reported
    under = base.copy()
    under[[70_000, 30_000]] = [1e6, 5e5]
    with pytest.raises(ValueError) as exc:
        oracle.nll(under, comps)
    with pytest.raises(ValueError) as got_exc:
        hk.nll(_model(hk, *pt), _store(hk, under), ["x0"])
    assert str(got_exc.value) == str(exc.value)
    # a rising exponential (tau < 0) overflows to inf
    pt2 = (5.0, 0.5, -3.0, 4e4, 6e4)
    comps2 = oracle.gauss_exp_components(*pt2)
    over = base.copy()
    over[[4242]] = [2500.0]
    with pytest.raises(ValueError) as exc, np.errstate(over="ignore"):   # the overflow is the point
        oracle.nll(over, comps2)
    with pytest.raises(ValueError) as got_exc:
        hk.nll(_model(hk, *pt2), _store(hk, over), ["x0"])
    assert str(got_exc.value) == str(exc.value)
    # and the regular rising-exponential case sums like the oracle
    assert hk.nll(_model(hk, *pt2), _store(hk, base), ["x0"]) == pytest.approx(oracle.nll(base, comps2),
                                                                                 rel=1e-10)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_row_sharded_nll(cuda, hk, oracle, world):
    """C4 at N GPUs, emulated on one: per-shard fused passes over zero-copy row
    views, folded in rank order (parallel.combine_nll_parts), equal the
    one-pass nll and the oracle; a bad event keeps its global index."""
    from paper_1711_05683_b200 import parallel
    from paper_1711_05683_b200.fitting import nll_event_sum
    rs = np.random.default_rng(11)
    x = np.concatenate([rs.normal(5.0, 0.5, 400_000), rs.exponential(3.0, 600_000)])
    x = x[(x > 0) & (x < 10)]
    pt = (4.9, 0.55, 2.8, 4e5, 6e5)
    model = _model(hk, *pt)
    data = _store(hk, x)

    def sharded(store):
        parts = []
        for r in range(world):
            shard, a = parallel.shard_rows(store, r, world)
            logsum, problem = nll_event_sum(model, shard, ["x0"])
            rec = np.zeros(parallel._PART + 1)
            rec[0], rec[1] = logsum, -1.0
            if problem is not None:
                row, kind, payload = problem
                rec[1], rec[2], rec[3], rec[-1] = a + row, kind, float(payload), 1
            parts.append(rec)
        return parallel.combine_nll_parts(parts, model.expected_total())

    got = sharded(data)
    assert got == pytest.approx(hk.nll(model, data, ["x0"]), rel=1e-12)
    assert got == pytest.approx(oracle.nll(x, oracle.gauss_exp_components(*pt)), rel=1e-10)
    assert parallel.sharded_nll(model, data, ["x0"], 0) == hk.nll(model, data, ["x0"])  # world 1
    bad = x.copy()
    bad[[len(x) - 5, len(x) // 2 + 3]] = np.nan
    with pytest.raises(ValueError) as want:
        hk.nll(model, _store(hk, bad), ["x0"])
    with pytest.raises(ValueError) as exc:
        sharded(_store(hk, bad))
    assert str(exc.value) == str(want.value)


def test_nll_data_stays_resident(cuda, hk):
    data = _store(hk, np.linspace(1.0, 9.0, 100_001))
    m = _model(hk, 5.0, 0.5, 3.0, 2e4, 3e4)
    a = hk.nll(m, data, ["x0"])
    t = data.device_column("x0")
    b = hk.nll(m, data, ["x0"])
    assert a == b and data.device_column("x0") is t


def test_sample_and_fit_end_to_end(cuda, hk):
    truth = dict(mean=5.0, sigma=0.5, tau=3.0, n_sig=4000.0, n_bkg=6000.0)
    model = _model(hk, **truth)
    ps = model.param_set()
    ps["sigma"].lower, ps["tau"].lower = 1e-4, 1e-4
    ps["n_sig"].lower = ps["n_bkg"].lower = 0.0
    ps["n_sig"].step, ps["n_bkg"].step = 60.0, 80.0
    ps["mean"].step, ps["sigma"].step, ps["tau"].step = 0.1, 0.05, 0.2
    data = hk.generate_model_sample(model, hk.RngKey(61, 2), poisson=False)
    assert len(data) == 10_000
    x = np.asarray(data.column("x0"))
    assert np.all((x >= 0) & (x < 10))
    again = hk.generate_model_sample(model, hk.RngKey(61, 2), poisson=False)
    assert np.array_equal(np.asarray(again.column("x0")), x)
    ps["mean"].set(4.7)
    ps["sigma"].set(0.6)
    ps["tau"].set(2.6)
    res = hk.fit(model, data, ["x0"])
    assert res.status is hk.FitStatus.CONVERGED
    assert ps["n_sig"].value + ps["n_bkg"].value == pytest.approx(len(data), rel=1e-6)
    for name in ("mean", "sigma", "tau"):
        assert abs(ps[name].value - truth[name]) / res.errors[name] < 5
    from paper_1711_05683_b200.fitting import _yield_stationarity
    g, _ = _yield_stationarity(model, data, ["x0"])
    assert np.max(np.abs(g)) < 1e-9


def test_sample_pdf_gaussian_ks(cuda, hk):
    g = hk.shape_gaussian(hk.Parameter("mean", 0.0), hk.Parameter("sigma", 1.0))
    n = 100_000
    x = np.sort(np.asarray(hk.sample_pdf(g, hk.BoundedRegion(((-6.0, 6.0),)), n, hk.RngKey(12, 0)).column("x0")))
    cdf = 0.5 * (1.0 + np.vectorize(math.erf)(x / math.sqrt(2.0)))
    dist = max(float(np.max(np.arange(1, n + 1) / n - cdf)), float(np.max(cdf - np.arange(n) / n)))
    assert dist < 1.63 / math.sqrt(n)
    with pytest.raises(hk.CeilingError, match="exceeds ceiling"):
        hk.sample_pdf(g, hk.BoundedRegion(((-6.0, 6.0),)), 1000, hk.RngKey(4, 0), ceiling=0.2)


# ------------------------------------------------- GPU-count invariance ----
def test_sharded_runs_bitwise_invariant(cuda, hk):
    """Shards generated separately (what N GPUs do) concatenate to the
    one-shot block, and their super-chunk records (hk_fold_supers, 1024 per
    run) fold to the same bits as the one-GPU total -- for weight moments and
    for a fused C5-style integration, at 2, 3, 4 and 8 shards."""
    from paper_1711_05683_b200 import _lib
    from paper_1711_05683_b200.parallel import shard_range, super_span
    from paper_1711_05683_b200.phasespace import _IntegrateRun
    torch = cuda
    spec, mother = _b0(hk)
    n = 2_000_003
    one = hk.phsp_generate(spec, mother, n, hk.RngKey(1, 1))
    ref_tot = _lib.weight_totals(one.meta["weight_partials"], n).cpu().numpy()
    ref_avg = hk.phsp_integrate(hk.identity(), spec, mother, n, hk.RngKey(1, 1), m12sq_builder)
    run = _IntegrateRun(hk.identity(), spec, mother, hk.RngKey(1, 1), m12sq_builder, "reference")
    for world in (2, 3, 4, 8):
        wsup, asup, cols = [], [], []
        for r in range(world):
            a, b = shard_range(n, r, world)
            s0, s1 = super_span(r, world)
            s = hk.phsp_generate(spec, mother, b - a, hk.RngKey(1, 1), row_offset=a)
            wsup.append(_lib.fold_supers(s.meta["weight_partials"], n, s0, s1, _lib.HK_WARP_SLICES, 2))
            cols.append(s.device_column("p2_px"))
            parts, flags = run.partials(b - a, a)
            assert flags == [_lib.HK_NO_BAD_ROW] * 2
            asup.append(_lib.fold_supers(parts, n, s0, s1, 1, 5))
        assert torch.equal(torch.cat(cols), one.device_column("p2_px"))
        tot = _lib.fold(torch.cat(wsup), _lib.HK_SUPERS, 2).cpu().numpy()
        assert np.array_equal(tot, ref_tot), world
        avg = _lib.fold(torch.cat(asup), _lib.HK_SUPERS, 5).cpu().numpy()
        assert avg[1] / avg[0] == ref_avg.value, world


def test_sharded_api_single_rank_matches_api(cuda, hk):
    """parallel.sharded_weight_moments / sharded_integrate without a process
    group (world 1) return the one-GPU API's bits, including an empty run's
    error and a store whose partials went stale after push()."""
    from paper_1711_05683_b200 import parallel
    spec, mother = _b0(hk)
    n = 300_017
    blk = hk.phsp_generate(spec, mother, n, hk.RngKey(1, 1))
    wm = hk.phsp_weight_moments(blk)
    tot = parallel.sharded_weight_moments(blk, n).cpu().numpy()
    assert (float(tot[0]), float(tot[1])) == (wm.sum_w, wm.sum_w2)
    got = parallel.sharded_integrate(hk.identity(), spec, mother, n, hk.RngKey(1, 1), m12sq_builder)
    want = hk.phsp_integrate(hk.identity(), spec, mother, n, hk.RngKey(1, 1), m12sq_builder)
    assert (got.value, got.error) == (want.value, want.error)
    with pytest.raises(ValueError, match="empty"):
        parallel.sharded_integrate(hk.identity(), spec, mother, 0, hk.RngKey(1, 1), m12sq_builder)
    small = hk.phsp_generate(spec, mother, 10, hk.RngKey(1, 1))
    before = hk.phsp_weight_moments(small)
    small.push([2.5] + [0.0] * 12)
    after = hk.phsp_weight_moments(small)
    assert after.n == 11 and after.sum_w == pytest.approx(before.sum_w + 2.5, rel=1e-15)


@pytest.mark.parametrize("n", [1, 2, 4095, 4096, 4097, 10_001, 123_457])
def test_nll_ragged_sizes_and_generic_models_vs_oracle(cuda, hk, oracle, n):
    """The FCN's tail tile and last-CTA fold at ragged sizes (factored
    Gaussian + exponential path), and the generic density path (three
    components: two Gaussians and an exponential) -- both within 1e-10 of the
    oracle's reference-order NLL."""
    rs = np.random.default_rng(n)
    x = np.clip(np.concatenate([rs.normal(5.0, 0.5, n // 2 + 1), rs.exponential(3.0, n)]), 1e-3, 9.999)[:n]
    region = hk.BoundedRegion(((0.0, 10.0),))
    g = hk.shape_gaussian(hk.Parameter("mean", 5.0), hk.Parameter("sigma", 0.5))
    e = hk.shape_exponential(hk.Parameter("tau", 3.0))
    store = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
    two = hk.add_pdfs([hk.Parameter("n_sig", 0.4 * n), hk.Parameter("n_bkg", 0.6 * n)],
                      [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])
    want = oracle.nll(x, oracle.gauss_exp_components(5.0, 0.5, 3.0, 0.4 * n, 0.6 * n))
    assert hk.nll(two, store, ["x0"]) == pytest.approx(want, rel=1e-10, abs=1e-9)
    g2 = hk.shape_gaussian(hk.Parameter("mean2", 2.0), hk.Parameter("sigma2", 1.5))
    three = hk.add_pdfs([hk.Parameter("a", 0.3 * n), hk.Parameter("b", 0.2 * n), hk.Parameter("c", 0.5 * n)],
                        [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(g2, hk.gaussian_norm(g2), region),
                         hk.make_pdf(e, hk.exponential_norm(e), region)])
    comps = [("gauss", 0.3 * n, 5.0, 0.5, oracle.gaussian_norm(5.0, 0.5, 0.0, 10.0)),
             ("gauss", 0.2 * n, 2.0, 1.5, oracle.gaussian_norm(2.0, 1.5, 0.0, 10.0)),
             ("exp", 0.5 * n, 3.0, oracle.exponential_norm(3.0, 0.0, 10.0))]
    assert hk.nll(three, store, ["x0"]) == pytest.approx(oracle.nll(x, comps), rel=1e-10, abs=1e-9)


def test_random_decays_and_fused_chains_vs_oracle(cuda, hk, oracle):
    """Randomised decays (2..8 daughters, random masses with thresholds of a
    few percent to wide open, mothers at rest or boosted) and fused chains
    (parent 2..6 daughters, sub-decay 2..4, random decaying daughter) against
    the oracle: weights bit-exact, momenta within 1e-12 E, and the fused
    chain's parent columns bit-identical to generate + decay_chain."""
    import os
    rs = np.random.default_rng(1717)
    for case in range(int(os.environ.get("HK_TEST_RANDOM_CASES", "16"))):
        n_d = int(rs.integers(2, 9))
        masses = tuple(float(v) for v in rs.uniform(0.0, 1.0, n_d) * rs.choice([0.0, 1.0], n_d, p=[0.15, 0.85]))
        M = sum(masses) + float(10 ** rs.uniform(-1.5, 0.7))
        if rs.random() < 0.4:
            p = tuple(float(v) for v in rs.normal(0, 2 * M, 3))
            mother = (math.sqrt(M * M + sum(c * c for c in p)), *p)
        else:
            mother = (M, 0.0, 0.0, 0.0)
        n = int(rs.integers(1, 3 * 4096 + 500))
        key = (int(rs.integers(0, 1 << 62)), int(rs.integers(0, 5)))
        spec = hk.DecaySpec(M, masses)
        blk = _arr(hk.phsp_generate(spec, hk.FourVector(*mother), n, hk.RngKey(*key)))
        ref = oracle.generate(masses, M, n, key[0], key[1], mother=mother, threads=4)
        assert_block_parity(blk, np.stack(list(ref.values())), n_d, f"random decay {case}")
        if n_d > 6:
            continue
        k = int(rs.integers(1, n_d + 1))
        if masses[k - 1] <= 0.0:
            continue
        n_s = int(rs.integers(2, 5))
        sub_m = tuple(float(v) for v in rs.uniform(0.0, masses[k - 1] / (n_s + 0.5), n_s))
        sub = hk.DecaySpec(masses[k - 1], sub_m)
        skey = (int(rs.integers(0, 1 << 62)), 1)
        # the frame mass sqrt(E^2 - p^2) of a daughter boosted to gamma_k loses
        # ~gamma_k^2 ulps to cancellation in the reference formula itself
        # (phasespace.py:259-262), so ulp-level differences in the parent's
        # momenta reach the sub-daughters as ~3e-16 gamma_k^2 E
        # (profiles/r02_chain_gamma.txt): the 1e-12 E budget holds to gamma_k ~ 50
        if float(np.max(ref[f"p{k}_e"])) > 40.0 * masses[k - 1]:
            continue
        fused = _arr(hk.phsp_generate_chain(spec, hk.FourVector(*mother), n, hk.RngKey(*key), k, sub,
                                            hk.RngKey(*skey)))
        two = _arr(hk.phsp_decay_chain(hk.phsp_generate(spec, hk.FourVector(*mother), n, hk.RngKey(*key)), k,
                                       sub, hk.RngKey(*skey)))
        _fused_vs_two_step(fused, two, k, n_s)
        cref = oracle.decay_chain(ref, k, sub_m, masses[k - 1], skey[0], skey[1], threads=4)
        assert_block_parity(fused, np.stack(list(cref.values())), n_d - 1 + n_s, f"random chain {case}")
