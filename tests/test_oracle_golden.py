"""Pin the CPU oracle (oracle/) against the golden vectors frozen from the
reference implementation itself (tests/golden/make_golden.py).  Bit-exact."""

from __future__ import annotations

import numpy as np

from tests.common import B0_DAUGHTERS, B0_MASS, M_JPSI, M_MU, m12sq_builder


def test_rng_known_answers(golden, oracle):
    arrays, _ = golden
    ctr = arrays["rng_counters"]
    for i, k in enumerate(arrays["rng_keys"]):
        seed, stream, counter = (int(v) for v in k)
        assert oracle.base(seed, stream) == int(arrays["rng_base"][i])
        assert np.array_equal(oracle.raw64(seed, stream, counter, ctr), arrays["rng_raw64"][i])
        assert np.array_equal(oracle.uniform(seed, stream, counter, ctr), arrays["rng_uniform"][i])
    u = oracle.uniform(7, 1, 0, np.arange(4096, dtype=np.uint64))
    assert np.array_equal(u, arrays["rng_uniform_seq_7_1"])


def test_survey_appendix_a_values(oracle):
    # SURVEY.md Appendix A (computed with the reference)
    assert oracle.base(1, 1) == 0xF2C5EBC6A20B2953
    assert oracle.base(0, 0) == 0
    assert [hex(int(v)) for v in oracle.raw64(0, 0, 0, np.arange(4, dtype=np.uint64))] == \
        ["0x0", "0xe220a8397b1dcdaf", "0x6e789e6aa1b965f4", "0x6c45d188009454f"]
    u = oracle.uniform(7, 1, 0, np.arange(5, dtype=np.uint64))
    assert u.tolist() == [0.6555391811506788, 0.9725041819223492, 0.35404652295342276,
                          0.11243334523693238, 0.4496469353302388]


def test_generated_blocks_bit_exact(golden, oracle):
    arrays, scalars = golden
    for b in scalars["gen_blocks"]:
        cols = oracle.generate(b["masses"], b["M"], b["rows"], *b["key"], mother=b["mother"], threads=2)
        got = np.stack(list(cols.values()))
        assert np.array_equal(got, arrays["gen_" + b["name"]], equal_nan=True), b["name"]


def test_c1_full_block_checksums(golden, oracle):
    _, scalars = golden
    c1 = oracle.generate(B0_DAUGHTERS, B0_MASS, 100_000, 1, 1, threads=4)
    assert [float(np.sum(v)) for v in c1.values()] == scalars["c1"]["colsum"]
    w = c1["weight"]
    assert float(np.sum(w)) == scalars["c1"]["wsum"]
    assert float(np.var(w)) == scalars["c1"]["wvar"]
    assert float(np.max(w)) == scalars["c1"]["wmax"]
    v, e, _ = oracle.average(w, oracle.pair_mass2(c1, 1, 2))
    assert [v, e] == scalars["c1"]["avg_m12sq"]
    mbw, gbw = scalars["c1"]["avg_bw_kstar"][2:]
    v, e, _ = oracle.average(w, oracle.breit_wigner(oracle.pair_mass2(c1, 2, 3), mbw, gbw))
    assert [v, e] == scalars["c1"]["avg_bw_kstar"][:2]
    # constant integrand: value 1, error 0 (test_phasespace.py:203-209)
    v, e, _ = oracle.average(w, np.ones_like(w))
    assert [v, e] == scalars["c1"]["avg_one"]


def test_unweight_accept_mask(golden, oracle):
    arrays, scalars = golden
    c1 = oracle.generate(B0_DAUGHTERS, B0_MASS, 100_000, 1, 1, threads=4)
    acc = oracle.unweight_accept(c1["weight"], scalars["kat"]["max_weight_b0"], 1, 4)
    assert np.array_equal(np.packbits(acc), arrays["c1_unweight_accept_bits"])
    assert int(acc.sum()) == scalars["c1"]["unweight_count"]


def test_decay_chain_bit_exact(golden, oracle):
    arrays, scalars = golden
    small = oracle.generate(B0_DAUGHTERS, B0_MASS, 256, 1, 1)
    ch = oracle.decay_chain(small, 1, (M_MU, M_MU), M_JPSI, 2, 1)
    assert np.array_equal(np.stack(list(ch.values())), arrays["chain_c3"])
    par = oracle.generate((0.3, 1.2), 3.0, 128, 21, 1)
    ch = oracle.decay_chain(par, 2, (0.2, 0.3, 0.4), 1.2, 22, 1)
    assert np.array_equal(np.stack(list(ch.values())), arrays["chain_three_sub"])
    par = oracle.generate(B0_DAUGHTERS, B0_MASS, 64, 1, 1, 5000)
    ch = oracle.decay_chain(par, 1, (M_MU, M_MU), M_JPSI, 2, 1, 5000)
    assert np.array_equal(np.stack(list(ch.values())), arrays["chain_c3_window_5000"])
    c1 = oracle.generate(B0_DAUGHTERS, B0_MASS, 100_000, 1, 1, threads=4)
    c3 = oracle.decay_chain(c1, 1, (M_MU, M_MU), M_JPSI, 2, 1, threads=4)
    assert [float(np.sum(v)) for v in c3.values()] == scalars["c3"]["colsum"]


def test_nll_values(golden, oracle):
    arrays, scalars = golden
    x = arrays["nll_x"]
    for pt, val in zip(scalars["nll"]["points"], scalars["nll"]["values"]):
        comps = oracle.gauss_exp_components(pt["mean"], pt["sigma"], pt["tau"], pt["n_sig"], pt["n_bkg"])
        assert oracle.nll(x, comps) == val
    single = oracle.nll(np.array([0.0]), [("gauss", 1.0, 0.0, 1.0, oracle.gaussian_norm(0.0, 1.0, -10.0, 10.0))])
    assert single == scalars["nll"]["single_event"] == 1.9189385332046727


def test_nll_first_bad_message(golden, oracle):
    arrays, scalars = golden
    x = arrays["nll_x"].copy()
    for j in (2500, 700, 2000):
        x[j] = np.nan
    comps = oracle.gauss_exp_components(5.0, 0.5, 3.0, 4000.0, 6000.0)
    try:
        oracle.nll(x, comps)
    except ValueError as exc:
        assert str(exc) == scalars["nll"]["bad_message"]
    else:
        raise AssertionError("no error")


def test_window_property(oracle):
    """Rows [s, s+n) regenerated with counter offset s equal rows s.. of a full
    run -- the property the large-N GPU checks rely on."""
    full = oracle.generate(B0_DAUGHTERS, B0_MASS, 20_000, 3, 1, threads=4)
    win = oracle.generate(B0_DAUGHTERS, B0_MASS, 1000, 3, 1, counter=12_345)
    via_begin = oracle.generate(B0_DAUGHTERS, B0_MASS, 1000, 3, 1, ev_begin=12_345)
    for name in full:
        assert np.array_equal(win[name], full[name][12_345:13_345])
        assert np.array_equal(via_begin[name], full[name][12_345:13_345])


def test_average_builder_matches_oracle_pair_mass(oracle):
    c = oracle.generate(B0_DAUGHTERS, B0_MASS, 5000, 4, 1)
    assert np.array_equal(m12sq_builder(c)[0], oracle.pair_mass2(c, 1, 2))


# Random123 known-answer vectors for philox4x32 with R = 10 rounds (Random123
# distribution, examples/kat_vectors: ctr[4] key[2] -> out[4]).  They pin the
# oracle's Philox restatement, which in turn is the checker for the device's
# production stream (tests/test_parity_pins_gpu.py).
PHILOX_KAT = [
    ((0x00000000, 0x00000000, 0x00000000, 0x00000000), (0x00000000, 0x00000000),
     (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF), (0xFFFFFFFF, 0xFFFFFFFF),
     (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def test_oracle_philox_known_answers(oracle):
    got = oracle.philox4x32_10([c for c, _, _ in PHILOX_KAT], [k for _, k, _ in PHILOX_KAT])
    assert got.tolist() == [list(o) for _, _, o in PHILOX_KAT]


def test_oracle_philox_stream_mapping(oracle):
    """The production stream's draw layout (hk_device.cuh draw_bits) from the
    raw blocks: event e's raw64 in Philox mode is words (0, 1) of block
    (e lo, e hi, 0, "hkph") under key base(seed, stream)."""
    seed, stream, kc = 7, 1, 5
    ctr = np.array([0, 1, 2**32 + 3, 2**63 + 11], dtype=np.uint64)
    b = oracle.base(seed, stream)
    ev = ctr + np.uint64(kc)
    blocks = oracle.philox4x32_10(
        np.stack([ev & np.uint64(0xFFFFFFFF), ev >> np.uint64(32), np.zeros_like(ev),
                  np.full_like(ev, 0x686B7068)], axis=1),
        np.tile(np.array([b & 0xFFFFFFFF, b >> 32], dtype=np.uint64), (len(ev), 1)))
    want = (blocks[:, 0].astype(np.uint64) << np.uint64(32)) | blocks[:, 1].astype(np.uint64)
    assert np.array_equal(oracle.philox_raw64(seed, stream, kc, ctr), want)
    # a Philox-mode generation is a valid phase-space sample: conservation at rest
    cols = oracle.generate(B0_DAUGHTERS, B0_MASS, 2000, 1, 1, rng="philox")
    e = sum(cols[f"p{j}_e"] for j in (1, 2, 3))
    px = sum(cols[f"p{j}_px"] for j in (1, 2, 3))
    assert np.allclose(e, B0_MASS, rtol=1e-13) and np.allclose(px, 0.0, atol=1e-13)
    ref = oracle.generate(B0_DAUGHTERS, B0_MASS, 2000, 1, 1)
    assert not np.array_equal(cols["weight"], ref["weight"])
