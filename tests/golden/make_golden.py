"""Freeze golden vectors from the REFERENCE implementation (run in the build
container only -- /root/reference does not exist on the GPU box).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/golden.npz (arrays) and tests/golden/golden.json
(scalars, repr-exact).  The oracle (oracle/) is pinned against these in
tests/test_oracle_golden.py; the CUDA path is then checked against the oracle
and, at fixture sizes, against these vectors directly.

Every array here is produced by calling the reference's public API
(`hepkit`, /root/reference/pkg/src) -- nothing is restated.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path[:0] = [REF_SRC, REF_TESTS]
sys.dont_write_bytecode = True

import hepkit as hk  # noqa: E402
from hepkit.rng import raw64, uniform_array, _base  # noqa: E402
from hepkit.fitting import generate_model_sample  # noqa: E402
import toymodel  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from generic_models import G12_MEANS, GENERIC_POINTS, generic_models  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# pinned decay inputs (GeV)
M_B0, M_JPSI, M_K, M_PI, M_MU = 5.27966, 3.0969, 0.493677, 0.13957039, 0.1056583755

# (name, mother mass, daughters, mother 4-vector or None for at-rest, key, rows)
BLOCKS = [
    ("c1_b0_jpsikpi", M_B0, (M_JPSI, M_K, M_PI), None, (1, 1, 0), 256),
    ("c1_window_99000", M_B0, (M_JPSI, M_K, M_PI), None, (1, 1, 99_000), 128),
    ("two_body", 1.0, (0.3, 0.3), None, (1, 1, 0), 64),
    ("three_body_light", 1.0, (0.1, 0.1, 0.1), None, (7, 1, 0), 128),
    ("four_body", 2.0, (0.3, 0.1, 0.4, 0.2), None, (3, 1, 0), 128),
    ("five_body", 3.0, (0.1, 0.2, 0.3, 0.4, 0.5), None, (5, 1, 0), 64),
    ("eight_body", 2.0, (0.1,) * 8, None, (8, 1, 0), 32),
    ("massless_three", 1.0, (0.0, 0.0, 0.0), None, (9, 1, 0), 64),
    ("big_counter", 1.5, (0.3, 0.1, 0.4), None, (4, 1, (1 << 62) + 12345), 64),
    ("neg_seed", 1.5, (0.3, 0.1, 0.4), None, (-17, 3, 0), 32),
]


def moving_mother(M: float, p: tuple[float, float, float]) -> "hk.FourVector":
    e = math.sqrt(M * M + p[0] * p[0] + p[1] * p[1] + p[2] * p[2])
    return hk.FourVector(e, *p)


MOVING = [
    ("moving_two_body_z", 1.0, (0.2, 0.2), hk.FourVector(1.0 / math.sqrt(1 - 0.64), 0.0, 0.0,
                                                         0.8 / math.sqrt(1 - 0.64)), (5, 1, 0), 64),
    ("moving_b0", M_B0, (M_JPSI, M_K, M_PI), moving_mother(M_B0, (1.3, -0.7, 4.1)), (11, 1, 0), 64),
]


def block_array(block) -> np.ndarray:
    return np.stack([np.asarray(block.column(n)) for n in block.schema.names], axis=0)


def m12sq_builder(cols):
    e = cols["p1_e"] + cols["p2_e"]
    px = cols["p1_px"] + cols["p2_px"]
    py = cols["p1_py"] + cols["p2_py"]
    pz = cols["p1_pz"] + cols["p2_pz"]
    return (e * e - px * px - py * py - pz * pz,)



def _x(store) -> np.ndarray:
    return np.asarray(store.column("x0"))


def add_c4(arrays, scalars) -> None:
    """The bench's FCN data set (config C4): build_model(scale=200),
    generate_model_sample(RngKey(7, 2), poisson=False) -> 1e7 events.  Only
    fingerprints are frozen (the full column is 80 MB): head, sum, a SHA-256
    of the bytes, a strided sample, and nll at two points."""
    import hashlib
    from hepkit.fitting import _poisson_count

    model = toymodel.build_model(scale=200)
    data = generate_model_sample(model, hk.RngKey(7, 2), poisson=False, workers=8)
    x = _x(data)
    idx = np.arange(0, len(x), 99_991, dtype=np.int64)
    arrays["c4_strided_idx"] = idx
    arrays["c4_strided_x"] = x[idx]
    c4 = {"n": len(x), "head": x[:8].tolist(), "xsum": float(np.sum(x)),
          "sha256": hashlib.sha256(x.tobytes()).hexdigest(),
          "nll_truth": hk.nll(model, data, ["x0"], workers=8)}
    ps = model.param_set()
    ps["mean"].set(4.9)
    ps["sigma"].set(0.55)
    ps["tau"].set(2.8)
    c4["nll_alt"] = hk.nll(model, data, ["x0"], workers=8)
    c4["alt_point"] = {"mean": 4.9, "sigma": 0.55, "tau": 2.8}
    # Poisson component counts (fitting.py:519-523) for the same key and yields
    c4["poisson_counts"] = [_poisson_count(y.value, hk.RngKey(7, 2), c)
                            for c, (y, _) in enumerate(toymodel.build_model(scale=200).components)]
    # a poisson=True toy at scale 0.2: count and bits
    small = generate_model_sample(toymodel.build_model(scale=0.2), hk.RngKey(7, 2), poisson=True)
    xs = _x(small)
    arrays["c4_poisson_small_x"] = xs
    c4["poisson_small_n"] = len(xs)
    scalars["c4"] = c4


def add_yields_splot(arrays, scalars, data) -> None:
    """Reference yield-stationarity sums and sPlot outputs on the scale-0.2 toy
    data (golden nll_x): at the truth, at an off-optimum point, and -- for
    sPlot -- at the parameters of the reference's own fit."""
    from hepkit.fitting import _yield_stationarity
    from hepkit.splot import splot_matrix, splot_weights

    out = {"points": []}
    for pt in ({}, {"mean": 5.1, "sigma": 0.45, "tau": 3.3, "n_sig": 3900.0, "n_bkg": 6200.0}):
        m = toymodel.build_model(scale=0.2, **pt)
        g, A = _yield_stationarity(m, data, ["x0"], 1)
        out["points"].append({"values": {p.name: p.value for p in m.param_set()},
                              "g": g.tolist(), "A": A.tolist()})
    m = toymodel.build_model(scale=0.2)
    res = hk.fit(m, data, ["x0"])
    V = splot_matrix(m, data, ["x0"])
    sw = splot_weights(m, data, ["x0"], V)
    out["fit_values"] = {p.name: p.value for p in m.param_set()}
    out["fit_status"] = res.status.value
    out["V"] = V.tolist()
    arrays["splot_sw"] = np.stack([np.asarray(sw.column(n)) for n in sw.schema.names])
    scalars["yields_splot"] = out


def add_generic_models(arrays, scalars) -> None:
    rs = np.random.default_rng(20251018)
    n = 3 * 4096 + 17
    # G1 data on [0.6, 1.2]: a Cauchy peak + uniform
    xb = rs.standard_cauchy(n) * 0.0237 + 0.8955
    xb = np.where((xb > 0.6) & (xb < 1.2), xb, rs.uniform(0.6, 1.2, n))
    arrays["g1_x"] = xb
    # G2 data on [0, 10]^2
    arrays["g2_x"] = np.clip(rs.normal(5.0, 0.8, n), 0.01, 9.99)
    arrays["g2_y"] = np.clip(rs.exponential(2.5, n), 0.01, 9.99)
    # G6 data on [0, 10]
    arrays["g6_x"] = np.clip(np.concatenate([rs.normal(mu, s, n // 6) for mu, s in
                                             ((2.0, 0.3), (4.0, 0.5), (6.0, 0.4), (8.0, 0.6))]
                                            + [rs.exponential(3.0, n // 6), rs.uniform(0, 10, n - 5 * (n // 6))]),
                             0.01, 9.99)
    s1 = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [arrays["g1_x"]])
    s2 = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0", "x1"), [arrays["g2_x"], arrays["g2_y"]])
    s6 = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [arrays["g6_x"]])
    # G12 data on [0, 10] (its own generator: the arrays above stay as they were)
    r12 = np.random.default_rng(20261019)
    n12 = 2 * 4096 + 29
    arrays["g12_x"] = np.clip(np.concatenate([r12.normal(mu, 0.3, n12 // 12) for mu in G12_MEANS]
                                             + [r12.exponential(2.5, n12 // 12),
                                                r12.uniform(0, 10, n12 - 11 * (n12 // 12))]), 0.01, 9.99)
    s12 = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [arrays["g12_x"]])
    out = {"points": GENERIC_POINTS, "g1": [], "g2": [], "g6": [], "g6_yields": [], "g12": [], "g12_yields": []}
    from hepkit.fitting import _yield_stationarity
    for pt in GENERIC_POINTS:
        ms = generic_models(hk, np, pt)
        out["g1"].append(hk.nll(ms["g1"], s1, ["x0"]))
        out["g2"].append(hk.nll(ms["g2"], s2, ["x0", "x1"]))
        out["g6"].append(hk.nll(ms["g6"], s6, ["x0"]))
        g, A = _yield_stationarity(ms["g6"], s6, ["x0"], 1)
        out["g6_yields"].append({"g": g.tolist(), "A": A.tolist()})
        out["g12"].append(hk.nll(ms["g12"], s12, ["x0"]))
        g, A = _yield_stationarity(ms["g12"], s12, ["x0"], 1)
        out["g12_yields"].append({"g": g.tolist(), "A": A.tolist()})
    # sWeights of G12 at the first point with V = A^-1 (splot_weights takes any V)
    m12 = generic_models(hk, np, GENERIC_POINTS[0])["g12"]
    V12 = np.linalg.inv(np.asarray(out["g12_yields"][0]["A"]))
    arrays["g12_V"] = V12
    sw = hk.splot_weights(m12, s12, ["x0"], V12)
    arrays["g12_sw"] = np.stack([np.asarray(sw.column(n)) for n in sw.schema.names])
    scalars["generic"] = out

def main() -> None:
    arrays: dict[str, np.ndarray] = {}
    scalars: dict[str, object] = {}

    # ---- RNG known answers (rng.py:98-130) --------------------------------
    keys = [(0, 0, 0), (7, 1, 0), (1, 1, 0), (2, 1, 0), (123, 0, 42),
            ((1 << 64) - 1, 5, 1 << 63), (-1, 3, 7), (2024, 0, 0)]
    counters = np.array([0, 1, 2, 3, 1000, 1 << 40, (1 << 64) - 1, 987654321], dtype=np.uint64)
    arrays["rng_keys"] = np.array([[k[0] % (1 << 64), k[1] % (1 << 64), k[2] % (1 << 64)]
                                   for k in keys], dtype=np.uint64)
    arrays["rng_counters"] = counters
    arrays["rng_base"] = np.array([_base(k[0], k[1]) for k in keys], dtype=np.uint64)
    arrays["rng_raw64"] = np.stack([raw64(hk.RngKey(*k), counters) for k in keys])
    arrays["rng_uniform"] = np.stack([uniform_array(hk.RngKey(*k), counters) for k in keys])
    arrays["rng_uniform_seq_7_1"] = uniform_array(hk.RngKey(7, 1), np.arange(4096, dtype=np.uint64))

    # ---- generated blocks (phasespace.py:162-188) -------------------------
    meta = []
    for name, M, ms, mother, key, rows in BLOCKS + MOVING:
        mother = mother if mother is not None else hk.FourVector.at_rest(M)
        spec = hk.DecaySpec(M, ms)
        blk = hk.phsp_generate(spec, mother, rows, hk.RngKey(*key))
        arrays[f"gen_{name}"] = block_array(blk)
        meta.append({"name": name, "M": M, "masses": list(ms),
                     "mother": [mother.e, mother.px, mother.py, mother.pz],
                     "key": [int(key[0]), int(key[1]), int(key[2])], "rows": rows,
                     "max_weight": hk.phsp_max_weight(spec)})
    scalars["gen_blocks"] = meta

    # ---- C1 full block: column checksums + weight/average reductions ------
    spec_b0 = hk.DecaySpec(M_B0, (M_JPSI, M_K, M_PI))
    c1 = hk.phsp_generate(spec_b0, hk.FourVector.at_rest(M_B0), 100_000, hk.RngKey(1, 1), workers=8)
    w = np.asarray(c1.column("weight"))
    scalars["c1"] = {
        "n": 100_000,
        "colsum": [float(np.sum(np.asarray(c1.column(n)))) for n in c1.schema.names],
        "wsum": float(np.sum(w)), "wmean": float(np.mean(w)), "wvar": float(np.var(w)),
        "wmax": float(np.max(w)), "wmin": float(np.min(w)),
    }
    r = hk.phsp_average(hk.identity(), c1, m12sq_builder)
    scalars["c1"]["avg_m12sq"] = [r.value, r.error]
    one = hk.wrap_closure(lambda x, p: np.ones_like(np.asarray(x[0], dtype=float)))
    r1 = hk.phsp_average(one, c1, lambda cols: (cols["weight"] * 0 + 1,))
    scalars["c1"]["avg_one"] = [r1.value, r1.error]
    # K*(892) Breit-Wigner on m^2(K pi) = daughters 2,3 (SURVEY 8(d) C5 secondary f)
    Mbw, Gbw = 0.89555, 0.0473
    bw = hk.wrap_closure(lambda x, p: 1.0 / ((x[0] - Mbw * Mbw) ** 2 + (Mbw * Mbw) * (Gbw * Gbw)))

    def m23sq(cols):
        e = cols["p2_e"] + cols["p3_e"]
        px = cols["p2_px"] + cols["p3_px"]
        py = cols["p2_py"] + cols["p3_py"]
        pz = cols["p2_pz"] + cols["p3_pz"]
        return (e * e - px * px - py * py - pz * pz,)

    rb = hk.phsp_average(bw, c1, m23sq)
    scalars["c1"]["avg_bw_kstar"] = [rb.value, rb.error, Mbw, Gbw]

    # unweighting (phasespace.py:206-234): accept mask of C1 at max weight
    wmax = hk.phsp_max_weight(spec_b0)
    acc = uniform_array(hk.RngKey(1, 4), np.arange(100_000, dtype=np.uint64)) * wmax < w
    arrays["c1_unweight_accept_bits"] = np.packbits(acc)
    uw = hk.phsp_unweight(c1, wmax, hk.RngKey(1, 4))
    scalars["c1"]["unweight_count"] = len(uw)
    scalars["c1"]["unweight_colsum"] = [float(np.sum(np.asarray(uw.column(n))))
                                        for n in uw.schema.names]

    # ---- C3 chain (phasespace.py:237-288) --------------------------------
    sub_jpsi = hk.DecaySpec(M_JPSI, (M_MU, M_MU))
    c3_small = hk.phsp_decay_chain(
        hk.phsp_generate(spec_b0, hk.FourVector.at_rest(M_B0), 256, hk.RngKey(1, 1)),
        1, sub_jpsi, hk.RngKey(2, 1))
    arrays["chain_c3"] = block_array(c3_small)
    c3 = hk.phsp_decay_chain(c1, 1, sub_jpsi, hk.RngKey(2, 1), workers=8)
    scalars["c3"] = {"n": 100_000,
                     "colsum": [float(np.sum(np.asarray(c3.column(n)))) for n in c3.schema.names]}
    # chain of a 3-body sub-decay on daughter 2 of a 2-body parent
    par = hk.phsp_generate(hk.DecaySpec(3.0, (0.3, 1.2)), hk.FourVector.at_rest(3.0), 128,
                           hk.RngKey(21, 1))
    arrays["chain_three_sub"] = block_array(
        hk.phsp_decay_chain(par, 2, hk.DecaySpec(1.2, (0.2, 0.3, 0.4)), hk.RngKey(22, 1)))
    # chain with a key counter offset, on a window of the parent
    par_w = hk.phsp_generate(spec_b0, hk.FourVector.at_rest(M_B0), 64, hk.RngKey(1, 1, 5000))
    arrays["chain_c3_window_5000"] = block_array(
        hk.phsp_decay_chain(par_w, 1, sub_jpsi, hk.RngKey(2, 1, 5000)))

    # ---- FCN / NLL (fitting.py:175-210) -----------------------------------
    model = toymodel.build_model(scale=0.2)
    data = generate_model_sample(model, hk.RngKey(7, 2), poisson=False)
    x = np.asarray(data.column("x0"))
    arrays["nll_x"] = x
    points = [
        {"mean": 5.0, "sigma": 0.5, "tau": 3.0, "n_sig": 4000.0, "n_bkg": 6000.0},
        {"mean": 4.9, "sigma": 0.55, "tau": 2.8, "n_sig": 4000.0, "n_bkg": 6000.0},
        {"mean": 5.3, "sigma": 0.41, "tau": 7.5, "n_sig": 3500.5, "n_bkg": 7000.25},
        {"mean": 0.5, "sigma": 2.0, "tau": -4.0, "n_sig": 1.0, "n_bkg": 10.0},
    ]
    nll_vals = []
    for pt in points:
        m = toymodel.build_model(scale=0.2)
        ps = m.param_set()
        for k, v in pt.items():
            ps[k].set(v) if k != "tau" or v > 1e-4 else None
        if pt["tau"] <= 1e-4:  # tau lower bound 1e-4 in toymodel: rebuild unbounded
            tau = hk.Parameter("tau", pt["tau"])
            g = hk.shape_gaussian(hk.Parameter("mean", pt["mean"]), hk.Parameter("sigma", pt["sigma"]))
            e = hk.shape_exponential(tau)
            reg = hk.BoundedRegion((toymodel.RANGE,))
            m = hk.add_pdfs([hk.Parameter("n_sig", pt["n_sig"]), hk.Parameter("n_bkg", pt["n_bkg"])],
                            [hk.make_pdf(g, hk.gaussian_norm(g), reg),
                             hk.make_pdf(e, hk.exponential_norm(e), reg)])
        nll_vals.append(hk.nll(m, data, ["x0"]))
    scalars["nll"] = {"points": points, "values": nll_vals, "n": len(x),
                      "xsum": float(np.sum(x))}
    # single-event definitional value (test_fitting.py:90-98)
    g = hk.shape_gaussian(hk.Parameter("mean", 0.0), hk.Parameter("sigma", 1.0))
    m1 = hk.add_pdfs([hk.Parameter("n", 1.0)],
                     [hk.make_pdf(g, hk.gaussian_norm(g), hk.BoundedRegion(((-10.0, 10.0),)))])
    one_store = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [np.array([0.0])])
    scalars["nll"]["single_event"] = hk.nll(m1, one_store, ["x0"])
    # first-bad-event contract: NaNs planted at 2500, 700, 2000 -> event 700
    xb = x.copy()
    for j in (2500, 700, 2000):
        xb[j] = np.nan
    bad_store = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [xb])
    try:
        hk.nll(toymodel.build_model(scale=0.2), bad_store, ["x0"])
        scalars["nll"]["bad_message"] = None
    except ValueError as exc:
        scalars["nll"]["bad_message"] = str(exc)

    # ---- host scalar KATs --------------------------------------------------
    scalars["kat"] = {
        "breakup_2_05_03": hk.breakup_momentum(2.0, 0.5, 0.3),
        "max_weight_b0": hk.phsp_max_weight(spec_b0),
    }

    # ---- C4 data set pins (cli.py:321-323) ---------
    add_c4(arrays, scalars)
    # ---- yield stationarity + sPlot (fitting.py:401-434, splot.py:45-117) --
    add_yields_splot(arrays, scalars, data)
    # ---- FCN of generic shapes / observable arity 2 (fitting.py:160-199) ---
    add_generic_models(arrays, scalars)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(scalars, fh, indent=1, default=float)
    sizes = {k: v.nbytes for k, v in arrays.items()}
    print("wrote", len(arrays), "arrays,", sum(sizes.values()), "bytes raw")


if __name__ == "__main__":
    main()
