"""Generic extended models for the FCN parity tests (no reference import, so
the GPU tests can build them too): the same builder runs against the
reference package in make_golden.py and against the drop-in package in
tests/test_fcn_generic_gpu.py.

* g1 -- Breit-Wigner + linear polynomial (closures, closed-form norms), 1-D;
* g2 -- observable arity 2: Gaussian(x) * exponential(y) through
  compose/coordinate/combine, plus a 2-D closure background;
* g6 -- six components (four Gaussians, an exponential, a flat closure);
* g12 -- twelve components (ten Gaussians, an exponential, a flat closure).
"""

from __future__ import annotations

import math


def _bw_norm(m0, g, lo, hi):
    h = 0.5 * g
    return (math.atan((hi - m0) / h) - math.atan((lo - m0) / h)) / h


def generic_models(hk_mod, np_mod, values):
    """Model builders shared with the device tests (tests/test_fcn_generic_gpu.py
    builds the same models against the drop-in package).  values: name -> float."""
    P = hk_mod.Parameter
    v = values
    out = {}
    # G1: Breit-Wigner + linear polynomial on [0.6, 1.2] (closures + closed-form norms)
    lo, hi = 0.6, 1.2
    m0, g = P("m0", v["m0"]), P("g", v["g"])
    c0, c1 = P("c0", v["c0"]), P("c1", v["c1"])
    bw = hk_mod.wrap_closure(lambda x, p: 1.0 / ((x[0] - p["m0"].value) ** 2 + (0.5 * p["g"].value) ** 2),
                             [m0, g])
    poly = hk_mod.wrap_closure(lambda x, p: p["c0"].value + p["c1"].value * x[0], [c0, c1])
    reg1 = hk_mod.BoundedRegion(((lo, hi),))
    out["g1"] = hk_mod.add_pdfs(
        [P("n_bw", v["n_bw"]), P("n_poly", v["n_poly"])],
        [hk_mod.make_pdf(bw, lambda r: _bw_norm(m0.value, g.value, lo, hi), reg1),
         hk_mod.make_pdf(poly, lambda r: c0.value * (hi - lo) + 0.5 * c1.value * (hi * hi - lo * lo), reg1)])
    # G2: 2-D, Gaussian(x) * exponential(y) through compose/coordinate and a
    # 2-D closure background (observable arity 2)
    lo2, hi2 = 0.0, 10.0
    mx, sx, ty = P("mx", v["mx"]), P("sx", v["sx"]), P("ty", v["ty"])
    a2 = P("a2", v["a2"])
    sig = hk_mod.combine("*", hk_mod.compose(hk_mod.shape_gaussian(mx, sx), [hk_mod.coordinate(0, 2)]),
                         hk_mod.compose(hk_mod.shape_exponential(ty), [hk_mod.coordinate(1, 2)]))
    bkg = hk_mod.wrap_closure(lambda x, p: 1.0 + p["a2"].value * x[0] * x[1], [a2], arity=2)
    reg2 = hk_mod.BoundedRegion(((lo2, hi2), (lo2, hi2)))

    def sig_norm(r):
        s2 = sx.value * math.sqrt(2.0)
        gx = 0.5 * (math.erf((hi2 - mx.value) / s2) - math.erf((lo2 - mx.value) / s2))
        ey = ty.value * (math.exp(-lo2 / ty.value) - math.exp(-hi2 / ty.value))
        return gx * ey

    out["g2"] = hk_mod.add_pdfs(
        [P("n_sig2", v["n_sig2"]), P("n_bkg2", v["n_bkg2"])],
        [hk_mod.make_pdf(sig, sig_norm, reg2),
         hk_mod.make_pdf(bkg, lambda r: (hi2 - lo2) ** 2 + a2.value * ((hi2 ** 2 - lo2 ** 2) / 2.0) ** 2, reg2)])
    # G6: six components (four Gaussians, an exponential, a flat closure):
    # more than the old 4-component device limit
    comps, ys = [], []
    reg6 = hk_mod.BoundedRegion(((0.0, 10.0),))
    for i, (mu, s) in enumerate(((2.0, 0.3), (4.0, 0.5), (6.0, 0.4), (8.0, 0.6))):
        gs = hk_mod.shape_gaussian(P(f"mu{i}", v.get(f"mu{i}", mu)), P(f"s{i}", v.get(f"s{i}", s)))
        comps.append(hk_mod.make_pdf(gs, hk_mod.gaussian_norm(gs), reg6))
        ys.append(P(f"y{i}", v[f"y{i}"]))
    ex = hk_mod.shape_exponential(P("tau6", v["tau6"]))
    comps.append(hk_mod.make_pdf(ex, hk_mod.exponential_norm(ex), reg6))
    ys.append(P("y4", v["y4"]))
    flat = hk_mod.wrap_closure(lambda x, p: np_mod.ones_like(x[0]) * 1.0, [])
    comps.append(hk_mod.make_pdf(flat, lambda r: 10.0, reg6))
    ys.append(P("y5", v["y5"]))
    out["g6"] = hk_mod.add_pdfs(ys, comps)
    # G12: twelve components (ten Gaussians, an exponential, a flat closure):
    # above the device's pinned-slot limit (HK_MAX_COMPONENTS = 8), so the
    # ratio sums and sWeights run in passes
    comps, ys = [], []
    for i in range(10):
        mu, s = G12_MEANS[i], 0.2 + 0.03 * i
        gs = hk_mod.shape_gaussian(P(f"m12_{i}", v.get(f"m12_{i}", mu)), P(f"s12_{i}", v.get(f"s12_{i}", s)))
        comps.append(hk_mod.make_pdf(gs, hk_mod.gaussian_norm(gs), reg6))
        ys.append(P(f"z{i}", v.get(f"z{i}", 800.0 + 40.0 * i)))
    ex12 = hk_mod.shape_exponential(P("tau12", v.get("tau12", 2.5)))
    comps.append(hk_mod.make_pdf(ex12, hk_mod.exponential_norm(ex12), reg6))
    ys.append(P("z10", v.get("z10", 2000.0)))
    flat12 = hk_mod.wrap_closure(lambda x, p: np_mod.ones_like(x[0]) * 1.0, [])
    comps.append(hk_mod.make_pdf(flat12, lambda r: 10.0, reg6))
    ys.append(P("z11", v.get("z11", 1200.0)))
    out["g12"] = hk_mod.add_pdfs(ys, comps)
    return out


G12_MEANS = [0.5 + 0.95 * i for i in range(10)]


GENERIC_POINTS = [
    {"m0": 0.8955, "g": 0.0473, "c0": 1.0, "c1": 0.5, "n_bw": 3000.0, "n_poly": 9000.0,
     "mx": 5.0, "sx": 0.8, "ty": 2.5, "a2": 0.05, "n_sig2": 4000.0, "n_bkg2": 8000.0,
     "y0": 1500.0, "y1": 2500.0, "y2": 2000.0, "y3": 1800.0, "y4": 3000.0, "y5": 1500.0, "tau6": 3.0},
    {"m0": 0.90, "g": 0.052, "c0": 1.1, "c1": 0.3, "n_bw": 3100.0, "n_poly": 8800.0,
     "mx": 5.2, "sx": 0.7, "ty": 2.2, "a2": 0.08, "n_sig2": 4200.0, "n_bkg2": 7700.0,
     "y0": 1400.0, "y1": 2600.0, "y2": 1900.0, "y3": 1900.0, "y4": 3100.0, "y5": 1400.0, "tau6": 3.3,
     "mu1": 4.1, "s2": 0.45, "z3": 950.0, "m12_4": 4.3, "s12_7": 0.35, "tau12": 2.8},
]
