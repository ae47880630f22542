"""Small driver for ncu captures: each hot kernel launched a few times.

    python tools/prof_kernels.py [--n 100000000]

Order of launches (for -k/-s/-c selection): k_generate x3, k_integrate x2,
k_generate_chain x2, k_nll x3, k_nll_many x2 (52 points each).
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_05683_b200 as hk  # noqa: E402
from paper_1711_05683_b200 import _lib  # noqa: E402
from paper_1711_05683_b200.fitting import lower_model  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--rng", default="reference")
    args = ap.parse_args()
    M, ms = 5.27966, (3.0969, 0.493677, 0.13957039)
    spec, mother = hk.DecaySpec(M, ms), hk.FourVector.at_rest(M)
    n = args.n
    for _ in range(3):
        blk = hk.phsp_generate(spec, mother, n, hk.RngKey(1, 1), rng=args.rng)
    torch.cuda.synchronize()
    del blk

    def m12(cols):
        e = cols["p1_e"] + cols["p2_e"]
        px = cols["p1_px"] + cols["p2_px"]
        py = cols["p1_py"] + cols["p2_py"]
        pz = cols["p1_pz"] + cols["p2_pz"]
        return (e * e - px * px - py * py - pz * pz,)

    for _ in range(2):
        r = hk.phsp_integrate(hk.identity(), spec, mother, n, hk.RngKey(1, 1), m12, rng=args.rng)
    sub = hk.DecaySpec(3.0969, (0.1056583755, 0.1056583755))
    for _ in range(2):
        ch = hk.phsp_generate_chain(spec, mother, n // 2, hk.RngKey(1, 1), 1, sub, hk.RngKey(2, 1), rng=args.rng)
    torch.cuda.synchronize()
    del ch
    rs = np.random.default_rng(7)
    x = np.clip(np.concatenate([rs.normal(5.0, 0.5, 4_000_000), rs.exponential(3.0, 6_000_000)]), 1e-3, 9.999)
    region = hk.BoundedRegion(((0.0, 10.0),))
    g = hk.shape_gaussian(hk.Parameter("mean", 5.0), hk.Parameter("sigma", 0.5))
    e = hk.shape_exponential(hk.Parameter("tau", 3.0))
    model = hk.add_pdfs([hk.Parameter("n_sig", 4e6), hk.Parameter("n_bkg", 6e6)],
                        [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])
    data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
    for _ in range(3):
        v = hk.nll(model, data, ["x0"])
    # the batched multi-point pass: 52 points (26 groups of 2) in one launch
    from paper_1711_05683_b200.fitting import nll_many
    base = model.param_set().values()
    names = model.param_set().names
    pts = [tuple(b * (1.0 + 1e-4 * (k + 1)) if nm in ("mean", "sigma", "tau") else b for nm, b in zip(names, base))
           for k in range(52)]
    for _ in range(2):
        nll_many(model, data, ["x0"], pts)
    torch.cuda.synchronize()
    print(f"ok <m12^2>={r.value:.12g} nll={v:.12g}")


if __name__ == "__main__":
    main()
