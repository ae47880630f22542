"""Largest four-momentum deviation from the oracle, |dc| / E_daughter, over
generated blocks: B0 -> J/psi K pi (1e6 rows at rest and boosted), 4- and
8-body decays -- the figure DESIGN.md quotes against the 1e-12 E budget."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1711_05683_b200 as hk  # noqa: E402
from oracle import oracle  # noqa: E402

cases = {
    "B0_rest": (5.27966, (3.0969, 0.493677, 0.13957039), None),
    "B0_boosted": (5.27966, (3.0969, 0.493677, 0.13957039), (0.7, -1.9, 3.3)),
    "4body": (2.0, (0.1, 0.2, 0.3, 0.4), None),
    "8body": (3.0, (0.1, 0.05, 0.2, 0.13, 0.3, 0.01, 0.25, 0.15), None),
}
out = {}
for name, (M, ms, p) in cases.items():
    mother = (M, 0.0, 0.0, 0.0) if p is None else (math.sqrt(M * M + sum(c * c for c in p)), *p)
    n = 1_000_000
    blk = hk.phsp_generate(hk.DecaySpec(M, ms), hk.FourVector(*mother), n, hk.RngKey(1, 1))
    ref = oracle.generate(ms, M, n, 1, 1, mother=mother, threads=16)
    worst, wbits = 0.0, True
    wbits = np.array_equal(np.asarray(blk.column("weight")), ref["weight"])
    for j in range(len(ms)):
        e = np.abs(ref[f"p{j + 1}_e"])
        for c in ("e", "px", "py", "pz"):
            d = np.abs(np.asarray(blk.column(f"p{j + 1}_{c}")) - ref[f"p{j + 1}_{c}"]) / np.maximum(e, 1e-300)
            worst = max(worst, float(np.nanmax(d)))
    out[name] = {"max_dc_over_E": worst, "weights_bit_exact": bool(wbits)}
print(json.dumps(out))
