"""Fused-chain momentum error against the oracle as a function of the
decaying daughter's largest boost (gamma_k = E_k / m_k): random decays as in
tests/test_gpu_parity.py::test_random_decays_and_fused_chains_vs_oracle."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1711_05683_b200 as hk  # noqa: E402
from oracle import oracle  # noqa: E402


def arr(b):
    return np.stack([np.asarray(b.column(c)) for c in b.schema.names])


rs = np.random.default_rng(1717)
rows = []
for case in range(int(sys.argv[1]) if len(sys.argv) > 1 else 150):
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
    if n_d > 6:
        continue
    k = int(rs.integers(1, n_d + 1))
    if masses[k - 1] <= 0.0:
        continue
    n_s = int(rs.integers(2, 5))
    sub_m = tuple(float(v) for v in rs.uniform(0.0, masses[k - 1] / (n_s + 0.5), n_s))
    skey = (int(rs.integers(0, 1 << 62)), 1)
    spec, sub = hk.DecaySpec(M, masses), hk.DecaySpec(masses[k - 1], sub_m)
    fused = arr(hk.phsp_generate_chain(spec, hk.FourVector(*mother), n, hk.RngKey(*key), k, sub, hk.RngKey(*skey)))
    ref = oracle.generate(masses, M, n, key[0], key[1], mother=mother, threads=4)
    cref = np.stack(list(oracle.decay_chain(ref, k, sub_m, masses[k - 1], skey[0], skey[1], threads=4).values()))
    gamma = float(np.max(ref[f"p{k}_e"]) / masses[k - 1])
    worst = 0.0
    for j in range((fused.shape[0] - 1) // 4):
        e = np.abs(cref[1 + 4 * j])
        for c in range(4):
            worst = max(worst, float(np.max(np.abs(fused[1 + 4 * j + c] - cref[1 + 4 * j + c]) / np.maximum(e, 1e-300))))
    rows.append((gamma, worst))
rows.sort()
for g, w in rows:
    print(f"gamma_k {g:10.2f}  worst |dc|/E {w:.2e}")
