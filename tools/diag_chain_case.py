import sys, os, math
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_1711_05683_b200 as hk
from oracle import oracle
from paper_1711_05683_b200 import _lib
def arr(b): return np.stack([np.asarray(b.column(c)) for c in b.schema.names])
rs = np.random.default_rng(1717)
for case in range(23):
    n_d = int(rs.integers(2, 9))
    masses = tuple(float(v) for v in rs.uniform(0.0, 1.0, n_d) * rs.choice([0.0, 1.0], n_d, p=[0.15, 0.85]))
    M = sum(masses) + float(10 ** rs.uniform(-1.5, 0.7))
    if rs.random() < 0.4:
        p = tuple(float(v) for v in rs.normal(0, 2 * M, 3)); mother = (math.sqrt(M * M + sum(c * c for c in p)), *p)
    else:
        mother = (M, 0.0, 0.0, 0.0)
    n = int(rs.integers(1, 3 * 4096 + 500))
    key = (int(rs.integers(0, 1 << 62)), int(rs.integers(0, 5)))
    if n_d > 6: continue
    k = int(rs.integers(1, n_d + 1))
    if masses[k - 1] <= 0.0: continue
    n_s = int(rs.integers(2, 5))
    sub_m = tuple(float(v) for v in rs.uniform(0.0, masses[k - 1] / (n_s + 0.5), n_s))
    skey = (int(rs.integers(0, 1 << 62)), 1)
    if case != 22: continue
    spec = hk.DecaySpec(M, masses); sub = hk.DecaySpec(masses[k-1], sub_m)
    print("case", case, "masses", masses, "M", M, "mother", mother, "k", k, "sub", sub_m, "n", n)
    print("fixed frame mass:", _lib.lib().hk_chain_fixed_frame_mass(_lib.make_decay(spec, hk.FourVector(*mother), M), k, _lib.make_decay(sub)))
    fused = arr(hk.phsp_generate_chain(spec, hk.FourVector(*mother), n, hk.RngKey(*key), k, sub, hk.RngKey(*skey)))
    two = arr(hk.phsp_decay_chain(hk.phsp_generate(spec, hk.FourVector(*mother), n, hk.RngKey(*key)), k, sub, hk.RngKey(*skey)))
    ref = oracle.generate(masses, M, n, key[0], key[1], mother=mother, threads=4)
    cref = np.stack(list(oracle.decay_chain(ref, k, sub_m, masses[k - 1], skey[0], skey[1], threads=4).values()))
    for name, got in (("fused", fused), ("two", two)):
        worst = 0
        for j in range((got.shape[0]-1)//4):
            e = np.abs(cref[1+4*j])
            for c in range(4):
                d = np.abs(got[1+4*j+c] - cref[1+4*j+c]) / np.maximum(e, 1e-300)
                if d.max() > worst: worst, where = d.max(), (j+1, c, int(np.argmax(d)))
        print(name, "worst |d|/E", worst, "at daughter/comp/row", where)
    j, c, r = where
    print("row", r, "E", cref[1+4*(j-1)][r], "mother-frame: parent daughter k E", ref[f"p{k}_e"][r], "px", ref[f"p{k}_px"][r])
