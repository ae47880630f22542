import cProfile, pstats, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1711_05683_b200 as hk
M, ms = 5.27966, (3.0969, 0.493677, 0.13957039)
spec, mother = hk.DecaySpec(M, ms), hk.FourVector.at_rest(M)
key = hk.RngKey(1, 1)
for _ in range(100): hk.phsp_generate(spec, mother, 100_000, key)
torch.cuda.synchronize()
import time
t = time.perf_counter()
for _ in range(5000): hk.phsp_generate(spec, mother, 100_000, key)
torch.cuda.synchronize()
print("per call us", (time.perf_counter() - t) / 5000 * 1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(5000): hk.phsp_generate(spec, mother, 100_000, key)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
