"""phsp_unweight of a stored 1e8-event C2 block (accept flags + order-
preserving compaction), per-kernel device times and the API call."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1711_05683_b200 as hk  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
spec = hk.DecaySpec(5.27966, (3.0969, 0.493677, 0.13957039))
blk = hk.phsp_generate(spec, hk.FourVector.at_rest(5.27966), n, hk.RngKey(1, 1))
w_max = hk.phsp_max_weight(spec)
for _ in range(2):
    out = hk.phsp_unweight(blk, w_max, hk.RngKey(1, 4))
torch.cuda.synchronize()
reps = 10
t0 = time.perf_counter()
for _ in range(reps):
    out = hk.phsp_unweight(blk, w_max, hk.RngKey(1, 4))
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / reps
m = len(out)
print(json.dumps({"n": n, "accepted": m, "ms": dt * 1e3, "ev_per_s": n / dt,
                  "GBps_algorithmic": (9 * n + n + 2 * 104 * m) / dt / 1e9}))
