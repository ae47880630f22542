"""The row-sharded FCN's collective cost at world size 1: parallel.sharded_nll
through a 1-rank NCCL group (_force_collective: async pass, NCCL all-gather of
the 8-double record, hk_nll_combine, one host sync) against the plain
one-GPU evaluation, C4 model at 1e7 events -- the fixed cost an N-GPU FCN
evaluation adds (a lower bound: no peer traffic)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1711_05683_b200 as hk  # noqa: E402
from paper_1711_05683_b200.parallel import sharded_nll  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29531")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
P = hk.Parameter
region = hk.BoundedRegion(((0.0, 10.0),))
mean, sigma, tau = P("mean", 5.0), P("sigma", 0.5), P("tau", 3.0)
g, e = hk.shape_gaussian(mean, sigma), hk.shape_exponential(tau)
model = hk.add_pdfs([P("n_sig", 4e6), P("n_bkg", 6e6)],
                    [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])
rs = np.random.default_rng(7)
x = np.clip(np.concatenate([rs.normal(5.0, 0.5, 4_000_000), rs.exponential(3.0, 6_000_000)]), 1e-3, 9.999)
data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
pts = [(5.0, 0.5, 3.0), (4.9, 0.55, 2.8)]
out = {}
for name, force in (("plain", False), ("nccl_1rank", True)):
    def one(i, force=force):
        p = pts[i % 2]
        mean.set(p[0]); sigma.set(p[1]); tau.set(p[2])
        return sharded_nll(model, data, ["x0"], 0, _force_collective=force)
    vals = [one(i) for i in range(20)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(500):
        one(i)
    out[name + "_us"] = (time.perf_counter() - t0) / 500 * 1e6
    out[name + "_value"] = vals[0]
assert out["plain_value"] == out["nccl_1rank_value"]
# the pieces: one all_gather_into_tensor of an 8-double record, and a tiny torch op + sync
rec = torch.zeros(8, dtype=torch.float64, device="cuda")
gathered = torch.empty(8, dtype=torch.float64, device="cuda")
for _ in range(50):
    dist.all_gather_into_tensor(gathered, rec)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000):
    dist.all_gather_into_tensor(gathered, rec)
torch.cuda.synchronize()
out["all_gather_enqueue_us"] = (time.perf_counter() - t0) / 2000 * 1e6
t0 = time.perf_counter()
for _ in range(500):
    dist.all_gather_into_tensor(gathered, rec)
    torch.cuda.synchronize()
out["all_gather_sync_us"] = (time.perf_counter() - t0) / 500 * 1e6
print(json.dumps(out))
dist.destroy_process_group()
