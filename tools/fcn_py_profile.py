"""Where the host time of one FCN evaluation goes (the bench's C4 loop:
three parameter sets, then parallel.sharded_nll at world 1): cumulative
stage timings per call (us) and a cProfile of the whole call."""
import cProfile
import io
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_05683_b200 as hk  # noqa: E402
from paper_1711_05683_b200 import fitting  # noqa: E402
from paper_1711_05683_b200.parallel import sharded_nll  # noqa: E402

rs = np.random.default_rng(7)
x = np.clip(np.concatenate([rs.normal(5.0, 0.5, 4_000_000), rs.exponential(3.0, 6_000_000)]), 1e-3, 9.999)
P = hk.Parameter
region = hk.BoundedRegion(((0.0, 10.0),))
mean, sigma, tau = P("mean", 5.0), P("sigma", 0.5), P("tau", 3.0)
g = hk.shape_gaussian(mean, sigma)
e = hk.shape_exponential(tau)
model = hk.add_pdfs([P("n_sig", 4e6), P("n_bkg", 6e6)],
                    [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])
data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
pts = [(5.0, 0.5, 3.0), (4.9, 0.55, 2.8)]
xd = data.device_column("x0")


def sets(i):
    p = pts[i % 2]
    mean.set(p[0]); sigma.set(p[1]); tau.set(p[2])


stages = {
    "loop": lambda i: None,
    "param_sets": sets,
    "sets+norms": lambda i: (sets(i), [pdf.norm() for _, pdf in model.components]),
    "sets+lower_model": lambda i: (sets(i), fitting.lower_model(model, xd)),
    "sets+nll_event_sum": lambda i: (sets(i), fitting.nll_event_sum(model, data, ["x0"])),
    "sets+nll": lambda i: (sets(i), hk.nll(model, data, ["x0"])),
    "sets+sharded_nll": lambda i: (sets(i), sharded_nll(model, data, ["x0"], 0)),
}
for fn in stages.values():
    for i in range(50):
        fn(i)
torch.cuda.synchronize()
N = 3000
out = {}
for name, fn in stages.items():
    t0 = time.perf_counter()
    for i in range(N):
        fn(i)
    out[name] = round((time.perf_counter() - t0) / N * 1e6, 2)
print(out)
pr = cProfile.Profile()
pr.enable()
for i in range(2000):
    stages["sets+sharded_nll"](i)
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(18)
print(s.getvalue())
