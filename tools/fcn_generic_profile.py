"""cProfile of nll() for the density-program model (bench.fcn_generic)."""
import cProfile
import io
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1711_05683_b200 as hk  # noqa: E402

out = bench.fcn_generic(hk, torch, evals=20, keep=True)
model, data = out["_model"], out["_data"]
ps = model.param_set()
m0, g = ps["m0"], ps["g"]
pts = [(0.8955, 0.0473), (0.8900, 0.0500)]
pr = cProfile.Profile()
pr.enable()
for i in range(500):
    m0.set(pts[i % 2][0]); g.set(pts[i % 2][1])
    hk.nll(model, data, ["x0"])
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue())
