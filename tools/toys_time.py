"""generate_model_sample of the C4 model (1e7 events): wall time per call
(bench TOYS) -- run under ncu for the per-kernel split."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1711_05683_b200 as hk  # noqa: E402

print(json.dumps(bench.toy_sample(hk, torch)))
t0 = time.perf_counter()
from paper_1711_05683_b200.rng import estimate_ceiling  # noqa: E402
g = hk.shape_gaussian(hk.Parameter("mean", 5.0), hk.Parameter("sigma", 0.5))
region = hk.BoundedRegion(((0.0, 10.0),))
for _ in range(10):
    estimate_ceiling(g, region)
torch.cuda.synchronize()
print(json.dumps({"estimate_ceiling_ms": (time.perf_counter() - t0) / 10 * 1e3}))
