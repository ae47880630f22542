import sys, os, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, bench
import paper_1711_05683_b200 as hk
from paper_1711_05683_b200 import fitting, _lib
out = bench.fcn_generic(hk, torch, evals=10, keep=True)
model, data = out["_model"], out["_data"]
ps = model.param_set(); m0, g = ps["m0"], ps["g"]
pts = [(0.8955, 0.0473), (0.8900, 0.0500)]
def sets(i): m0.set(pts[i % 2][0]); g.set(pts[i % 2][1])
obs = fitting._observables(data, ["x0"], model)
st = {"sets": sets,
      "sets+norms": lambda i: (sets(i), [p.norm() for _, p in model.components]),
      "sets+lower_density": lambda i: (sets(i), fitting.lower_density(model)),
      "sets+ptr_array": lambda i: (sets(i), _lib.ptr_array(obs)),
      "sets+nll_event_sum": lambda i: (sets(i), fitting.nll_event_sum(model, data, ["x0"])),
      "sets+nll": lambda i: (sets(i), hk.nll(model, data, ["x0"]))}
res = {}
for k, f in st.items():
    for i in range(20): f(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(1000): f(i)
    res[k] = round((time.perf_counter() - t0) / 1000 * 1e6, 2)
print(res)
