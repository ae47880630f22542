"""FCN timing on the C4 data set (1e7 events, build_model(scale=200), RngKey(7,2)):
single-point nll() rate, the batched 51-point Hessian pass (hk_nll_eval_many)
and the whole C4 fit wall time, serial objective vs batched."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_05683_b200 as hk  # noqa: E402
from paper_1711_05683_b200.fitting import NllObjective, nll_many, numeric_errors  # noqa: E402


def model(scale=200.0):
    P = hk.Parameter
    region = hk.BoundedRegion(((0.0, 10.0),))
    g = hk.shape_gaussian(P("mean", 5.0, step=0.1), P("sigma", 0.5, step=0.05, lower=1e-4))
    e = hk.shape_exponential(P("tau", 3.0, step=0.2, lower=1e-4))
    ns, nb = 20000.0 * scale, 30000.0 * scale
    return hk.add_pdfs([P("n_sig", ns, step=ns ** 0.5, lower=0.0), P("n_bkg", nb, step=nb ** 0.5, lower=0.0)],
                       [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])


m = model()
data = hk.generate_model_sample(m, hk.RngKey(7, 2), poisson=False)
ps = m.param_set()
out = {}
pts = [(5.0, 0.5, 3.0), (4.9, 0.55, 2.8)]
for i in range(20):
    ps["mean"].set(pts[i % 2][0]); ps["sigma"].set(pts[i % 2][1]); ps["tau"].set(pts[i % 2][2])
    hk.nll(m, data, ["x0"])
torch.cuda.synchronize()
N = 400
t0 = time.perf_counter()
for i in range(N):
    p = pts[i % 2]
    ps["mean"].set(p[0]); ps["sigma"].set(p[1]); ps["tau"].set(p[2])
    hk.nll(m, data, ["x0"])
dt = (time.perf_counter() - t0) / N
out["single_nll_us"] = dt * 1e6
out["single_nll_evals_per_s"] = 1.0 / dt
with hk.fcn_session(m, data, ["x0"]):
    for i in range(20):
        p = pts[i % 2]
        ps["mean"].set(p[0]); ps["sigma"].set(p[1]); ps["tau"].set(p[2])
        hk.nll(m, data, ["x0"])
    t0 = time.perf_counter()
    for i in range(N):
        p = pts[i % 2]
        ps["mean"].set(p[0]); ps["sigma"].set(p[1]); ps["tau"].set(p[2])
        hk.nll(m, data, ["x0"])
    dt = (time.perf_counter() - t0) / N
    from paper_1711_05683_b200 import _lib as _L  # noqa: E402
    from paper_1711_05683_b200.fitting import lower_model as _lm  # noqa: E402
    import ctypes as _ct  # noqa: E402
    lms = []
    for p in pts:
        ps["mean"].set(p[0]); ps["sigma"].set(p[1]); ps["tau"].set(p[2])
        lm_ = _L.hk_model_t()
        _ct.memmove(_ct.byref(lm_), _ct.byref(_lm(m, data.device_column("x0"))), _ct.sizeof(lm_))
        lms.append(lm_)
    ls_, fb_ = _ct.c_double(), _ct.c_uint64()
    f = _L.lib().hk_fcn_session_eval
    t1 = time.perf_counter()
    for i in range(N):
        f(lms[i & 1], _ct.byref(ls_), _ct.byref(fb_))
    out["session_c_abi_us"] = (time.perf_counter() - t1) / N * 1e6
out["session_nll_us"] = dt * 1e6
out["session_nll_evals_per_s"] = 1.0 / dt
ps.set_values((4e6, 5.0, 0.5, 6e6, 3.0))
base = np.array(ps.values())
rs = np.random.default_rng(1)
for k in (51, 64):
    P = [tuple(base * (1 + 1e-4 * rs.standard_normal(5))) for _ in range(k)]
    nll_many(m, data, ["x0"], P)
    torch.cuda.synchronize()
    reps = 20
    t0 = time.perf_counter()
    for _ in range(reps):
        nll_many(m, data, ["x0"], P)
    dt = (time.perf_counter() - t0) / reps
    out[f"many{k}_ms"] = dt * 1e3
    out[f"many{k}_evals_per_s"] = k / dt
st = torch.cuda.current_stream()
from paper_1711_05683_b200 import _lib  # noqa: E402
from paper_1711_05683_b200.fitting import _ManyWorkspace, lower_model  # noqa: E402
import ctypes  # noqa: E402
k = 51
models = (_lib.hk_model_t * k)()
for i in range(k):
    ctypes.memmove(ctypes.byref(models, i * ctypes.sizeof(_lib.hk_model_t)), ctypes.byref(lower_model(m, data.device_column("x0"))),
                   ctypes.sizeof(_lib.hk_model_t))
x = data.device_column("x0")
work = _ManyWorkspace.get(len(data), k, _lib.stream_ptr())
sums, bad = (ctypes.c_double * k)(), (ctypes.c_uint64 * k)()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(20):
    _lib.lib().hk_nll_eval_many(x.data_ptr(), len(data), models, k, work.data_ptr(), sums, bad, st.cuda_stream)
e1.record(st)
e1.synchronize()
out["many51_kernel_ms"] = e0.elapsed_time(e1) / 20
out["many51_kernel_events_per_s"] = k * len(data) / (out["many51_kernel_ms"] * 1e-3)
# the single-point API kernel alone (k_nll_fused, kFcnFast), back to back
lm1 = lower_model(m, x)
w1 = torch.zeros(int(_lib.lib().hk_nll_work_doubles(len(data))), dtype=torch.float64, device="cuda")
for _ in range(5):
    _lib.lib().hk_nll_eval(x.data_ptr(), len(data), lm1, w1.data_ptr(), None, None, st.cuda_stream)
e0.record(st)
for _ in range(200):
    _lib.lib().hk_nll_eval(x.data_ptr(), len(data), lm1, w1.data_ptr(), None, None, st.cuda_stream)
e1.record(st)
e1.synchronize()
out["single_kernel_us"] = e0.elapsed_time(e1) / 200 * 1e3
# whole C4 fit from a displaced start, serial objective vs batched
for mode in ("serial", "batched"):
    mm = model()
    pp = mm.param_set()
    pp["mean"].set(4.8); pp["sigma"].set(0.6); pp["tau"].set(2.6)
    if mode == "serial":
        import paper_1711_05683_b200.fitting as F
        orig = F.NllObjective.many
        F.NllObjective.many = None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = hk.fit(mm, data, ["x0"])
    dt = time.perf_counter() - t0
    if mode == "serial":
        F.NllObjective.many = orig
    out[f"fit_{mode}_s"] = dt
    out[f"fit_{mode}_calls"] = res.n_calls
    out[f"fit_{mode}_status"] = res.status.value
    out[f"fit_{mode}_params"] = dict(zip(pp.names, pp.values()))
print(json.dumps(out))
