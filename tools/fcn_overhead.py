"""Where the per-call FCN time goes on the host (1e7-event gauss+exp model)."""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_05683_b200 as hk  # noqa: E402
from paper_1711_05683_b200 import _lib  # noqa: E402
from paper_1711_05683_b200.fitting import _Workspace, _observable, lower_model  # noqa: E402


def per_call(fn, n=2000):
    for _ in range(50):
        fn()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t) / n * 1e6


region = hk.BoundedRegion(((0.0, 10.0),))
mean, sigma, tau = hk.Parameter("mean", 5.0), hk.Parameter("sigma", 0.5), hk.Parameter("tau", 3.0)
g, e = hk.shape_gaussian(mean, sigma), hk.shape_exponential(tau)
model = hk.add_pdfs([hk.Parameter("n_sig", 4e6), hk.Parameter("n_bkg", 6e6)],
                    [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])
rs = np.random.default_rng(1)
x = np.clip(np.concatenate([rs.normal(5, 0.5, 4_000_000), rs.exponential(3.0, 6_000_000)]), 1e-3, 9.999)
store = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
hk.nll(model, store, ["x0"])
xd = store.device_column("x0")
lm = lower_model(model)
work = _Workspace.get(len(store), _lib.stream_ptr())
ls, fb = ctypes.c_double(), ctypes.c_uint64()
L = _lib.lib()
sp = _lib.stream_ptr()
pts = [(5.0, 0.5, 3.0), (4.9, 0.55, 2.8)]
it = [0]


def setp():
    p = pts[it[0] & 1]
    it[0] += 1
    mean.set(p[0]); sigma.set(p[1]); tau.set(p[2])


out = {
    "stream_ptr": per_call(_lib.stream_ptr),
    "current_device": per_call(torch.cuda.current_device),
    "workspace_get": per_call(lambda: _Workspace.get(len(store), sp)),
    "observable": per_call(lambda: _observable(store, ["x0"], model)),
    "set_params": per_call(setp),
    "set_params+lower_model": per_call(lambda: (setp(), lower_model(model))),
    "c_abi_nll_eval": per_call(lambda: L.hk_nll_eval(_lib.ptr(xd), len(store), lm, _lib.ptr(work),
                                                     ctypes.byref(ls), ctypes.byref(fb), sp)),
    "python_nll_fixed_params": per_call(lambda: hk.nll(model, store, ["x0"])),
    "python_nll_changing_params": per_call(lambda: (setp(), hk.nll(model, store, ["x0"]))),
}
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(200):
    L.hk_nll_eval(_lib.ptr(xd), len(store), lm, _lib.ptr(work), ctypes.byref(ls), ctypes.byref(fb), sp)
e1.record(st)
e1.synchronize()
out["device_time_per_eval_us"] = e0.elapsed_time(e1) / 200 * 1e3
print(json.dumps({k: round(v, 2) for k, v in out.items()}))
