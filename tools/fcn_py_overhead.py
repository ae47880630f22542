"""Break down the Python-side cost of fitting.nll() on the GPU (per call, us)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_05683_b200 as hk  # noqa: E402
from paper_1711_05683_b200 import _lib, fitting  # noqa: E402

rs = np.random.default_rng(7)
x = np.clip(np.concatenate([rs.normal(5.0, 0.5, 4_000_000), rs.exponential(3.0, 6_000_000)]), 1e-3, 9.999)
region = hk.BoundedRegion(((0.0, 10.0),))
g = hk.shape_gaussian(hk.Parameter("mean", 5.0), hk.Parameter("sigma", 0.5))
e = hk.shape_exponential(hk.Parameter("tau", 3.0))
model = hk.add_pdfs([hk.Parameter("n_sig", 4e6), hk.Parameter("n_bkg", 6e6)],
                    [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])
data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
cols = ["x0"]
for _ in range(20):
    hk.nll(model, data, cols)
torch.cuda.synchronize()
N = 2000
ps = model.param_set()


def t(fn, n=N):
    t0 = time.perf_counter()
    for i in range(n):
        fn(i)
    return (time.perf_counter() - t0) / n * 1e6


out = {}
out["nll_total"] = t(lambda i: hk.nll(model, data, cols))
out["nll_param_change"] = t(lambda i: (setattr(ps["mean"], "value", 5.0 + 1e-6 * (i % 7)), hk.nll(model, data, cols)))
out["observable"] = t(lambda i: fitting._observable(data, cols, model))
xo = fitting._observable(data, cols, model)
out["lower_model"] = t(lambda i: fitting.lower_model(model, xo))
out["lower_model_param_change"] = t(lambda i: (setattr(ps["mean"], "value", 5.0 + 1e-6 * (i % 7)), fitting.lower_model(model, xo)))
out["param_set_only"] = t(lambda i: setattr(ps["mean"], "value", 5.0 + 1e-6 * (i % 7)))
out["norms_param_change"] = t(lambda i: (setattr(ps["mean"], "value", 5.0 + 1e-6 * (i % 7)), [p.norm() for _, p in model.components]))
out["column_stats"] = t(lambda i: fitting.column_stats(xo))
out["stream_ptr"] = t(lambda i: _lib.stream_ptr())
out["workspace"] = t(lambda i: fitting._Workspace.get(len(data), 0))
out["expected_total"] = t(lambda i: model.expected_total())
xd = fitting._observable(data, cols, model)
lm = fitting.lower_model(model, xo)
work = fitting._Workspace.get(len(data), _lib.stream_ptr())
L = _lib.lib()
st = _lib.stream_ptr()


def raw(i):
    a, b = ctypes.c_double(), ctypes.c_uint64()
    L.hk_nll_eval(xd.data_ptr(), len(data), lm, work.data_ptr(), ctypes.byref(a), ctypes.byref(b), st)


out["c_abi_call"] = t(raw)
print({k: round(v, 2) for k, v in out.items()})
