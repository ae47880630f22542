"""kFcnFast FCN at 1e7 events through the C ABI (HK_LIB_PATH selects a build):
the kernel back to back (async hk_nll_eval, CUDA events) and the synchronous
one-launch call (wall clock)."""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_05683_b200 as hk  # noqa: E402
from paper_1711_05683_b200 import _lib  # noqa: E402
from paper_1711_05683_b200.fitting import lower_model  # noqa: E402

P = hk.Parameter
region = hk.BoundedRegion(((0.0, 10.0),))
g = hk.shape_gaussian(P("mean", 5.0), P("sigma", 0.5))
e = hk.shape_exponential(P("tau", 3.0))
model = hk.add_pdfs([P("n_sig", 4e6), P("n_bkg", 6e6)],
                    [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])
rs = np.random.default_rng(1)
xs = np.clip(np.concatenate([rs.normal(5, 0.5, 4_000_000), rs.exponential(3.0, 6_000_000)]), 1e-3, 9.999)
N = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
xs = np.resize(xs, N)
x = torch.from_numpy(xs).cuda()
n = x.numel()
L = _lib.lib()
lm = lower_model(model, x)
st = torch.cuda.current_stream()
work = torch.zeros(int(L.hk_nll_work_doubles(n)), dtype=torch.float64, device="cuda")
ls, fb = ctypes.c_double(), ctypes.c_uint64()
for _ in range(20):
    L.hk_nll_eval(x.data_ptr(), n, lm, work.data_ptr(), None, None, st.cuda_stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for rep in range(5):
    e0.record(st)
    for _ in range(200):
        L.hk_nll_eval(x.data_ptr(), n, lm, work.data_ptr(), None, None, st.cuda_stream)
    e1.record(st)
    e1.synchronize()
    best = min(best, e0.elapsed_time(e1) / 200 * 1e3)
for _ in range(20):
    L.hk_nll_eval(x.data_ptr(), n, lm, work.data_ptr(), ctypes.byref(ls), ctypes.byref(fb), st.cuda_stream)
t0 = time.perf_counter()
for _ in range(500):
    L.hk_nll_eval(x.data_ptr(), n, lm, work.data_ptr(), ctypes.byref(ls), ctypes.byref(fb), st.cuda_stream)
call = (time.perf_counter() - t0) / 500 * 1e6
print(json.dumps({"lib": os.environ.get("HK_LIB_PATH", "default"), "n": n, "kernel_us": best, "c_abi_us": call,
                  "ns_per_1k_events": best * 1e3 / n * 1e3,
                  "logsum": ls.value}))
