"""Fixed per-call cost of the FCN paths: C-ABI time per call for the launched
kernel (hk_nll_eval) and the resident session (hk_fcn_session_eval) at data
sizes from one tile to the C4 1e7 events."""
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
xall = np.clip(np.concatenate([rs.normal(5, 0.5, 4_000_000), rs.exponential(3.0, 6_000_000)]), 1e-3, 9.999)
L = _lib.lib()
out = []
for n in (4096, 4096 * 148, 4096 * 592, 1_000_000, 10_000_000):
    x = torch.from_numpy(xall[:n].copy()).cuda()
    lm = lower_model(model, x)   # with the column statistics: the kFcnFast path
    work = torch.zeros(int(L.hk_nll_work_doubles(n)), dtype=torch.float64, device="cuda")
    ls, fb = ctypes.c_double(), ctypes.c_uint64()
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(50):
        L.hk_nll_eval(x.data_ptr(), n, lm, work.data_ptr(), ctypes.byref(ls), ctypes.byref(fb), st)
    N = 500
    t0 = time.perf_counter()
    for _ in range(N):
        L.hk_nll_eval(x.data_ptr(), n, lm, work.data_ptr(), ctypes.byref(ls), ctypes.byref(fb), st)
    launched = (time.perf_counter() - t0) / N * 1e6
    v_launched = ls.value
    work2 = torch.zeros(int(L.hk_nll_work_doubles(n)), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    _lib.check(L.hk_fcn_session_start(x.data_ptr(), n, work2.data_ptr(), 200_000), "start")
    for _ in range(50):
        L.hk_fcn_session_eval(lm, ctypes.byref(ls), ctypes.byref(fb))
    t0 = time.perf_counter()
    for _ in range(N):
        L.hk_fcn_session_eval(lm, ctypes.byref(ls), ctypes.byref(fb))
    session = (time.perf_counter() - t0) / N * 1e6
    dev_ns = L.hk_fcn_session_device_ns()
    _lib.check(L.hk_fcn_session_stop(), "stop")
    out.append({"n": n, "launched_us": round(launched, 2), "session_us": round(session, 2), "session_device_us": dev_ns / 1e3,
                "same_value": ls.value == v_launched})
print(json.dumps(out))
