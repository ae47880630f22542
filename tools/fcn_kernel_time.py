"""Device time per FCN evaluation on 1e7 events: back-to-back hk_nll_eval
launches (CUDA events), one-launch C-ABI call and the resident session, plus
the batched 51-point kernel; value against the libdevice-exp reference."""
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
data = hk.generate_model_sample(model, hk.RngKey(7, 2), poisson=False)
x = data.device_column("x0")
n = len(data)
L = _lib.lib()
lm = lower_model(model)
st = torch.cuda.current_stream()
work = torch.zeros(int(L.hk_nll_work_doubles(n)), dtype=torch.float64, device="cuda")
ls, fb = ctypes.c_double(), ctypes.c_uint64()
out = {"lib": os.environ.get("HK_LIB_PATH", "default")}
# back-to-back asynchronous launches: pure device time per evaluation
for _ in range(20):
    L.hk_nll_eval(x.data_ptr(), n, lm, work.data_ptr(), None, None, st.cuda_stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
R = 200
for _ in range(R):
    L.hk_nll_eval(x.data_ptr(), n, lm, work.data_ptr(), None, None, st.cuda_stream)
e1.record(st)
e1.synchronize()
out["kernel_us"] = e0.elapsed_time(e1) / R * 1e3
t0 = time.perf_counter()
for _ in range(R):
    L.hk_nll_eval(x.data_ptr(), n, lm, work.data_ptr(), ctypes.byref(ls), ctypes.byref(fb), st.cuda_stream)
out["c_abi_us"] = (time.perf_counter() - t0) / R * 1e6
out["logsum"] = ls.value
work2 = torch.zeros(int(L.hk_nll_work_doubles(n)), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
_lib.check(L.hk_fcn_session_start(x.data_ptr(), n, work2.data_ptr(), 200_000), "start")
for _ in range(20):
    L.hk_fcn_session_eval(lm, ctypes.byref(ls), ctypes.byref(fb))
t0 = time.perf_counter()
for _ in range(R):
    L.hk_fcn_session_eval(lm, ctypes.byref(ls), ctypes.byref(fb))
out["session_us"] = (time.perf_counter() - t0) / R * 1e6
out["session_device_us"] = L.hk_fcn_session_device_ns() / 1e3
out["session_same"] = ls.value == out["logsum"]
_lib.check(L.hk_fcn_session_stop(), "stop")
from paper_1711_05683_b200.fitting import nll_many  # noqa: E402
ps = model.param_set()
base = np.array(ps.values())
pts = [tuple(base * (1 + 1e-4 * np.random.default_rng(i).standard_normal(5))) for i in range(51)]
nll_many(model, data, ["x0"], pts)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    nll_many(model, data, ["x0"], pts)
out["many51_us_per_point"] = (time.perf_counter() - t0) / 10 / 51 * 1e6
print(json.dumps(out))
