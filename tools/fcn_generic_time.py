"""FCN for a model outside the closed-form kernels (bench.fcn_generic: Breit-
Wigner + linear polynomial closures, NVRTC density program) at 1e7 events:
nll() rate, and the program kernel alone through the C ABI (async, back to
back, CUDA events)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1711_05683_b200 as hk  # noqa: E402
from paper_1711_05683_b200 import _lib  # noqa: E402
from paper_1711_05683_b200.fitting import _Workspace, lower_density  # noqa: E402

out = bench.fcn_generic(hk, torch, keep=True)
model, data = out.pop("_model"), out.pop("_data")
n = len(data)
st = _lib.stream_ptr()
dm = lower_density(model)
obs = _lib.ptr_array([data.device_column("x0")])
work = _Workspace.get(n, st)
L = _lib.lib()
for _ in range(10):
    L.hk_nll_program_eval(obs, n, dm, work.data_ptr(), None, None, None, st)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    L.hk_nll_program_eval(obs, n, dm, work.data_ptr(), None, None, None, st)
e1.record()
e1.synchronize()
out["kernel_us"] = e0.elapsed_time(e1) / 200 * 1e3
import ctypes  # noqa: E402
import time  # noqa: E402
ls, fb, fz = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_uint64()
for _ in range(10):
    L.hk_nll_program_eval(obs, n, dm, work.data_ptr(), ctypes.byref(ls), ctypes.byref(fb), ctypes.byref(fz), st)
t0 = time.perf_counter()
for _ in range(200):
    L.hk_nll_program_eval(obs, n, dm, work.data_ptr(), ctypes.byref(ls), ctypes.byref(fb), ctypes.byref(fz), st)
out["c_abi_us"] = (time.perf_counter() - t0) / 200 * 1e6
from paper_1711_05683_b200.fitting import lower_density as _ld  # noqa: E402
t0 = time.perf_counter()
for _ in range(2000):
    _ld(model)
out["lower_density_us"] = (time.perf_counter() - t0) / 2000 * 1e6
print(json.dumps(out))
