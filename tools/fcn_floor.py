import ctypes, os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_1711_05683_b200 as hk
from paper_1711_05683_b200 import _lib
from paper_1711_05683_b200.fitting import lower_model
region = hk.BoundedRegion(((0.0, 10.0),))
g = hk.shape_gaussian(hk.Parameter("mean", 5.0), hk.Parameter("sigma", 0.5)); e = hk.shape_exponential(hk.Parameter("tau", 3.0))
model = hk.add_pdfs([hk.Parameter("n_sig", 4e6), hk.Parameter("n_bkg", 6e6)], [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])
lm = lower_model(model); L = _lib.lib(); st = torch.cuda.current_stream()
rs = np.random.default_rng(1)
xs = torch.from_numpy(np.clip(rs.exponential(3.0, 10_000_000), 1e-3, 9.99)).cuda()
ls, fb = ctypes.c_double(), ctypes.c_uint64()
for n in (4096, 100_000, 1_000_000, 10_000_000):
    work = torch.zeros(int(L.hk_nll_work_doubles(n)), dtype=torch.float64, device="cuda")
    for _ in range(50): L.hk_nll_eval(_lib.ptr(xs), n, lm, _lib.ptr(work), ctypes.byref(ls), ctypes.byref(fb), st.cuda_stream)
    t = time.perf_counter()
    for _ in range(1000): L.hk_nll_eval(_lib.ptr(xs), n, lm, _lib.ptr(work), ctypes.byref(ls), ctypes.byref(fb), st.cuda_stream)
    dt = (time.perf_counter() - t) / 1000 * 1e6
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    parts = _lib.empty(_lib.num_fcn_tiles(n)); bad = _lib.bad_cells(1)
    e0.record()
    for _ in range(200): L.hk_nll_partials(_lib.ptr(xs), n, lm, _lib.ptr(parts), _lib.ptr(bad), st.cuda_stream)
    e1.record(); e1.synchronize()
    print(n, "c_abi_us", round(dt, 2), "kernel_us(k_nll back-to-back)", round(e0.elapsed_time(e1) / 200 * 1e3, 2))
# empty-ish sync floor: a torch tiny kernel + sync
t = time.perf_counter()
a = torch.zeros(1, device="cuda")
for _ in range(1000):
    a.add_(1); torch.cuda.synchronize()
print("torch tiny kernel + synchronize us", round((time.perf_counter() - t) / 1000 * 1e6, 2))
