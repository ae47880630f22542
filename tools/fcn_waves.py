"""FCN kernel time against the number of 4096-row tiles (waves of 592 resident
CTAs on 148 SMs): separates launch/ramp, steady state and tail."""
import ctypes, os, sys
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
xs = torch.from_numpy(np.clip(np.concatenate([rs.normal(5, .5, 4_000_000), rs.exponential(3.0, 6_000_000)]), 1e-3, 9.99)[rs.permutation(10_000_000)]).cuda()
for tiles in (592, 1184, 1776, 2368, 2369, 2442, 2960):
    n = tiles * 4096 if tiles * 4096 <= 10_000_000 else 10_000_000
    parts = _lib.empty(_lib.num_fcn_tiles(n)); bad = _lib.bad_cells(1)
    for _ in range(20): L.hk_nll_partials(_lib.ptr(xs), n, lm, _lib.ptr(parts), _lib.ptr(bad), st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200): L.hk_nll_partials(_lib.ptr(xs), n, lm, _lib.ptr(parts), _lib.ptr(bad), st.cuda_stream)
    e1.record(); e1.synchronize()
    us = e0.elapsed_time(e1) / 200 * 1e3
    print(tiles, n, round(us, 2), "us", round(us / n * 1e6, 3), "ns/1k-ev")
