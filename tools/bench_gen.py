"""Micro-benchmark of the generator kernel through the C ABI (HK_LIB_PATH selects a build).

    HK_LIB_PATH=... python tools/bench_gen.py [--n 1e8] [--reps 10] [--rng reference]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1711_05683_b200 as hk  # noqa: E402
from paper_1711_05683_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e8)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--rng", default="reference")
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--chain", action="store_true", help="also time the fused C3 chain")
    a = ap.parse_args()
    n = int(a.n)
    M, ms = 5.27966, (3.0969, 0.493677, 0.13957039)
    spec = hk.DecaySpec(M, ms)
    d = _lib.make_decay(spec)
    k = _lib.make_key(hk.RngKey(1, 1), hk.rng.rng_mode(a.rng))
    cols = [_lib.empty(n) for _ in range(13)]
    cp = _lib.ptr_array(cols)
    wp = _lib.empty(2 * _lib.num_weight_slices(n))
    st = torch.cuda.current_stream()
    L = _lib.lib()
    for _ in range(3):
        _lib.check(L.hk_phsp_generate(d, k, 0, n, cp, _lib.ptr(wp), st.cuda_stream), "gen")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        L.hk_phsp_generate(d, k, 0, n, cp, _lib.ptr(wp), st.cuda_stream)
    e1.record()
    e1.synchronize()
    ms_ = e0.elapsed_time(e1) / a.reps
    out = {"lib": os.environ.get("HK_LIB_PATH", "default"), "n": n, "ms": ms_, "ev_per_s": n / ms_ * 1e3,
           "GBps": 104 * n / ms_ / 1e6}
    # fused chain (C3): B0 -> J/psi(-> mu mu) K pi, 1.25e8 events, 17 columns
    if a.chain:
        gen_check = [c[:200_000].clone() for c in cols] if a.check else None
        del cols
        torch.cuda.empty_cache()
        nc = 125_000_000
        ccols = [_lib.empty(nc) for _ in range(17)]
        ccp = _lib.ptr_array(ccols)
        cw = _lib.empty(2 * _lib.num_weight_slices(nc))
        cbad = _lib.bad_cells(1)
        sub = _lib.make_decay(hk.DecaySpec(3.0969, (0.1056583755, 0.1056583755)))
        sk = _lib.make_key(hk.RngKey(2, 1), hk.rng.rng_mode(a.rng))
        for _ in range(2):
            _lib.check(L.hk_phsp_generate_chain(d, k, 1, sub, sk, 0, nc, ccp, _lib.ptr(cw), _lib.ptr(cbad),
                                                st.cuda_stream), "chain")
        e0.record()
        for _ in range(5):
            L.hk_phsp_generate_chain(d, k, 1, sub, sk, 0, nc, ccp, _lib.ptr(cw), _lib.ptr(cbad), st.cuda_stream)
        e1.record()
        e1.synchronize()
        cms = e0.elapsed_time(e1) / 5
        out.update({"chain_ms": cms, "chain_ev_per_s": nc / cms * 1e3, "chain_GBps": 136 * nc / cms / 1e6})
        del ccols
        torch.cuda.empty_cache()
        cols = gen_check
    # FCN kernel on 1e7 gauss+exp events (hk_nll_partials, one launch per eval)
    rs = np.random.default_rng(7)
    xs = np.clip(np.concatenate([rs.normal(5.0, 0.5, 4_000_000), rs.exponential(3.0, 6_000_000)]), 1e-3, 9.999)
    x = torch.from_numpy(xs).cuda()
    from paper_1711_05683_b200.fitting import lower_model
    g = hk.shape_gaussian(hk.Parameter("mean", 5.0), hk.Parameter("sigma", 0.5))
    e = hk.shape_exponential(hk.Parameter("tau", 3.0))
    reg = hk.BoundedRegion(((0.0, 10.0),))
    model = hk.add_pdfs([hk.Parameter("n_sig", 4e6), hk.Parameter("n_bkg", 6e6)],
                        [hk.make_pdf(g, hk.gaussian_norm(g), reg), hk.make_pdf(e, hk.exponential_norm(e), reg)])
    lm = lower_model(model)
    parts = _lib.empty(_lib.num_fcn_tiles(x.numel()))
    bad = _lib.bad_cells(1)
    for _ in range(3):
        L.hk_nll_partials(_lib.ptr(x), x.numel(), lm, _lib.ptr(parts), _lib.ptr(bad), st.cuda_stream)
    e0.record()
    for _ in range(50):
        L.hk_nll_partials(_lib.ptr(x), x.numel(), lm, _lib.ptr(parts), _lib.ptr(bad), st.cuda_stream)
    e1.record()
    e1.synchronize()
    out["fcn_kernel_us"] = e0.elapsed_time(e1) / 50 * 1e3
    # one-launch FCN through the C ABI (k_nll_fused + mailbox), synchronous per call
    import ctypes
    import time
    work = torch.zeros(int(_lib.lib().hk_nll_work_doubles(x.numel())), dtype=torch.float64, device="cuda")
    ls, fb = ctypes.c_double(), ctypes.c_uint64()
    for _ in range(20):
        L.hk_nll_eval(_lib.ptr(x), x.numel(), lm, _lib.ptr(work), ctypes.byref(ls), ctypes.byref(fb), st.cuda_stream)
    t0 = time.perf_counter()
    for _ in range(200):
        L.hk_nll_eval(_lib.ptr(x), x.numel(), lm, _lib.ptr(work), ctypes.byref(ls), ctypes.byref(fb), st.cuda_stream)
    out["fcn_eval_us"] = (time.perf_counter() - t0) / 200 * 1e6
    if a.check:
        from oracle import oracle as O
        want = O.nll(xs, O.gauss_exp_components(5.0, 0.5, 3.0, 4e6, 6e6))
        got = hk.nll(model, hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [xs]), ["x0"])
        out["fcn_rel_err"] = abs(got - want) / abs(want)
    if a.check:
        from oracle import oracle as O
        ref = O.generate(ms, M, 200_000, 1, 1, threads=8)
        worst = 0.0
        for j in range(3):
            e = np.abs(ref[f"p{j+1}_e"])
            for c in ("e", "px", "py", "pz"):
                g = cols[1 + 4 * j + "e px py pz".split().index(c)][:200_000].cpu().numpy()
                worst = max(worst, float(np.max(np.abs(g - ref[f"p{j+1}_{c}"]) / e)))
        out["max_dc_over_E"] = worst
        out["weights_bit_exact"] = bool(np.array_equal(cols[0][:200_000].cpu().numpy(), ref["weight"]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
