import sys, time, json, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1711_05683_b200 as hk
import paper_1711_05683_b200.fitting as F
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
out = {}
for rep in range(3):
    for mode in ("serial", "batched"):
        mm = model(); pp = mm.param_set()
        pp["mean"].set(4.8); pp["sigma"].set(0.6); pp["tau"].set(2.6)
        if mode == "serial":
            orig = F.NllObjective.many; F.NllObjective.many = None
        torch.cuda.synchronize()
        t0 = time.perf_counter(); res = hk.fit(mm, data, ["x0"]); dt = time.perf_counter() - t0
        if mode == "serial":
            F.NllObjective.many = orig
        out[f"{mode}{rep}"] = dt
print(json.dumps(out))
import cProfile, pstats
mm = model(); pp = mm.param_set(); pp["mean"].set(4.8); pp["sigma"].set(0.6); pp["tau"].set(2.6)
cProfile.run('hk.fit(mm, data, ["x0"])', '/tmp/fit.prof')
pstats.Stats('/tmp/fit.prof').sort_stats('cumtime').print_stats(25)
