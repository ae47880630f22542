"""GPU: run-to-run bitwise determinism of every kernel family with a
cross-thread or cross-CTA reduction -- the race detector available on this
pool (compute-sanitizer is not).  A missing barrier or fence in the cluster
fold, the CTA trees, the FCN's last-CTA fold + mapped mailbox or the CSV
block scan would show up as results that differ between identical runs."""

from __future__ import annotations

import io

import numpy as np
import pytest

from tests.common import B0_DAUGHTERS, B0_MASS, m12sq_builder

pytestmark = pytest.mark.gpu
REPEATS = 6


def _bits(x) -> bytes:
    return np.asarray(x, dtype=np.float64).tobytes()


def test_reductions_are_bitwise_repeatable(cuda, hk):
    from paper_1711_05683_b200 import _lib
    spec, mother = hk.DecaySpec(B0_MASS, B0_DAUGHTERS), hk.FourVector.at_rest(B0_MASS)
    n = 2_000_000 + 517                                   # ragged last chunk
    rs = np.random.default_rng(11)
    x = np.clip(np.concatenate([rs.normal(5, 0.5, 400_000), rs.exponential(3.0, 600_000)]), 1e-3, 9.999)
    region = hk.BoundedRegion(((0.0, 10.0),))
    g = hk.shape_gaussian(hk.Parameter("mean", 5.0), hk.Parameter("sigma", 0.5))
    e = hk.shape_exponential(hk.Parameter("tau", 3.0))
    model = hk.add_pdfs([hk.Parameter("n_sig", 4e5), hk.Parameter("n_bkg", 6e5)],
                        [hk.make_pdf(g, hk.gaussian_norm(g), region),
                         hk.make_pdf(e, hk.exponential_norm(e), region)])
    data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
    seen = None
    for _ in range(REPEATS):
        blk = hk.phsp_generate(spec, mother, n, hk.RngKey(3, 1))
        wm = hk.phsp_weight_moments(blk)                  # warp slots -> chunk fold -> cluster fold
        avg = hk.phsp_average(hk.identity(), blk, m12sq_builder)          # CTA tree + fold
        fused = hk.phsp_integrate(hk.identity(), spec, mother, n, hk.RngKey(3, 1), m12sq_builder,
                                  return_partials=True)
        with _lib.jit_mode(_lib.JIT_OFF):                 # the interpreter kernels too
            interp = hk.phsp_integrate(hk.identity() * hk.identity(), spec, mother, n, hk.RngKey(3, 1),
                                       m12sq_builder, return_partials=True)
        fcn = hk.nll(model, data, ["x0"])                 # last-CTA fold + mapped mailbox
        buf = io.BytesIO()
        blk.where_mask(np.arange(n) < 300_000).write_csv(buf)   # block scan + pack
        got = (_bits([wm.sum_w, wm.mean, wm.variance]), _bits([avg.value, avg.error]),
               fused.cpu().numpy().tobytes(), interp.cpu().numpy().tobytes(), _bits([fcn]),
               buf.getvalue())
        if seen is None:
            seen = got
        else:
            for name, a, b in zip(("weights", "average", "fused", "interpreter", "fcn", "csv"), seen, got):
                assert a == b, f"{name} differs between identical runs"


def test_sampler_streams_are_independent(hk, cuda):
    """The work-stealing sampler keeps one event counter per (device, stream):
    two samples enqueued on two streams at once equal the same samples taken
    one after the other."""
    import numpy as np
    torch = cuda
    region = hk.BoundedRegion(((0.0, 10.0),))
    g = hk.shape_gaussian(hk.Parameter("m", 5.0), hk.Parameter("s", 0.5))
    want = [np.asarray(hk.sample_pdf(g, region, 400_000, hk.RngKey(k, 2), ceiling=1.0).column("x0"))
            for k in (1, 2)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        a = hk.sample_pdf(g, region, 400_000, hk.RngKey(1, 2), ceiling=1.0)
    with torch.cuda.stream(s2):
        b = hk.sample_pdf(g, region, 400_000, hk.RngKey(2, 2), ceiling=1.0)
    torch.cuda.synchronize()
    assert np.array_equal(np.asarray(a.column("x0")), want[0])
    assert np.array_equal(np.asarray(b.column("x0")), want[1])
