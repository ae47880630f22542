"""GPU: library lifetime (hk_init / hk_shutdown) and the single-process device
clique collectives (csrc/hk_comm.cu), on the one GPU the box has.

A one-device clique still runs NCCL end to end.  The multi-device claim --
gathered chunk partials folded in device order equal the one-device fold --
is the same arithmetic the torch.distributed path is tested for under gloo
(tests/test_dist_gloo.py); here it is checked through NCCL at clique size 1
with the gathered sequence split the way a 2-device clique would hold it."""

from __future__ import annotations

import numpy as np
import pytest

from tests.common import B0_DAUGHTERS, B0_MASS, m12sq_builder

pytestmark = pytest.mark.gpu


@pytest.fixture()
def clique(hk, cuda):
    from paper_1711_05683_b200 import _lib
    _lib.init(1)
    yield _lib
    _lib.shutdown()


def test_init_validates_device_count(hk, cuda):
    import torch
    from paper_1711_05683_b200 import _lib
    with pytest.raises(ValueError, match="visible"):
        _lib.init(torch.cuda.device_count() + 1)
    assert _lib.clique_size() == 0


def test_allreduce_and_allgather_one_device(clique):
    import torch
    x = torch.arange(1000, dtype=torch.float64, device="cuda") * 0.5 + 1.0 / 3.0
    ref = x.clone()
    clique.allreduce_partials([x])
    torch.cuda.synchronize()
    assert torch.equal(x, ref)
    (g,) = clique.allgather_partials([x])
    torch.cuda.synchronize()
    assert torch.equal(g, ref)
    with pytest.raises(ValueError, match="clique has 1"):
        clique.check(clique.lib().hk_allreduce_partials(clique.ptr_array([x, x]), 2, 1000, None), "ar")


def test_gathered_chunk_partials_fold_like_one_device(hk, clique):
    """Generation weight partials -> super-chunk records -> allgather -> fold,
    bit-identical to weight_totals of the same block."""
    import torch
    n = 64 * 4096
    spec = hk.DecaySpec(B0_MASS, B0_DAUGHTERS)
    wpart = clique.empty(clique.num_weight_slices(n) * 2)
    cols = [clique.empty(n) for _ in range(13)]
    d = clique.make_decay(spec)
    k = clique.make_key(hk.RngKey(5, 1))
    clique.check(clique.lib().hk_phsp_generate(d, k, 0, n, clique.ptr_array(cols), clique.ptr(wpart),
                                               clique.stream_ptr()), "generate")
    total = clique.weight_totals(wpart, n)
    supers = clique.fold_supers(wpart, n, 0, clique.HK_SUPERS, clique.HK_WARP_SLICES, 2)
    (gathered,) = clique.allgather_partials([supers])
    folded = clique.fold(gathered, clique.HK_SUPERS, 2)
    torch.cuda.synchronize()
    assert torch.equal(folded, total)
    w = cols[0].double()
    assert folded[0].item() == pytest.approx(w.sum().item(), rel=1e-12)
    assert folded[1].item() == pytest.approx((w * w).sum().item(), rel=1e-12)
    # two "devices" holding 32 chunks (512 supers) each: their super records in device order
    # are the same sequence
    half = clique.num_weight_slices(n)  # 2 doubles per slice: the first half of wpart is chunks 0..31
    halves = [clique.fold_supers(wpart[:half], n, 0, 512, clique.HK_WARP_SLICES, 2),
              clique.fold_supers(wpart[half:], n, 512, 1024, clique.HK_WARP_SLICES, 2)]
    assert torch.equal(clique.fold(torch.cat(halves), clique.HK_SUPERS, 2), total)


def test_shutdown_releases_and_library_stays_usable(hk, cuda):
    import torch
    from paper_1711_05683_b200 import _lib
    L = _lib.lib()
    spec = hk.DecaySpec(B0_MASS, B0_DAUGHTERS)
    mother = hk.FourVector.at_rest(B0_MASS)
    block = hk.phsp_generate(spec, mother, 20_000, hk.RngKey(3, 1))
    expr = hk.identity() * hk.constant(0.987654321)
    with _lib.jit_mode(_lib.JIT_ALWAYS):
        r0 = hk.phsp_average(expr, block, m12sq_builder)
        assert L.hk_jit_count() >= 1
    host0, sums0 = hk.phsp_generate_to_host(spec, mother, 50_000, hk.RngKey(4, 1), stage_bytes=1 << 22)
    rs = np.random.default_rng(3)
    x = np.clip(np.concatenate([rs.normal(5.0, 0.5, 40_000), rs.exponential(3.0, 60_000)]), 1e-3, 9.999)
    region = hk.BoundedRegion(((0.0, 10.0),))
    g = hk.shape_gaussian(hk.Parameter("mean", 5.0), hk.Parameter("sigma", 0.5))
    e = hk.shape_exponential(hk.Parameter("tau", 3.0))
    model = hk.add_pdfs([hk.Parameter("n_sig", 4e4), hk.Parameter("n_bkg", 6e4)],
                        [hk.make_pdf(g, hk.gaussian_norm(g), region),
                         hk.make_pdf(e, hk.exponential_norm(e), region)])
    data = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [x])
    v0 = hk.nll(model, data, ["x0"])
    torch.cuda.synchronize()

    _lib.init(1)
    assert _lib.clique_size() == 1
    _lib.shutdown()
    assert _lib.clique_size() == 0
    assert L.hk_jit_count() == 0

    # every cache rebuilds on demand with identical results
    with _lib.jit_mode(_lib.JIT_ALWAYS):
        r1 = hk.phsp_average(expr, block, m12sq_builder)
        assert L.hk_jit_count() >= 1
    assert (r1.value, r1.error) == (r0.value, r0.error)
    host1, sums1 = hk.phsp_generate_to_host(spec, mother, 50_000, hk.RngKey(4, 1), stage_bytes=1 << 22)
    assert sums1 == sums0
    for name in host0.schema.names:
        assert np.array_equal(host1.column(name), host0.column(name))
    assert hk.nll(model, data, ["x0"]) == v0
