"""Deterministic data parallelism across GPUs (reference parallel.py:1-92).

The reference splits every bulk operation into fixed 65 536-row batches and
4096-row chunk partials folded in a fixed order, so results do not depend on
the worker count.  Here the "workers" are GPUs, one process per GPU
(torch.distributed, NCCL over NVLink/NVSwitch):

* events shard as contiguous, chunk-aligned global row ranges
  (``shard_range``); each rank generates/evaluates its range with the
  *global* row index, so shards are bit-identical to the same rows of a
  one-GPU run (RNG counters are global, phasespace.py:105-109);
* the only exchange is the chunk partials: ``gather_partials`` all-gathers
  them (a few KB per rank) into global chunk order and every rank folds the
  same array with the same fixed tree -- so the reduced value is bitwise
  independent of the number of GPUs (the analogue of the reference's
  worker-invariance tests, test_phasespace.py:87-93, test_fitting.py:120-124).
"""

from __future__ import annotations

import os

from . import _lib

CHUNK = _lib.HK_CHUNK          # parallel.py:18
EVAL_BATCH = 16 * CHUNK        # parallel.py:21


def resolve_workers(workers: int | None) -> int:
    """Reference knob (parallel.py:42-48); accepted and ignored by the GPU path."""
    if workers is None or workers == 0:
        return os.cpu_count() or 1
    if workers < 0:
        raise ValueError(f"workers must be >= 0, got {workers}")
    return workers


def batch_ranges(n: int, batch: int = EVAL_BATCH) -> list[tuple[int, int]]:
    return [(s, min(s + batch, n)) for s in range(0, n, batch)]


def chunk_bounds(start: int, stop: int, chunk: int = CHUNK) -> list[tuple[int, int]]:
    first = (start // chunk) * chunk
    return [(max(s, start), min(s + chunk, stop)) for s in range(first, stop, chunk)
            if max(s, start) < min(s + chunk, stop)]


def shard_range(n: int, rank: int, world: int, chunk: int = CHUNK) -> tuple[int, int]:
    """Contiguous chunk-aligned [a, b) of rank's rows; shards cover [0, n)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    nch = (n + chunk - 1) // chunk
    c0 = nch * rank // world
    c1 = nch * (rank + 1) // world
    return min(c0 * chunk, n), min(c1 * chunk, n)


def dist_info(group=None) -> tuple[int, int]:
    """(rank, world) of the default process group, (0, 1) when not initialised."""
    torch = _lib.torch()
    dist = torch.distributed
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def gather_partials(local, n_total: int, width: int, group=None):
    """All-gather per-chunk partials (local: flat tensor of this rank's chunks
    x width) into global chunk order on every rank.

    Shards are chunk-aligned, so the concatenation of the ranks' partials in
    rank order is exactly the global chunk sequence.  Unequal shard sizes are
    padded to the largest and trimmed after the gather.
    """
    torch = _lib.torch()
    rank, world = dist_info(group)
    if world == 1:
        return local
    dist = torch.distributed
    nch = (n_total + CHUNK - 1) // CHUNK
    sizes = [(nch * (r + 1) // world - nch * r // world) for r in range(world)]
    cap = max(sizes) * width
    # NCCL gathers device tensors in place; CPU backends (gloo) go through host memory
    dev = local.device if dist.get_backend(group) == "nccl" else "cpu"
    buf = torch.zeros(cap, dtype=local.dtype, device=dev)
    buf[: local.numel()] = local.to(dev)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    return torch.cat([o[: s * width] for o, s in zip(out, sizes)]).to(local.device)


def sharded_weight_moments(block_shard, n_total: int, group=None):
    """Global (sum w, sum w^2) of a sharded generation: gather + same fold."""
    parts = block_shard.meta["weight_partials"]   # 2 doubles per warp-slice, 8 slices per chunk
    # fold each chunk's 8 slices locally (fixed order), so only one record per
    # chunk crosses GPUs; every rank then folds the same global chunk sequence
    local = _lib.weight_chunk_partials(parts, len(block_shard))
    full = gather_partials(local, n_total, 2, group)
    return _lib.fold(full, _lib.num_chunks(n_total), 2)


def sharded_integrate(expr, spec, mother, n_total: int, key, arg_builder, group=None,
                      rng: str = "reference"):
    """phsp_integrate over n_total events sharded across the process group
    (config C5 at 1/2/4/8 GPUs); returns the IntegrationResult on every rank."""
    from .phasespace import _finish_average, phsp_integrate  # noqa: PLC0415

    rank, world = dist_info(group)
    a, b = shard_range(n_total, rank, world)
    if b > a:
        parts = phsp_integrate(expr, spec, mother, b - a, key, arg_builder, rng=rng,
                               row_offset=a, return_partials=True)
    else:
        parts = _lib.empty(0)
    full = gather_partials(parts, n_total, 5, group)
    tot = _lib.fold(full, (n_total + CHUNK - 1) // CHUNK, 5)
    return _finish_average(tot.cpu().numpy(), n_total)


def shard_rows(store, rank: int, world: int):
    """The rank's contiguous row range of a store, as a zero-copy device view
    (the C4 layout: the data set split by row range once, resident per GPU)."""
    from .store import ColumnStore  # noqa: PLC0415
    a, b = shard_range(len(store), rank, world)
    cols = [store.device_column(name)[a:b] for name in store.schema.names]
    return ColumnStore._from_device(store.schema, cols), a


def combine_nll_parts(parts, expected_total: float) -> float:
    """Fold per-rank (event log-sum, global first-bad row or -1, its density)
    triples in rank order: deterministic for a fixed GPU count.  The smallest
    bad row wins, as in the reference (fitting.py:200-205)."""
    import numpy as np  # noqa: PLC0415
    bad = [(int(row), val) for _, row, val in parts if row >= 0]
    if bad:
        row, val = min(bad)
        raise ValueError(f"model density {np.float64(val)!r} is not positive at event {row}")
    total = 0.0
    for logsum, _, _ in parts:
        total += logsum
    return expected_total - total


def sharded_nll(model, shard, observable_columns, row_offset: int, group=None) -> float:
    """nll (fitting.py:175-210) over a data set split by row range across the
    process group: each rank runs the fused FCN pass over its resident rows,
    then one all-gather of 3 doubles per rank and the same rank-order fold on
    every rank, so all ranks return the same value (a minimiser can run in
    lock-step on every rank).  `row_offset` is the shard's first global row,
    so a bad event is reported by its global index."""
    from .fitting import nll_event_sum  # noqa: PLC0415
    rank, world = dist_info(group)
    if len(shard):
        logsum, first, val = nll_event_sum(model, shard, observable_columns)
    else:
        logsum, first, val = 0.0, None, None
    if world == 1:
        if first is not None:
            raise ValueError(f"model density {val!r} is not positive at event {row_offset + first}")
        return model.expected_total() - logsum
    mine = (logsum, -1.0 if first is None else float(row_offset + first), 0.0 if val is None else float(val))
    torch = _lib.torch()
    dist = torch.distributed
    dev = _lib.device() if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor(mine, dtype=torch.float64, device=dev)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    parts = torch.stack(out).cpu().tolist()
    return combine_nll_parts([tuple(p) for p in parts], model.expected_total())
