"""Deterministic data parallelism across GPUs (reference parallel.py:1-92).

The reference splits every bulk operation into fixed 65 536-row batches and
4096-row chunk partials folded in a fixed order, so results do not depend on
the worker count.  Here the "workers" are GPUs, one process per GPU
(torch.distributed, NCCL over NVLink/NVSwitch), and the exchange follows
SURVEY.md 8(e) option (ii):

* a run's chunks are cut into HK_SUPERS = 1024 fixed super-chunks
  (``_lib.super_chunks``); rank r of W owns supers [1024 r / W, 1024 (r+1) / W)
  and so a contiguous, chunk-aligned row range (``shard_range``).  Each rank
  generates/evaluates its range with the *global* row index, so shards are
  bit-identical to the same rows of a one-GPU run (RNG counters are global,
  phasespace.py:105-109);
* each rank folds its chunk partials into one record per super-chunk on the
  device (hk_fold_supers), and the only exchange is those records:
  ``gather_supers`` all-gathers 1024 x width doubles (40 KB for the 5-wide
  averages, whatever the event count), and every rank folds the same array
  with the same fixed tree.  A one-GPU total (``_lib.total``) runs the same
  two levels, so every reduced value is bitwise independent of the GPU count
  (the analogue of the reference's worker-invariance tests,
  test_phasespace.py:87-93, test_fitting.py:120-124);
* per-rank error rows travel with the records, so a bad event on one rank
  raises the same exception on every rank instead of leaving the others
  waiting in the collective.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib

CHUNK = _lib.HK_CHUNK          # parallel.py:18
EVAL_BATCH = 16 * CHUNK        # parallel.py:21
SUPERS = _lib.HK_SUPERS


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


def super_span(rank: int, world: int) -> tuple[int, int]:
    """Super-chunks [s0, s1) owned by `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return SUPERS * rank // world, SUPERS * (rank + 1) // world


def shard_range(n: int, rank: int, world: int, chunk: int = CHUNK) -> tuple[int, int]:
    """Contiguous chunk-aligned [a, b) of rank's rows: the rows of its
    super-chunks.  Shards cover [0, n); for world | 1024 this is the even
    chunk split [N r / W, N (r+1) / W) chunks."""
    if chunk != CHUNK:
        raise ValueError(f"shards are cut on {CHUNK}-row chunks")
    s0, s1 = super_span(rank, world)
    c0, c1 = _lib.super_chunks(n, s0, s1)
    return min(c0 * chunk, n), min(c1 * chunk, n)


def dist_info(group=None) -> tuple[int, int]:
    """(rank, world) of the default process group, (0, 1) when not initialised."""
    torch = _lib.torch()
    dist = torch.distributed
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def _all_gather_padded(local, sizes: list[int], group=None) -> list:
    """All-gather 1-D tensors of the given per-rank sizes; returns the ranks'
    tensors (on local's device) in rank order.  NCCL gathers device tensors in
    place; CPU backends (gloo) go through host memory."""
    torch = _lib.torch()
    dist = torch.distributed
    rank, world = dist_info(group)
    if local.numel() != sizes[rank]:
        raise ValueError(f"rank {rank} holds {local.numel()} values, the layout expects {sizes[rank]}")
    dev = local.device if dist.get_backend(group) == "nccl" else "cpu"
    cap = max(sizes)
    if all(sz == cap for sz in sizes):
        buf = local.to(dev).contiguous()
    else:
        buf = torch.zeros(cap, dtype=local.dtype, device=dev)
        buf[: local.numel()] = local.to(dev)
    out = torch.empty(world * cap, dtype=local.dtype, device=dev)
    dist.all_gather_into_tensor(out, buf, group=group)
    return [out[r * cap: r * cap + sizes[r]].to(local.device) for r in range(world)]


def gather_supers(local, width: int, group=None, extra=None):
    """All-gather this rank's super-chunk records (flat, (s1 - s0) x width)
    into global super order on every rank: (1024 x width tensor, and with
    `extra` -- a small per-rank float64 vector such as error rows -- the
    ranks' extras as a (world, len) numpy array)."""
    torch = _lib.torch()
    rank, world = dist_info(group)
    k = 0 if extra is None else len(extra)
    if world == 1:
        ex = None if extra is None else np.asarray(extra, dtype=np.float64).reshape(1, k)
        return local, ex
    sizes = [(b - a) * width + k for a, b in (super_span(r, world) for r in range(world))]
    mine = local
    if k:
        mine = torch.cat([local, torch.tensor(list(extra), dtype=torch.float64, device=local.device)])
    parts = _all_gather_padded(mine, sizes, group)
    full = torch.cat([p[: p.numel() - k] for p in parts])
    ex = None
    if k:
        ex = torch.stack([p[p.numel() - k:] for p in parts]).cpu().numpy()
    return full, ex


def _min_row(rows) -> int:
    """Smallest valid global row among float-encoded rows (-1 = none)."""
    valid = [int(r) for r in rows if r >= 0]
    return min(valid) if valid else _lib.HK_NO_BAD_ROW


def sharded_weight_moments(block_shard, n_total: int, group=None):
    """Global (sum w, sum w^2) of a sharded generation (device tensor of 2):
    the shard's warp-slice partials -> its super-chunk records -> gather ->
    the same fixed fold on every rank.  An empty shard contributes zero
    records.  Equal bit for bit to phsp_weight_moments of the one-GPU run."""
    from .phasespace import _weight_partials  # noqa: PLC0415
    rank, world = dist_info(group)
    a, b = shard_range(n_total, rank, world)
    if len(block_shard) != b - a:
        raise ValueError(f"rank {rank} shard holds {len(block_shard)} rows, shard_range gives {b - a}")
    parts = _weight_partials(block_shard)
    if parts is None and b > a:
        raise ValueError("the shard carries no fused weight partials (generate it with phsp_generate)")
    s0, s1 = super_span(rank, world)
    local = _lib.fold_supers(parts, n_total, s0, s1, _lib.HK_WARP_SLICES, 2)
    full, _ = gather_supers(local, 2, group)
    return _lib.fold(full, SUPERS, 2)


def sharded_integrate(expr, spec, mother, n_total: int, key, arg_builder, group=None,
                      rng: str = "reference"):
    """phsp_integrate over n_total events sharded across the process group
    (config C5 at 1/2/4/8 GPUs); returns the IntegrationResult on every rank,
    bitwise the same for any GPU count.  The first bad rows of every rank
    ride along with the super records, so all ranks raise the reference's
    exception for the globally first bad event together."""
    from .phasespace import _finish_average, _IntegrateRun  # noqa: PLC0415

    n_total = int(n_total)
    if n_total == 0:
        raise ValueError("cannot average over an empty block")
    rank, world = dist_info(group)
    a, b = shard_range(n_total, rank, world)
    run = _IntegrateRun(expr, spec, mother, key, arg_builder, rng)
    parts, flags = run.partials(b - a, a)
    s0, s1 = super_span(rank, world)
    local = _lib.fold_supers(parts, n_total, s0, s1, 1, 5)
    rows = [-1.0 if f == _lib.HK_NO_BAD_ROW else float(f) for f in flags]
    full, ex = gather_supers(local, 5, group, extra=rows)
    run.raise_error([_min_row(ex[:, 0]), _min_row(ex[:, 1])])
    tot = _lib.fold(full, SUPERS, 5)
    return _finish_average(tot.cpu().numpy(), n_total)


def shard_rows(store, rank: int, world: int):
    """The rank's contiguous row range of a store, as a zero-copy device view
    (the C4 layout: the data set split by row range once, resident per GPU)."""
    from .store import ColumnStore  # noqa: PLC0415
    a, b = shard_range(len(store), rank, world)
    cols = [store.device_column(name)[a:b] for name in store.schema.names]
    return ColumnStore._from_device(store.schema, cols), a


_PART = 3 + _lib.HK_FCN_MAX_OBS   # host-path record: logsum, global row (-1), kind, payload
_OFFSET_SET: dict = {}             # id(FCN workspace) -> (its pointer, the row offset written into [6])
_GATHERED: dict = {}               # (device, stream, world, group) -> the all-gather target of the FCN records


def combine_nll_parts(parts, expected_total: float) -> float:
    """Fold per-rank records (event log-sum, global problem row or -1, kind,
    payload...) in rank order: deterministic for a fixed GPU count.  The
    problem the reference would raise wins (fitting.first_problem: earliest
    batch, zero divisor before density, smallest row)."""
    from .fitting import DIV0, EVAL_BATCH_ROWS, fcn_exception  # noqa: PLC0415
    probs = [(int(p[1]) // EVAL_BATCH_ROWS, int(p[2]), int(p[1]), p) for p in parts if p[1] >= 0]
    if probs:
        _, kind, row, p = min(probs, key=lambda t: t[:3])
        if kind == DIV0:
            payload = tuple(np.float64(v) for v in p[3:3 + int(p[-1])])
        else:
            payload = np.float64(p[3])
        raise fcn_exception(row, kind, payload)
    total = 0.0
    for p in parts:
        total += p[0]
    return expected_total - total


def sharded_nll(model, shard, observable_columns, row_offset: int, group=None,
                _force_collective: bool = False) -> float:
    """nll (fitting.py:175-210) over a data set split by row range across the
    process group; every rank returns the same value (a minimiser can run in
    lock-step on every rank).  `row_offset` is the shard's first global row,
    so a bad event is reported by its global index.

    Over NCCL one evaluation is: the fused FCN pass enqueued without waiting
    (fitting.nll_event_launch), one stream-ordered all-gather of each rank's
    8-double record, and hk_nll_combine -- a kernel that folds the records in
    rank order and publishes the result into mapped host memory -- so the
    host synchronises once.  Other backends (gloo: the CPU tests of this
    logic) exchange the same records through host memory."""
    from . import fitting  # noqa: PLC0415
    rank, world = dist_info(group)
    if world == 1 and not _force_collective:   # (forced: test hook for a 1-rank NCCL group)
        logsum, problem = fitting.nll_event_sum(model, shard, observable_columns) if len(shard) else (0.0, None)
        if problem is not None:
            row, kind, payload = problem
            raise fitting.fcn_exception(row_offset + row, kind, payload)
        return model.expected_total() - logsum
    torch = _lib.torch()
    dist = torch.distributed
    if dist.get_backend(group) != "nccl":
        return _sharded_nll_host(model, shard, observable_columns, row_offset, group)
    none = np.array([-1], dtype=np.int64).view(np.float64)[0]
    if len(shard):
        work = fitting.nll_event_launch(model, shard, observable_columns)
        # [6] = the shard's first global row: the kernel never writes it, so it
        # is set once per workspace and offset (a device write costs a launch)
        if _OFFSET_SET.get(id(work)) != (work.data_ptr(), row_offset):
            work[6] = float(row_offset)
            _OFFSET_SET[id(work)] = (work.data_ptr(), row_offset)
        rec = work[:8]
    else:
        rec = torch.from_numpy(np.array([0.0, none, 0, 0, 0, none, float(row_offset), 0.0])).to(_lib.device())
    key = (rec.device.index, _lib.stream_ptr(), world, id(group))
    gathered = _GATHERED.get(key)
    if gathered is None:   # the gather target is reused: stream-ordered, read by the combine kernel
        gathered = _GATHERED[key] = torch.empty(world * 8, dtype=torch.float64, device=rec.device)
    dist.all_gather_into_tensor(gathered, rec, group=group)
    logsum = _lib.ctypes.c_double()
    bad, zero = _lib.ctypes.c_uint64(), _lib.ctypes.c_uint64()
    _lib.check(_lib.lib().hk_nll_combine(gathered.data_ptr(), world, _lib.ctypes.byref(logsum),
                                         _lib.ctypes.byref(bad), _lib.ctypes.byref(zero), _lib.stream_ptr()),
               "hk_nll_combine")
    problem = fitting.first_problem(zero.value, bad.value)
    if problem is None:
        return model.expected_total() - logsum.value
    # slow path: the owning rank computes the message payload, everyone raises
    row, kind = problem
    mine = np.zeros(2 + _lib.HK_FCN_MAX_OBS)
    if row_offset <= row < row_offset + len(shard):
        pay = fitting.problem_payload(model, shard, observable_columns, row - row_offset, kind)
        vals = list(pay) if kind == fitting.DIV0 else [float(pay)]
        mine[0], mine[1] = 1.0, len(vals)
        mine[2:2 + len(vals)] = vals
    recs = torch.empty(world * mine.size, dtype=torch.float64, device=rec.device)
    dist.all_gather_into_tensor(recs, torch.from_numpy(mine).to(rec.device), group=group)
    owner = next(r for r in recs.view(world, -1).cpu().numpy() if r[0] == 1.0)
    vals = owner[2:2 + int(owner[1])]
    payload = tuple(np.float64(v) for v in vals) if kind == fitting.DIV0 else np.float64(vals[0])
    raise fitting.fcn_exception(row, kind, payload)


def _sharded_nll_host(model, shard, observable_columns, row_offset: int, group=None) -> float:
    from . import fitting  # noqa: PLC0415
    torch = _lib.torch()
    dist = torch.distributed
    _, world = dist_info(group)
    rec = np.zeros(_PART + 1)
    rec[1] = -1.0
    if len(shard):
        logsum, problem = fitting.nll_event_sum(model, shard, observable_columns)
        rec[0] = logsum
        if problem is not None:
            row, kind, payload = problem
            vals = list(payload) if kind == fitting.DIV0 else [float(payload)]
            rec[1], rec[2] = float(row_offset + row), float(kind)
            rec[3:3 + len(vals)] = vals
            rec[-1] = len(vals)
    t = torch.from_numpy(rec)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return combine_nll_parts([o.numpy() for o in out], model.expected_total())
