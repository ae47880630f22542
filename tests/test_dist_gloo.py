"""Multi-process (world size 2, gloo, CPU) coverage of the N>1 host logic:
super-chunk-aligned shards and the all-gather of super-chunk records into
global order (paper_1711_05683_b200/parallel.py).  The GPU box has one GPU,
so the NCCL path is exercised with the same code under gloo here."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _supers_for(s0: int, s1: int, width: int) -> np.ndarray:
    """Deterministic fake super-chunk records: value encodes (super, slot)."""
    return np.array([[s * 10.0 + w for w in range(width)] for s in range(s0, s1)], dtype=np.float64).ravel()


def _worker(rank: int, world: int, port: int, n_total: int, width: int, out_dir: str) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_05683_b200.parallel import dist_info, gather_supers, shard_range, super_span
        r, w = dist_info()
        assert (r, w) == (rank, world)
        s0, s1 = super_span(rank, world)
        local = torch.from_numpy(_supers_for(s0, s1, width))
        a, b = shard_range(n_total, rank, world)
        full, ex = gather_supers(local, width, extra=[float(a), float(b), -1.0])
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), full.numpy())
        np.save(os.path.join(out_dir, f"extra{rank}.npy"), ex)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("n_total", [1, 4096 * 5, 4096 * 7 + 3, 1_000_003])
def test_gather_supers_global_order(tmp_path, world, n_total):
    """Every rank receives the 1024 super-chunk records in global order (and
    the per-rank extras in rank order), including uneven super spans (world 3)
    and ranks whose row shard is empty (n_total smaller than world chunks)."""
    from paper_1711_05683_b200.parallel import SUPERS, shard_range
    width = 5
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, n_total, width, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    want = _supers_for(0, SUPERS, width)
    shards = np.array([[*shard_range(n_total, r, world), -1.0] for r in range(world)])
    for rank in range(world):
        got = np.load(tmp_path / f"rank{rank}.npy")
        assert np.array_equal(got, want), rank
        assert np.array_equal(np.load(tmp_path / f"extra{rank}.npy"), shards), rank


class _Shard:
    def __init__(self, x):
        self.x = x

    def __len__(self):
        return len(self.x)


class _Model:
    def expected_total(self):
        return 123.5


def _fake_event_sum(model, shard, cols):
    """Host stand-in for the GPU pass (fitting.nll_event_sum): sum of logs
    and the first problem of the shard -- a non-positive density, or (for
    inf entries, standing in for a zero divisor inside a shape) a DIV0."""
    from paper_1711_05683_b200.fitting import DENSITY, DIV0, first_problem
    d = shard.x
    bad = np.flatnonzero(~(d > 0) | np.isnan(d))
    zero = np.flatnonzero(np.isinf(d))
    first = first_problem(int(zero[0]) if zero.size else -1, int(bad[0]) if bad.size else -1)
    if first is None:
        return float(np.sum(np.log(d))), None
    row, kind = first
    payload = (np.float64(d[row]), np.float64(2.0)) if kind == DIV0 else np.float64(d[row])
    return 0.0, (row, kind, payload)


def _nll_worker(rank: int, world: int, port: int, dens: np.ndarray, out_dir: str) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_05683_b200 import fitting, parallel
        fitting.nll_event_sum = _fake_event_sum       # the combine + collective are under test
        a, b = parallel.shard_range(len(dens), rank, world)
        try:
            v = parallel.sharded_nll(_Model(), _Shard(dens[a:b]), ["x0"], a)
            res = ("ok", v)
        except ValueError as exc:
            res = ("err", str(exc))
        np.save(os.path.join(out_dir, f"nll{rank}.npy"), np.array(res, dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["clean", "bad", "div0", "div0_later_batch"])
def test_sharded_nll_combine(tmp_path, case):
    """Row-sharded FCN (parallel.sharded_nll): every rank returns the same
    value, the rank-order sum of the shard log-sums, and a bad density is
    reported by its smallest global row (fitting.py:200-205)."""
    from paper_1711_05683_b200.parallel import combine_nll_parts, shard_range
    world = 2
    rs = np.random.default_rng(1)
    dens = rs.uniform(0.1, 2.0, 3 * 4096 + 17)
    if case == "bad":
        dens[[9000, 8200, 100]] = [0.0, np.nan, -1.0]   # rank 1 holds 8200/9000, rank 0 holds 100
    if case == "div0":
        dens[[9000, 100]] = [np.inf, -1.0]   # same 65536-row batch: the zero divisor (rank 1) wins
    if case == "div0_later_batch":
        dens = np.concatenate([dens, rs.uniform(0.1, 2.0, 70_000)])
        dens[[70_000, 100]] = [np.inf, -1.0]  # the density problem's batch comes first
    port = _free_port()
    mp.start_processes(_nll_worker, args=(world, port, dens, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    got = [tuple(np.load(tmp_path / f"nll{r}.npy", allow_pickle=True)) for r in range(world)]
    assert got[0] == got[1]
    if case in ("bad", "div0_later_batch"):
        assert got[0] == ("err", "model density np.float64(-1.0) is not positive at event 100")
        return
    if case == "div0":
        assert got[0] == ("err", "division by zero at point (np.float64(inf), np.float64(2.0))")
        return
    parts = []
    for r in range(world):
        a, b = shard_range(len(dens), r, world)
        parts.append(np.array([float(np.sum(np.log(dens[a:b]))), -1.0] + [0.0] * 10))
    assert got[0] == ("ok", combine_nll_parts(parts, 123.5))
    assert got[0][1] == pytest.approx(123.5 - float(np.sum(np.log(dens))), rel=1e-12)
