"""Multi-process (world size 2, gloo, CPU) coverage of the N>1 host logic:
chunk-aligned shards and the all-gather of per-chunk partials into global
chunk order (paper_1711_05683_b200/parallel.py).  The GPU box has one GPU,
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


def _partials_for(a: int, b: int, width: int) -> np.ndarray:
    """Deterministic fake partials: value encodes (global chunk, slot)."""
    from paper_1711_05683_b200.parallel import CHUNK
    chunks = range(a // CHUNK, (b + CHUNK - 1) // CHUNK)
    return np.array([[c * 10.0 + w for w in range(width)] for c in chunks], dtype=np.float64).ravel()


def _worker(rank: int, world: int, port: int, n_total: int, width: int, out_dir: str) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_05683_b200.parallel import dist_info, gather_partials, shard_range
        r, w = dist_info()
        assert (r, w) == (rank, world)
        a, b = shard_range(n_total, rank, world)
        local = torch.from_numpy(_partials_for(a, b, width))
        full = gather_partials(local, n_total, width).numpy()
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), full)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [1, 4096 * 5, 4096 * 7 + 3, 1_000_003])
def test_gather_partials_global_order(tmp_path, n_total):
    from paper_1711_05683_b200.parallel import CHUNK
    world, width = 2, 5
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, n_total, width, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    want = _partials_for(0, n_total, width)
    nch = (n_total + CHUNK - 1) // CHUNK
    assert want.size == nch * width
    for rank in range(world):
        got = np.load(tmp_path / f"rank{rank}.npy")
        assert np.array_equal(got, want), rank


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
    and the first non-positive row of the shard."""
    d = shard.x
    bad = np.flatnonzero(~(d > 0))
    if bad.size:
        return 0.0, int(bad[0]), np.float64(d[bad[0]])
    return float(np.sum(np.log(d))), None, None


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


@pytest.mark.parametrize("case", ["clean", "bad"])
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
    port = _free_port()
    mp.start_processes(_nll_worker, args=(world, port, dens, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    got = [tuple(np.load(tmp_path / f"nll{r}.npy", allow_pickle=True)) for r in range(world)]
    assert got[0] == got[1]
    if case == "bad":
        assert got[0] == ("err", "model density np.float64(-1.0) is not positive at event 100")
        return
    parts = []
    for r in range(world):
        a, b = shard_range(len(dens), r, world)
        parts.append((float(np.sum(np.log(dens[a:b]))), -1.0, 0.0))
    assert got[0] == ("ok", combine_nll_parts(parts, 123.5))
    assert got[0][1] == pytest.approx(123.5 - float(np.sum(np.log(dens))), rel=1e-12)
