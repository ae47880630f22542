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
