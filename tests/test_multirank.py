"""Two-rank (gloo, CPU) test of the batch partitioning used by the multi-GPU bench.

Each rank solves its contiguous shard of a small batch with the CPU oracle (the
checker -- no GPU here), then the solutions are gathered; the result must equal the
single-process answer in order, and the shards must tile the batch exactly once.
"""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_04635_b200.inputs import generate_spd, make_rhs
from paper_2305_04635_b200.sharding import gather_rows, shard


def test_shard_tiles_batch():
    for batch in (0, 1, 7, 1024, 1025):
        for world in (1, 2, 3, 4, 8):
            covered = []
            for r in range(world):
                lo, hi = shard(batch, r, world)
                assert 0 <= lo <= hi <= batch
                covered.extend(range(lo, hi))
            assert covered == list(range(batch))
            sizes = [shard(batch, r, world)[1] - shard(batch, r, world)[0] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _worker(rank, world, port, batch, n, k, out):
    from oracle import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard(batch, rank, world)
    xs = []
    for s in range(lo, hi):
        a = generate_spd(n, k, s)
        oracle.factor_plain(n, k, k + 1, a.data)
        xs.append(oracle.solve(n, k, k + 1, a.data, make_rhs(n, s)))
    local = torch.from_numpy(np.stack(xs)) if xs else torch.zeros((0, n), dtype=torch.float64)
    full = gather_rows(local, batch, world, rank)
    if rank == 0:
        out.put(full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_matches_single_process():
    from oracle import oracle
    batch, n, k, world = 7, 60, 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, batch, n, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for s in range(batch):
        a = generate_spd(n, k, s)
        oracle.factor_plain(n, k, k + 1, a.data)
        want = oracle.solve(n, k, k + 1, a.data, make_rhs(n, s))
        assert np.array_equal(full[s], want)


def _strong_worker(rank, world, port, batch, n, k, out):
    """The bench's multi-GPU flow on CPU: rank r owns shard(batch, r, world) of ONE fixed global
    batch, factors + solves it (the oracle stands in for the GPU), and the max-over-ranks
    reduction picks the job time; the gathered x equals the single-process answer."""
    import time

    from oracle import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard(batch, rank, world)
    t0 = time.perf_counter()
    xs = []
    for s in range(lo, hi):
        a = generate_spd(n, k, s)
        oracle.factor_plain(n, k, k + 1, a.data)
        xs.append(oracle.solve(n, k, k + 1, a.data, make_rhs(n, s)))
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    local = torch.from_numpy(np.stack(xs)) if xs else torch.zeros((0, n), dtype=torch.float64)
    full = gather_rows(local, batch, world, rank)
    if rank == 0:
        out.put((hi - lo, float(t.item()), full.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_strong_split_of_a_fixed_batch():
    from oracle import oracle
    batch, n, k, world = 16, 80, 6, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_strong_worker, args=(r, world, port, batch, n, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    mine, tmax, full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert mine == batch // world and tmax > 0.0
    assert full.shape == (batch, n)
    for s in range(batch):
        a = generate_spd(n, k, s)
        oracle.factor_plain(n, k, k + 1, a.data)
        assert np.array_equal(full[s], oracle.solve(n, k, k + 1, a.data, make_rhs(n, s)))
