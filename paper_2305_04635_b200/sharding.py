"""Batch partitioning across ranks (one process per GPU) for the batched band solver.

BASELINE.json config C5 partitions a fixed batch of 1,024 independent systems over 1/2/4/8
GPUs with no collective on the data path: strong scaling, rank r of N
owns `shard(1024, r, N)` (1024/N matrices, global seeds).  `gather_rows` is the optional
gather of per-rank results (e.g. the solutions x) onto every rank, over whatever process
group torch.distributed was initialised with (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations


def shard(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous partition: rank r gets [lo, hi); sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of world {world}")
    if batch < 0:
        raise ValueError("batch must be non-negative")
    return (batch * rank) // world, (batch * (rank + 1)) // world


def gather_rows(local, batch: int, world: int, rank: int):
    """All-gather row blocks (local: [hi-lo, ...] tensor) into the full [batch, ...] tensor.

    Shards may differ in size by one, so every rank pads to the largest shard before the
    collective and the padding is dropped afterwards."""
    import torch
    import torch.distributed as dist

    sizes = [shard(batch, r, world)[1] - shard(batch, r, world)[0] for r in range(world)]
    cap = max(sizes) if sizes else 0
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)
