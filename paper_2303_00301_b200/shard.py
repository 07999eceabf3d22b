"""Multi-GPU plumbing for the sampler: chains are independent, so N > 1 shards
chains across ranks (one process per GPU) with no data-path collective.

A chain is identified only by its global index c: its root stream is
from_seed(seed).derive(kChain, c) (runner.cpp:132), so chain c produces the same
draws whichever rank runs it.  The only collectives are the timing reduction
(max over ranks) and, for callers that want them on one rank, result gathers.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    first: int  # global index of this rank's first chain
    count: int  # chains on this rank


def weak_shard(rank: int, world: int, per_rank: int) -> Shard:
    """Weak scaling: every rank runs `per_rank` chains, [rank*per_rank, (rank+1)*per_rank)."""
    if not 0 <= rank < world or per_rank < 0:
        raise ValueError(f"bad shard request rank={rank} world={world} per_rank={per_rank}")
    return Shard(rank, world, rank * per_rank, per_rank)


def strong_shard(rank: int, world: int, total: int) -> Shard:
    """Strong scaling: `total` chains split into contiguous, balanced ranges
    (the first total % world ranks take one extra chain)."""
    if not 0 <= rank < world or total < 0:
        raise ValueError(f"bad shard request rank={rank} world={world} total={total}")
    base, extra = divmod(total, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return Shard(rank, world, first, count)


def dist_env():
    """(rank, world, local_rank) from the torchrun environment (1 process if unset)."""
    import os
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def max_over_ranks(value: float, world: int, device="cpu") -> float:
    """All-reduce MAX of one float across the process group (NCCL tensors live on
    the rank's GPU, gloo tensors on the host)."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(t, world: int):
    """All-gather equally shaped per-rank tensors along dim 0 (rank order)."""
    if world <= 1:
        return t
    import torch
    import torch.distributed as dist
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t.contiguous())
    return torch.cat(parts, 0)
