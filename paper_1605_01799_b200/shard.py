"""Data-parallel sharding of query points across ranks (one process per GPU).

The Hopf evaluations are independent per point ("totally parallelizable", PAPER.md P:47-48;
the paper's 16-core runs share nothing), so the only parallel strategy is to
split the M points into contiguous shards by global index.  Inputs are regenerated on every
rank from (seed, global index) (inputs.py), so no data moves before the solve; the only
collective is the optional gather of results (phi, iters, and grad on request) after it.
"""
from __future__ import annotations


def shard_range(M: int, world: int, rank: int) -> tuple[int, int]:
    """[r0, r1) of rank `rank` when M points are split into `world` contiguous shards
    (rank r owns [floor(r M / P), floor((r+1) M / P)))."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} of world {world}")
    return (M * rank) // world, (M * (rank + 1)) // world


def weak_range(M_per_rank: int, rank: int) -> tuple[int, int]:
    """[r0, r1) for weak scaling: every rank owns M_per_rank points of a global set."""
    return rank * M_per_rank, (rank + 1) * M_per_rank


def gather_results(tensors, group=None, dst_all=True):
    """Gather per-rank result shards (equal or unequal lengths along dim 0) into full tensors.

    Uses torch.distributed (NCCL on GPUs, gloo on CPU).  Shards may have different lengths:
    lengths are exchanged first, shards are padded to the maximum, gathered, and trimmed.
    Returns the concatenation in rank order (on every rank when dst_all, else only rank 0
    gets the data and other ranks get None)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = tensors[0].device
    n_local = torch.tensor([tensors[0].shape[0]], device=dev, dtype=torch.int64)
    lens = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(lens, n_local, group=group)
    lens = [int(x.item()) for x in lens]
    mx = max(lens)
    out = []
    for t in tensors:
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
        pad[: t.shape[0]] = t
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        full = torch.cat([p[:l] for p, l in zip(parts, lens)], dim=0)
        out.append(full if (dst_all or dist.get_rank(group) == 0) else None)
    return out
