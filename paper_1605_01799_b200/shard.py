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

    One all_gather_into_tensor per result (ncclAllGather on GPUs, gloo on CPU) into a
    [world * max_len, ...] buffer; unequal shard lengths are exchanged first and the padding is
    trimmed.  Returns the concatenation in rank order (on every rank when dst_all, else only
    rank 0 gets the data and other ranks get None)."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "gloo" and tensors[0].is_cuda:
        # gloo gathers host tensors: round-trip through the host (tests, CPU fallbacks of the
        # process group; the GPU path is NCCL)
        out = gather_results([t.cpu() for t in tensors], group, dst_all)
        return [None if o is None else o.to(tensors[0].device) for o in out]
    world = dist.get_world_size(group)
    dev = tensors[0].device
    n_local = torch.tensor([tensors[0].shape[0]], device=dev, dtype=torch.int64)
    lens_t = torch.empty(world, device=dev, dtype=torch.int64)
    dist.all_gather_into_tensor(lens_t, n_local, group=group)
    lens = [int(x) for x in lens_t.tolist()]
    mx = max(lens)
    out = []
    for t in tensors:
        src = t.contiguous()
        if t.shape[0] != mx:
            src = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
            src[: t.shape[0]] = t
        buf = torch.empty((world * mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
        dist.all_gather_into_tensor(buf, src, group=group)
        if any(l != mx for l in lens):
            buf = torch.cat([buf[r * mx: r * mx + l] for r, l in enumerate(lens)], dim=0)
        out.append(buf if (dst_all or dist.get_rank(group) == 0) else None)
    return out


def eval_gather_pipelined(eval_chunk, n_local, chunk, outs_full, group=None):
    """Evaluate this rank's n_local points chunk by chunk and all-gather each chunk's results
    while the next chunk computes (the gather overlapped with compute).

    eval_chunk(lo, hi) enqueues the evaluation of local points [lo, hi) on the current stream
    and returns its result tensors (rows lo..hi of the local outputs).  outs_full[k] has shape
    [world * n_local, ...] (rank-major, equal shard sizes, as in weak scaling) and receives
    result k of every rank.  Each chunk's collectives are issued asynchronously after its
    kernels are enqueued, so NCCL runs them on its own stream (ordered after that chunk's
    kernels) concurrently with the next chunk's kernels; the chunk's rows are scattered into
    place when it lands.  Returns after every chunk is in outs_full (host not blocked on the
    device except through the final waits)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    host = dist.get_backend(group) == "gloo"   # gloo gathers host copies
    pending = []

    def land(item):
        lo, hi, works, bufs = item
        for w in works:
            w.wait()
        for full, buf in zip(outs_full, bufs):
            full.view((world, n_local) + tuple(full.shape[1:]))[:, lo:hi] = \
                buf.view((world, hi - lo) + tuple(buf.shape[1:])).to(full.device)

    for lo in range(0, n_local, chunk):
        hi = min(n_local, lo + chunk)
        res = eval_chunk(lo, hi)
        works, bufs = [], []
        for t in res:
            src = t.cpu() if host else t.contiguous()
            buf = torch.empty((world * (hi - lo),) + tuple(t.shape[1:]), dtype=t.dtype, device=src.device)
            works.append(dist.all_gather_into_tensor(buf, src.contiguous(), group=group, async_op=True))
            bufs.append(buf)
        pending.append((lo, hi, works, bufs))
        if len(pending) > 1:
            land(pending.pop(0))
    while pending:
        land(pending.pop(0))
    return outs_full
