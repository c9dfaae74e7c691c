"""Multi-GPU plumbing for the seeding path: contiguous problem shards per rank and a
single gather of the results to rank 0.  Problems are independent,
so there is no other collective; inputs and noise are keyed by the GLOBAL problem
index, which makes results bitwise identical for any world size."""

from __future__ import annotations


def shard(rank: int, world: int, problems_per_rank: int):
    """Weak scaling: rank r owns global problems [r*P, (r+1)*P)."""
    p0 = rank * problems_per_rank
    return p0, p0 + problems_per_rank


def gather_to_rank0(tensors, rank: int, world: int, group=None):
    """Gather equally shaped per-rank tensors to rank 0; returns the concatenations on
    rank 0 (in rank order) and None elsewhere.  Works with NCCL (CUDA tensors) and gloo
    (CPU tensors)."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return list(tensors)
    out = []
    for t in tensors:
        t = t.contiguous()
        if rank == 0:
            bufs = [torch.empty_like(t) for _ in range(world)]
            dist.gather(t, bufs, dst=0, group=group)
            out.append(torch.cat(bufs, dim=0))
        else:
            dist.gather(t, None, dst=0, group=group)
    return out if rank == 0 else None
