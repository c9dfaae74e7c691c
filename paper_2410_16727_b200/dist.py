"""Multi-GPU plumbing for the seeding path: contiguous problem shards per rank and a
single gather of the results to rank 0.  Problems are independent,
so there is no other collective; inputs and noise are keyed by the GLOBAL problem
index, which makes results bitwise identical for any world size.

Strong scaling (BASELINE config 3: "1024 problems ... sharded evenly across 1/2/4/8 GPUs"):
rank r owns global problems [r*P/N, (r+1)*P/N) of a fixed total P.  Weak scaling (every rank
plans its own fixed-size block) is kept as an option for the config-4 sweep.
"""

from __future__ import annotations


def shard(rank: int, world: int, problems_per_rank: int):
    """Weak scaling: rank r owns global problems [r*P, (r+1)*P)."""
    p0 = rank * problems_per_rank
    return p0, p0 + problems_per_rank


def shard_even(rank: int, world: int, total: int):
    """Strong scaling: an even split of `total` problems, rank r owns [r*total//N, (r+1)*total//N)
    (shards differ by at most one problem)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    return rank * total // world, (rank + 1) * total // world


def gather_to_rank0(tensors, rank: int, world: int, group=None, counts=None):
    """Gather per-rank tensors (dim 0 = the rank's rows) to rank 0; returns the concatenations on
    rank 0 (in rank order) and None elsewhere.  `counts[i]` = rows rank i holds for each tensor
    (list per tensor, or None when every rank holds the same number): uneven shards are padded to
    the largest for the collective and trimmed on rank 0.  Works with NCCL (CUDA tensors) and
    gloo (CPU tensors)."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return list(tensors)
    out = []
    for i, t in enumerate(tensors):
        t = t.contiguous()
        cnt = None if counts is None else counts[i]
        if cnt is not None and max(cnt) != t.shape[0]:
            pad = torch.zeros((max(cnt) - t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            t = torch.cat([t, pad])
        if rank == 0:
            bufs = [torch.empty_like(t) for _ in range(world)]
            dist.gather(t, bufs, dst=0, group=group)
            if cnt is not None:
                bufs = [b[:c] for b, c in zip(bufs, cnt)]
            out.append(torch.cat(bufs, dim=0))
        else:
            dist.gather(t, None, dst=0, group=group)
    return out if rank == 0 else None


def plan_sharded(planner, images, q_start, goal, boxes, p0: int, rank: int, world: int, total: int,
                 group=None):
    """The multi-GPU planning call: this rank's shard (problems [p0, p0 + len(q_start)) of `total`)
    from host arrays through BLPlanner.plan_batch_device, the single gather of trajectories, costs,
    feasibility flags and best-seed indices to rank 0, and rank 0's read-back of the whole job.
    Returns a PlanBatchResult of host tensors on rank 0 (None elsewhere)."""
    import torch

    from .planner import PlanBatchResult

    d = planner.upload(images, q_start, goal, boxes)
    r = planner.plan_batch_device(*d, p0=p0, images_ready=planner._img_chunks)
    S = planner.S
    per = [(rr + 1) * total // world - rr * total // world for rr in range(world)]
    cnt = [[n * S for n in per]] * 3 + [per]
    g = gather_to_rank0([r.trajectories, r.cost, r.feasible, r.best_index], rank, world, group, counts=cnt)
    if rank != 0:
        torch.cuda.current_stream().synchronize()
        return None
    host = [x.to("cpu", non_blocking=True) for x in g]
    torch.cuda.current_stream().synchronize()
    return PlanBatchResult(host[0], None, host[1], host[2], None, host[3])
