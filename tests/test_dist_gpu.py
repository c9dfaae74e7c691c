"""World-size invariance of the REAL planner (BLPlanner, bf16 tcgen05 sampler + refinement):
two ranks over gloo on one GPU, each planning its even shard of the problems (strong scaling,
dist.shard_even), gathered to rank 0, must equal one process planning every problem, bit for bit
(the reference's worker-count invariance, planseed tests/test_data.py:220-226).  The ranks never
wait on each other's kernels: each rank's GPU work completes before the gloo gather of host copies.
The ranks take turns on the GPU (a barrier between them): run concurrently on ONE device, the
cooperative persistent sampler may find the SMs held by the other process and fall back to the
layered kernels, whose bf16 results differ at the rounding level -- a property of sharing one
GPU, not of the sharding.  Both sampler paths are checked (PS_PERSIST=1 / 0)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOTAL, S = 5, 32          # uneven: rank 0 plans 2 problems, rank 1 plans 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _plan(P, p0):
    from paper_2410_16727_b200 import spec, synth
    from paper_2410_16727_b200.planner import BLPlanner
    params = spec.random_model(spec.ENCODER_CFG3)
    pl = BLPlanner(params, spec.ENCODER_CFG3, mode=1, S=S, max_problems=max(P, 1))
    pb = synth.config3_problems(P, p0=p0, seed=0)
    r = pl.plan_batch(pb.images, pb.q_start, pb.goal, pb.boxes, p0=p0)
    return r


def _worker(rank, world, port, q, persist):
    import torch
    import torch.distributed as dist

    from paper_2410_16727_b200 import dist as psd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), PS_PERSIST=persist)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p0, p1 = psd.shard_even(rank, world, TOTAL)
    per = [psd.shard_even(r, world, TOTAL)[1] - psd.shard_even(r, world, TOTAL)[0] for r in range(world)]
    for turn in range(world):
        if turn == rank:
            r = _plan(p1 - p0, p0)
        dist.barrier()
    cnt = [[n * S for n in per]] * 3 + [per]
    g = psd.gather_to_rank0([r.trajectories, r.cost, r.feasible, r.best_index], rank, world, counts=cnt)
    if rank == 0:
        q.put([x.numpy() for x in g])
    dist.destroy_process_group()


@pytest.mark.parametrize("persist", ["1", "0"])
def test_two_ranks_equal_single_process(persist):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.fail("GPU test without a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, persist)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    os.environ["PS_PERSIST"] = persist
    try:
        want = _plan(TOTAL, 0)
    finally:
        os.environ.pop("PS_PERSIST", None)
    for g, w, name in zip(got, (want.trajectories, want.cost, want.feasible, want.best_index),
                          ("trajectories", "cost", "feasible", "best_index")):
        assert np.array_equal(g, np.asarray(w)), name
