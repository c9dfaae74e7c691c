"""World-size invariance of the sharded pipeline plumbing on CPU (gloo, world size 2):
the per-rank shards generate exactly the problems a single process generates, and the
gather reassembles per-trajectory results in global order (the analogue of
planseed's worker-count invariance test, tests/test_data.py:220-226)."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_16727_b200 import dist as psd
from paper_2410_16727_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _surrogate(pb, S):
    # deterministic per-problem stand-in for the device pipeline's outputs
    traj = np.repeat(pb.q_start[:, None, None, :], S, axis=1) + pb.boxes[:, :S, None, :1].sum(-1)[..., None] * 0
    cost = pb.boxes.sum(axis=(1, 2)).repeat(S).astype(np.float32)
    best = (pb.q_start.sum(axis=1) * 1000).astype(np.int32) % S
    return torch.as_tensor(traj.reshape(-1, 1, 7).astype(np.float32)), torch.as_tensor(cost), torch.as_tensor(best)


def _worker(rank, world, port, P, S, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p0, p1 = psd.shard(rank, world, P)
    pb = synth.make_problems(p1 - p0, p0=p0, seed=0, image_shape=(16, 16), n_images=2, n_rect=3)
    res = psd.gather_to_rank0(list(_surrogate(pb, S)) + [torch.as_tensor(pb.images)], rank, world)
    if rank == 0:
        q.put([r.numpy() for r in res])
    dist.destroy_process_group()


def test_gloo_world2_matches_single_process():
    P, S, world = 3, 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, P, S, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pb = synth.make_problems(P * world, p0=0, seed=0, image_shape=(16, 16), n_images=2, n_rect=3)
    want = [r.numpy() for r in _surrogate(pb, S)] + [pb.images]
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def test_shard_ranges_cover_global_indices():
    P = 5
    ranges = [psd.shard(r, 4, P) for r in range(4)]
    assert ranges[0] == (0, 5) and ranges[-1] == (15, 20)
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))


def test_shard_even_strong_scaling():
    for total, world in ((1024, 8), (5, 2), (7, 4), (3, 4)):
        r = [psd.shard_even(k, world, total) for k in range(world)]
        assert r[0][0] == 0 and r[-1][1] == total
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        sizes = [b - a for a, b in r]
        assert max(sizes) - min(sizes) <= 1


def _uneven_worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p0, p1 = psd.shard_even(rank, world, total)
    per = [psd.shard_even(r, world, total)[1] - psd.shard_even(r, world, total)[0] for r in range(world)]
    rows = torch.arange(p0, p1, dtype=torch.float32)[:, None].repeat(1, 3)
    res = psd.gather_to_rank0([rows, rows[:, 0].to(torch.int32)], rank, world, counts=[per, per])
    if rank == 0:
        q.put([r.numpy() for r in res])
    dist.destroy_process_group()


def test_gloo_uneven_shards_gather_in_global_order():
    total, world = 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_uneven_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    rows, idx = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(idx, np.arange(total))
    assert np.array_equal(rows, np.repeat(np.arange(total, dtype=np.float32)[:, None], 3, 1))
