"""planseed-shaped planning entry points for the BASELINE profile.

planseed plans one request at a time: ``plan_diffusion(arm, net, schedule, req, weights,
guidance) -> PlanResult`` (src/pipeline.py:172-209), with ``PlanRequest`` (:37-54) and
``PlanResult`` / ``OptResult`` (:64-94, src/trajopt.py:39-46).  Here the arm, network, schedule
and weights live in a :class:`~paper_2410_16727_b200.planner.BLPlanner` (built once, buffers
preallocated), and ``plan_diffusion_batch(planner, reqs)`` plans a list of requests in ONE
batched GPU call (``BLPlanner.plan_batch``: ESDF build, encoder, sampler, refinement, flags,
select), returning one planseed ``PlanResult`` per request, in order.

Differences from planseed's request, all forced by the BASELINE profile:
  * the observation is the BASELINE depth images, the planner ESDF comes from the scene's boxes
    (``build_planner_esdf`` builds it from a planar scan);
  * the sampling noise is keyed by the global problem index (``p0 + i`` for ``reqs[i]``), not by
    a per-request ``seed``: any batch split gives the same bits per problem;
  * ``n_trajs`` / ``n_iters`` / ``n_denoising`` are properties of the planner's preallocated
    buffers and schedule; a request that asks for different values raises ``ValueError``;
  * refinement takes fixed gradient steps (no Armijo line search): ``OptResult.converged`` is
    False and ``n_accepted`` = ``iterations``; the success flag is the dense clearance check.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, replace
from typing import List, Sequence

import numpy as np

from . import _lib, bl, spec
from .ref.pipeline import PlanResult
from .ref.trajopt import OptResult

# planseed's cost-term names (src/trajopt.py:16); the BL cost has only the smoothness and world terms
TERM_NAMES = ("goal_pos", "goal_rot", "smooth", "self", "world")


@dataclass
class BLPlanRequest:
    """One planning problem (planseed PlanRequest, src/pipeline.py:37-54, in BASELINE form)."""

    images: np.ndarray          # (n_images, H, W) depth in metres
    q_start: np.ndarray         # (7,) joint angles
    goal: np.ndarray            # (7,) goal xyz (metres, base frame) + unit quaternion (w, x, y, z)
    boxes: np.ndarray           # (n_boxes, 6) axis-aligned scene boxes (lo xyz, hi xyz)
    n_trajs: int = 32
    n_iters: int = 10
    n_denoising: int = 100

    def __post_init__(self):
        if self.n_trajs < 1:
            raise ValueError("n_trajs must be >= 1")
        if self.n_iters < 1:
            raise ValueError("n_iters must be >= 1")


def _planner_denoising(planner) -> int:
    return spec.K_STEPS if planner.steps is None else len(planner.steps)


def _check_requests(planner, reqs: Sequence[BLPlanRequest]) -> None:
    if len(reqs) == 0:
        raise ValueError("need at least one request")
    if len(reqs) > planner.Pmax:
        raise ValueError(f"{len(reqs)} requests exceed the planner's max_problems={planner.Pmax}")
    n_den = _planner_denoising(planner)
    for i, r in enumerate(reqs):
        if r.n_trajs != planner.S:
            raise ValueError(f"request {i}: n_trajs={r.n_trajs}, the planner samples {planner.S} seeds per problem")
        if r.n_iters != planner.cost.n_iters:
            raise ValueError(f"request {i}: n_iters={r.n_iters}, the planner refines {planner.cost.n_iters} steps")
        if r.n_denoising != n_den:
            raise ValueError(f"request {i}: n_denoising={r.n_denoising}, the planner's schedule has {n_den} steps")


def _stack(reqs: Sequence[BLPlanRequest], field: str) -> np.ndarray:
    arrs = [np.asarray(getattr(r, field), dtype=np.float32) for r in reqs]
    if any(a.shape != arrs[0].shape for a in arrs):
        raise ValueError(f"requests disagree on the shape of {field}")
    return np.ascontiguousarray(np.stack(arrs))


def plan_diffusion_batch(planner, reqs: Sequence[BLPlanRequest], p0: int = 0,
                         return_seeds: bool = True) -> List[PlanResult]:
    """Plan every request in one batched call; ``reqs[i]`` is global problem ``p0 + i``.

    Timings follow planseed's fields, as device time of the batch shared by its requests:
    ``esdf_time`` the phase before sampling (ESDF build + encoder, the image upload overlapping
    them), ``plan_time`` the whole call including the uploads and the read-back."""
    _check_requests(planner, reqs)
    torch = _lib.require_cuda()
    images, q_start, goal, boxes = (_stack(reqs, f) for f in ("images", "q_start", "goal", "boxes"))
    P, S, T = len(reqs), planner.S, planner.T
    # host tensors over the stacked arrays (pageable: pinning ~0.6 GB per call would cost more than
    # the staged copy; BLPlanner.plan_batch with caller-pinned buffers is the zero-copy path)
    pin = [torch.from_numpy(a) for a in (images, q_start, goal, boxes)]
    ev = {k: torch.cuda.Event(enable_timing=True)
          for k in ("start", "sample_start", "sample_end", "refine_start", "refine_end", "end")}
    t0 = time.perf_counter()
    ev["start"].record()
    d = planner.upload(*pin)
    r = planner.plan_batch_device(*d, p0=p0, images_ready=planner._img_chunks, events=ev)
    # world term of the refined trajectories (the same kernel with the smoothness weights zeroed):
    # the planseed breakdown splits the total into smoothness and world
    w0 = replace(planner.cost, w_vel=0.0, w_acc=0.0, w_jerk=0.0)
    world, _, _ = bl.cost(r.trajectories, planner.esdf[:P], S, planner.robot, planner.grid, w0,
                          esdf_layout=planner.esdf_layout)
    host = [x.to("cpu", non_blocking=True) for x in (r.trajectories, r.cost, r.feasible, r.best_index, world)]
    seeds = r.seeds.to("cpu", non_blocking=True) if return_seeds else None
    ev["end"].record()
    torch.cuda.current_stream().synchronize()
    wall = time.perf_counter() - t0
    traj, cost, feas, best, wterm = (h.numpy() for h in host)
    traj = traj.reshape(P, S, T, 7)
    seeds_np = seeds.numpy().reshape(P, S, T, 7) if seeds is not None else None
    # start -> sample_start: the upload of the small inputs, the ESDF build and the encoder (the
    # image upload overlaps them); reported as esdf_time, planseed's pre-sampling phase
    esdf_s = ev["start"].elapsed_time(ev["sample_start"]) * 1e-3
    plan_s = ev["start"].elapsed_time(ev["end"]) * 1e-3
    out = []
    for p in range(P):
        results = []
        for s in range(S):
            b = p * S + s
            c = float(cost[b])
            wv = float(wterm[b])
            terms = {"goal_pos": 0.0, "goal_rot": 0.0, "smooth": c - wv, "self": 0.0, "world": wv}
            results.append(OptResult(trajectory=traj[p, s].astype(np.float64), cost=c,
                                     breakdown={k: terms[k] for k in TERM_NAMES},
                                     iterations=planner.cost.n_iters, converged=False,
                                     n_accepted=planner.cost.n_iters))
        bi = int(best[p])
        out.append(PlanResult(seeder="diffusion", best_index=bi, trajectory=results[bi].trajectory,
                              results=results, successes=[bool(f) for f in feas[p * S:(p + 1) * S]],
                              plan_time=plan_s, esdf_time=esdf_s,
                              seed_trajectories=None if seeds_np is None else seeds_np[p].astype(np.float64)))
    planner.timing["plan_diffusion_batch_wall_s"] = wall
    return out


def plan_diffusion(planner, req: BLPlanRequest, p0: int = 0) -> PlanResult:
    """planseed's single-request call shape (src/pipeline.py:172-209) over the batched path."""
    return plan_diffusion_batch(planner, [req], p0=p0)[0]


def requests_from_problems(problems, n_trajs: int = 32, n_iters: int = 10,
                           n_denoising: int = 100) -> List[BLPlanRequest]:
    """Split a synth.ProblemBatch (images, q_start, goal, boxes) into requests."""
    return [BLPlanRequest(problems.images[i], problems.q_start[i], problems.goal[i], problems.boxes[i],
                          n_trajs=n_trajs, n_iters=n_iters, n_denoising=n_denoising)
            for i in range(len(problems.q_start))]
