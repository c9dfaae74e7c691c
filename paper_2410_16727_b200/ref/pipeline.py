"""Drop-in for planseed.pipeline's planner API on the GPU (src/pipeline.py:37-209).

plan_diffusion keeps the reference's orchestration and timing split (esdf_time vs
plan_time) and its host-side noise draw `default_rng(req.seed).standard_normal`
(SURVEY.md §7.5 hard part 3: x_K is drawn exactly as the reference draws it and
uploaded); everything else runs in the ref-profile CUDA kernels.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from .. import _lib
from .diffusion import PlannerCost, ddim_sample_device, encode_condition, guided_ddim_sample_device
from .trajopt import CostWeights, OptResult, _ArmArgs, _grid_device, optimize
from .types import WORKSPACE, Pose2, Rect, SdfGrid


@dataclass
class PlanRequest:
    """src/pipeline.py:37-54."""

    q_start: np.ndarray
    goal: Pose2
    scan: object
    n_trajs: int = 12
    n_iters: int = 50
    n_denoising: int = 5
    seed: int = 0
    bounds: Rect = WORKSPACE
    esdf_cell: float = 0.01
    delta_t: float = 0.005
    delta_r_deg: float = 2.86
    world: Optional[object] = None

    def __post_init__(self):
        if self.n_trajs < 1:
            raise ValueError("n_trajs must be >= 1")


@dataclass
class GuidanceParams:
    k_guide_frac: float = 0.6
    n_grad: int = 20
    alpha_guide: float = 1.0


@dataclass
class PlanResult:
    """src/pipeline.py:64-94."""

    seeder: str
    best_index: int
    trajectory: np.ndarray
    results: List[OptResult]
    successes: List[bool]
    plan_time: float
    esdf_time: float
    attempts: int = 1
    seed_trajectories: Optional[np.ndarray] = None

    @property
    def best(self) -> OptResult:
        return self.results[self.best_index]

    def to_dict(self) -> dict:
        return {"seeder": self.seeder, "best_index": self.best_index, "attempts": self.attempts,
                "plan_time_s": self.plan_time, "esdf_time_s": self.esdf_time, "best_cost": self.best.cost,
                "cost_breakdown": self.best.breakdown,
                "planner_successes": [bool(s) for s in self.successes],
                "trajectory": self.trajectory.tolist()}

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True)


def build_planner_esdf(bounds, scan, cell_size: float = 0.01, inflate_cells: float = 1.5) -> SdfGrid:
    """src/pipeline.py:101-132: each scan hit becomes a disc of radius inflate*cell; the
    ESDF over the workspace nodes is the exact distance to the nearest disc (capped at the
    padded bounds' diagonal when nothing was hit)."""
    torch = _lib.require_cuda()
    r = inflate_cells * cell_size
    ext = np.array(bounds.hi) - np.array(bounds.lo)
    nx = int(np.ceil(ext[0] / cell_size)) + 1
    ny = int(np.ceil(ext[1] / cell_size)) + 1
    origin = np.array(bounds.lo, dtype=np.float64)
    pad_ext = ext + 2.0 * r
    cap = float(np.hypot(*pad_ext))
    pose = scan.pose
    depths = torch.as_tensor(np.asarray(scan.depths, dtype=np.float64), device="cuda")
    out = torch.empty((nx, ny), dtype=torch.float64, device="cuda")
    st = _lib.lib().ps_ref_planner_esdf(_lib.ptr(depths), int(depths.numel()), float(pose.position[0]),
                                        float(pose.position[1]), float(pose.heading), float(pose.fov),
                                        float(pose.max_range), float(r), cap, float(origin[0]),
                                        float(origin[1]), float(cell_size), nx, ny, _lib.ptr(out),
                                        _lib.stream_handle())
    _lib.check(st, "planner_esdf")
    grid = SdfGrid(origin=origin, h=float(cell_size), nx=nx, ny=ny, values=out.cpu().numpy())
    object.__setattr__(grid, "_ps_dev_fp64", out)
    return grid


def planner_success_batch(arm, esdf, goal, trajs, delta_t=0.005, delta_r_deg=2.86, interp_per_seg=4):
    torch = _lib.require_cuda()
    t = torch.as_tensor(np.asarray(trajs, dtype=np.float64), device="cuda").contiguous()
    S, T, D = t.shape
    A = _ArmArgs(arm, esdf, goal, CostWeights(), T, "fp64")
    ok = torch.empty(S, dtype=torch.uint8, device="cuda")
    st = _lib.lib().ps_ref_planner_success(_lib.ptr(t), S, T, D, *A.args, float(delta_t),
                                           float(delta_r_deg), int(interp_per_seg), _lib.ptr(ok),
                                           _lib.stream_handle())
    _lib.check(st, "planner_success")
    return ok.cpu().numpy().astype(bool)


def planner_success(arm, esdf, goal, traj, delta_t: float = 0.005, delta_r_deg: float = 2.86,
                    interp_per_seg: int = 4) -> bool:
    """src/pipeline.py:139-157."""
    return bool(planner_success_batch(arm, esdf, goal, np.asarray(traj)[None], delta_t, delta_r_deg,
                                      interp_per_seg)[0])


def select_best(results: Sequence[OptResult], successes: Sequence[bool]) -> int:
    """src/pipeline.py:160-165: lowest-cost success, else lowest cost; ties to the lower index."""
    torch = _lib.require_cuda()
    if len(results) == 0:
        raise ValueError("no results to select from")
    c = torch.as_tensor(np.array([r.cost for r in results], dtype=np.float64), device="cuda")
    f = torch.as_tensor(np.array([bool(s) for s in successes], dtype=np.uint8), device="cuda")
    best = torch.empty(1, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().ps_ref_select(_lib.ptr(c), _lib.ptr(f), 1, len(results), _lib.ptr(best),
                                        _lib.stream_handle()), "select_best")
    return int(best.item())


def plan_diffusion(arm, net, schedule, req: PlanRequest, weights: CostWeights = CostWeights(),
                   guidance: Optional[GuidanceParams] = None, dtype: str = "fp64") -> PlanResult:
    """src/pipeline.py:172-209.  dtype="fp32" runs the encoder, the unguided sampler and the
    optimizer in float32 (the fast mode; guidance stays float64)."""
    torch = _lib.require_cuda()
    t0 = time.perf_counter()
    esdf = build_planner_esdf(req.bounds, req.scan, req.esdf_cell)
    esdf_time = time.perf_counter() - t0

    t1 = time.perf_counter()
    rng = np.random.default_rng(req.seed)
    cond = encode_condition(net, req.scan, req.q_start, req.goal, dtype=dtype)
    x_K = rng.standard_normal((req.n_trajs, net.config.t_len, net.config.dof))
    if guidance is not None and guidance.alpha_guide != 0.0:
        cost_fn = PlannerCost(arm, esdf, req.goal, weights)
        seeds, _ = guided_ddim_sample_device(net, schedule, cond, x_K, req.q_start, arm, cost_fn,
                                             n_steps=req.n_denoising, k_guide_frac=guidance.k_guide_frac,
                                             n_grad=guidance.n_grad, alpha_guide=guidance.alpha_guide)
        seeds = seeds.cpu().numpy()
    else:
        seeds = ddim_sample_device(net, schedule, cond, x_K, req.q_start, arm,
                                   n_steps=req.n_denoising, dtype=dtype).cpu().numpy().astype(np.float64)
        seeds[:, 0] = np.asarray(req.q_start, dtype=np.float64)
    results = optimize(arm, esdf, req.goal, list(seeds), req.n_iters, weights, dtype=dtype)
    successes = [bool(s) for s in planner_success_batch(arm, esdf, req.goal,
                                                        np.stack([r.trajectory for r in results]),
                                                        req.delta_t, req.delta_r_deg)]
    best = select_best(results, successes)
    torch.cuda.synchronize()
    plan_time = time.perf_counter() - t1
    return PlanResult(seeder="diffusion", best_index=best, trajectory=results[best].trajectory,
                      results=results, successes=successes, plan_time=plan_time, esdf_time=esdf_time,
                      seed_trajectories=seeds)
