"""Drop-in for planseed.trajopt's refiner API on the GPU (src/trajopt.py).

Same names, arguments, return types and exceptions as the reference; the arithmetic
runs in the ref-profile CUDA kernels (`ps_ref_cost_terms`, `ps_ref_optimize`) in
float64 by default (parity mode), or float32 (`dtype="fp32"`).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache
from typing import Dict, List, Sequence, Tuple

import numpy as np

from .. import _lib
from .types import nonadjacent_point_pairs

DEFAULT_T = 32
TERM_NAMES = ("goal_pos", "goal_rot", "smooth", "self", "world")


@dataclass(frozen=True)
class CostWeights:
    """src/trajopt.py:19-36."""

    w_goal_pos: float = 100.0
    w_goal_rot: float = 10.0
    w_smooth: float = 1.0
    w_self: float = 50.0
    w_world: float = 50.0
    d_act: float = 0.05
    d_self: float = 0.03

    def __post_init__(self):
        for name in ("w_goal_pos", "w_goal_rot", "w_smooth", "w_self", "w_world"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be nonnegative")

    def as_array(self) -> np.ndarray:
        return np.array([self.w_goal_pos, self.w_goal_rot, self.w_smooth, self.w_self, self.w_world])


@dataclass
class OptResult:
    """src/trajopt.py:39-46."""

    trajectory: np.ndarray
    cost: float
    breakdown: Dict[str, float]
    iterations: int
    converged: bool
    n_accepted: int = 0


@lru_cache(maxsize=None)
def diff_matrix(n: int) -> np.ndarray:
    """numpy.gradient stencil (src/trajopt.py:64-73) -- an operator table, host-built."""
    d = np.zeros((n, n))
    for i in range(1, n - 1):
        d[i, i - 1] = -0.5
        d[i, i + 1] = 0.5
    d[0, 0], d[0, 1] = -1.0, 1.0
    d[-1, -2], d[-1, -1] = -1.0, 1.0
    return d


@lru_cache(maxsize=None)
def jerk_matrix(n: int) -> np.ndarray:
    d = diff_matrix(n)
    return d @ d @ d


@lru_cache(maxsize=None)
def _jerk_quad(n: int) -> np.ndarray:
    j = jerk_matrix(n)
    return 2.0 * (j.T @ j)


_DT = {"fp64": 0, "fp32": 1}


def _np_dtype(dtype: str):
    return np.float64 if dtype == "fp64" else np.float32


_dev_cache: Dict[Tuple, object] = {}


def _device(a: np.ndarray, dtype: str, key=None):
    torch = _lib.require_cuda()
    tdt = torch.float64 if dtype == "fp64" else torch.float32
    if key is not None and key in _dev_cache:
        return _dev_cache[key]
    t = torch.as_tensor(np.ascontiguousarray(a, dtype=_np_dtype(dtype)), device="cuda").to(tdt)
    if key is not None:
        _dev_cache[key] = t
    return t


def _grid_device(esdf, dtype: str):
    """Cache the device copy of an SdfGrid on the object (values are immutable)."""
    attr = "_ps_dev_" + dtype
    t = getattr(esdf, attr, None) if not isinstance(esdf, dict) else None
    if t is None:
        t = _device(esdf.values, dtype)
        try:
            object.__setattr__(esdf, attr, t)
        except Exception:
            pass
    return t


class _ArmArgs:
    """The 22 positional arm/grid/goal/weight arguments (src/trajopt.py:89-98)."""

    def __init__(self, arm, esdf, goal, w: CostWeights, t_len: int, dtype: str):
        pa, pb = nonadjacent_point_pairs(arm)
        self.keep = [np.ascontiguousarray(arm.lengths, dtype=np.float64),
                     np.ascontiguousarray(arm.point_fractions(), dtype=np.float64),
                     np.ascontiguousarray(pa, dtype=np.int64), np.ascontiguousarray(pb, dtype=np.int64),
                     np.ascontiguousarray(w.as_array(), dtype=np.float64)]
        self.grid = _grid_device(esdf, dtype)
        self.jm = _device(jerk_matrix(t_len), dtype, key=("jm", t_len, dtype))
        self.jq = _device(_jerk_quad(t_len), dtype, key=("jq", t_len, dtype))
        L, F, PA, PB, W = self.keep
        self.args = [
            _lib.hptr(L), float(arm.base[0]), float(arm.base[1]), _lib.hptr(F), len(F),
            _lib.hptr(PA), _lib.hptr(PB), len(PA),
            _lib.ptr(self.grid), int(esdf.values.shape[0]), int(esdf.values.shape[1]),
            float(esdf.origin[0]), float(esdf.origin[1]), float(esdf.h),
            float(goal.pos[0]), float(goal.pos[1]), float(goal.theta),
            _lib.hptr(W), float(w.d_act), float(w.d_self), _lib.ptr(self.jm), _lib.ptr(self.jq),
        ]


def cost_terms_batch_device(arm, esdf, goal, trajs, w: CostWeights, want_grad: bool = True,
                            dtype: str = "fp64"):
    """Raw kernel call: (terms (S,5), totals (S,), grads (S,T,D), clamped (S,)) as device tensors."""
    torch = _lib.require_cuda()
    q = _device(trajs, dtype) if not isinstance(trajs, torch.Tensor) else trajs
    S, T, D = q.shape
    A = _ArmArgs(arm, esdf, goal, w, T, dtype)
    tdt = q.dtype
    terms = torch.empty((S, 5), dtype=tdt, device="cuda")
    totals = torch.empty(S, dtype=tdt, device="cuda")
    grads = torch.empty_like(q)
    clamped = torch.empty(S, dtype=torch.uint8, device="cuda")
    st = _lib.lib().ps_ref_cost_terms(_DT[dtype], _lib.ptr(q), S, T, D, *A.args, int(bool(want_grad)),
                                      _lib.ptr(terms), _lib.ptr(totals), _lib.ptr(grads),
                                      _lib.ptr(clamped), _lib.stream_handle())
    _lib.check(st, "cost_terms_batch")
    return terms, totals, grads, clamped


def evaluate_cost_batch(arm, esdf, goal, trajs, w: CostWeights, want_grad: bool = True,
                        dtype: str = "fp64"):
    """src/trajopt.py:105-119: (totals (S,), grads (S,T,D), terms (S,5)); raises ValueError
    when any collision point leaves the ESDF extent."""
    trajs = np.asarray(trajs, dtype=np.float64)
    terms, totals, grads, clamped = cost_terms_batch_device(arm, esdf, goal, trajs, w, want_grad, dtype)
    cl = clamped.cpu().numpy().astype(bool)
    if np.any(cl):
        raise ValueError("trajectory collision points leave the ESDF extent "
                         f"(seeds {np.nonzero(cl)[0].tolist()})")
    f = np.float64
    return totals.cpu().numpy().astype(f), grads.cpu().numpy().astype(f), terms.cpu().numpy().astype(f)


def evaluate_cost(arm, esdf, goal, traj, w: CostWeights, dtype: str = "fp64"):
    totals, grads, _ = evaluate_cost_batch(arm, esdf, goal, np.asarray(traj)[None], w, dtype=dtype)
    return float(totals[0]), grads[0]


def cost_breakdown(arm, esdf, goal, traj, w: CostWeights, dtype: str = "fp64") -> Dict[str, float]:
    _, _, terms = evaluate_cost_batch(arm, esdf, goal, np.asarray(traj)[None], w, want_grad=False,
                                      dtype=dtype)
    return dict(zip(TERM_NAMES, terms[0].tolist()))


def optimize_device(arm, esdf, goal, stack, n_iters: int, w: CostWeights, momentum=0.9, armijo_c=1e-4,
                    shrink=0.5, max_backtracks=40, alpha0=1.0, alpha_max=4.0, dtype: str = "fp64"):
    """Raw `ps_ref_optimize` call -> (x, terms, totals, frozen, n_accepted) device tensors."""
    torch = _lib.require_cuda()
    q = _device(stack, dtype) if not isinstance(stack, torch.Tensor) else stack
    S, T, D = q.shape
    A = _ArmArgs(arm, esdf, goal, w, T, dtype)
    x = torch.empty_like(q)
    terms = torch.empty((S, 5), dtype=q.dtype, device="cuda")
    totals = torch.empty(S, dtype=q.dtype, device="cuda")
    frozen = torch.empty(S, dtype=torch.uint8, device="cuda")
    nacc = torch.empty(S, dtype=torch.int64, device="cuda")
    st = _lib.lib().ps_ref_optimize(_DT[dtype], _lib.ptr(q), S, T, D, int(n_iters), float(momentum),
                                    float(armijo_c), float(shrink), int(max_backtracks), float(alpha0),
                                    float(alpha_max), *A.args, _lib.ptr(x), _lib.ptr(terms),
                                    _lib.ptr(totals), _lib.ptr(frozen), _lib.ptr(nacc),
                                    _lib.stream_handle())
    _lib.check(st, "optimize_batch")
    return x, terms, totals, frozen, nacc


def optimize(arm, esdf, goal, seeds: Sequence[np.ndarray], n_iters: int, w: CostWeights,
             momentum: float = 0.9, armijo_c: float = 1e-4, shrink: float = 0.5,
             max_backtracks: int = 40, dtype: str = "fp64") -> List[OptResult]:
    """src/trajopt.py:140-177: exactly n_iters momentum/Armijo iterations per seed."""
    if n_iters < 1:
        raise ValueError("n_iters must be >= 1")
    if len(seeds) == 0:
        raise ValueError("need at least one seed")
    stack = np.stack([np.asarray(s, dtype=np.float64) for s in seeds])
    evaluate_cost_batch(arm, esdf, goal, stack, w, want_grad=False, dtype=dtype)
    x, terms, totals, frozen, nacc = optimize_device(arm, esdf, goal, stack, n_iters, w, momentum,
                                                     armijo_c, shrink, max_backtracks, 1.0, 4.0, dtype)
    x, terms, totals = (t.cpu().numpy().astype(np.float64) for t in (x, terms, totals))
    frozen, nacc = frozen.cpu().numpy().astype(bool), nacc.cpu().numpy()
    return [OptResult(trajectory=x[s], cost=float(totals[s]),
                      breakdown=dict(zip(TERM_NAMES, terms[s].tolist())), iterations=n_iters,
                      converged=bool(frozen[s]), n_accepted=int(nacc[s]))
            for s in range(stack.shape[0])]


# ----------------------------------------------------------------------------- ground truth
@dataclass
class TrajectoryMetrics:
    """src/trajopt.py:49-57."""

    success: bool
    plan_time: float
    max_jerk: float
    motion_time: float
    translation_error: float
    angle_error_deg: float
    collision_free: bool


def success_flag(collision_free: bool, translation_error: float, angle_error_deg: float,
                 delta_t: float, delta_r_deg: float) -> bool:
    """src/trajopt.py:232-236."""
    return bool(collision_free and translation_error <= delta_t and angle_error_deg <= delta_r_deg)


def metrics_device(arm, gt_world, goal, trajs, interp_per_seg: int = 4):
    """Raw `ps_ref_metrics` call: (S,6) device f64 rows [clearance, translation error,
    angle error deg, motion time, max jerk, dt] for trajectories (S,T,D)."""
    torch = _lib.require_cuda()
    t = trajs if isinstance(trajs, torch.Tensor) else torch.as_tensor(np.asarray(trajs, dtype=np.float64),
                                                                        device="cuda")
    t = t.to(torch.float64).contiguous()
    S, T, D = t.shape
    keep = [np.ascontiguousarray(arm.lengths, dtype=np.float64),
            np.ascontiguousarray(arm.point_fractions(), dtype=np.float64)]
    dev = lambda a, shape: torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(shape)),
                                           device="cuda")
    circ = dev(gt_world.circle_arr, (-1, 3))
    box = dev(gt_world.box_arr, (-1, 4))
    lims = [dev(arm.vel_limit, (-1,)), dev(arm.acc_limit, (-1,)), dev(arm.jerk_limit, (-1,))]
    jm = _device(jerk_matrix(T), "fp64", key=("jm", T, "fp64"))
    out = torch.empty((S, 6), dtype=torch.float64, device="cuda")
    st = _lib.lib().ps_ref_metrics(_lib.ptr(t), S, T, D, _lib.hptr(keep[0]), float(arm.base[0]),
                                   float(arm.base[1]), _lib.hptr(keep[1]), len(keep[1]), _lib.ptr(circ),
                                   circ.shape[0], _lib.ptr(box), box.shape[0], float(gt_world.sdf_cap),
                                   float(goal.pos[0]), float(goal.pos[1]), float(goal.theta), _lib.ptr(jm),
                                   *[_lib.ptr(x) for x in lims], int(interp_per_seg), _lib.ptr(out),
                                   _lib.stream_handle())
    _lib.check(st, "metrics")
    return out


def retime(arm, traj) -> Tuple[float, np.ndarray]:
    """src/trajopt.py:209-229: uniform waypoint spacing meeting the velocity /
    acceleration / jerk limits -> (motion_time, per-waypoint timestamps)."""
    from .types import Rect, World
    traj = np.asarray(traj, dtype=np.float64)
    T = traj.shape[0]
    dt = float(metrics_device(arm, World((), Rect((-1.0, -1.0), (1.0, 1.0))), _ZeroPose(), traj[None])[0, 5])
    return dt * (T - 1), dt * np.arange(T)


class _ZeroPose:
    pos = np.zeros(2)
    theta = 0.0


def metrics_batch(arm, gt_world, goal, trajs, plan_time=0.0, delta_t: float = 0.005,
                  delta_r_deg: float = 2.86, interp_per_seg: int = 4) -> List[TrajectoryMetrics]:
    """metrics() over a stack (S,T,D) in one launch; plan_time scalar or per trajectory."""
    m = metrics_device(arm, gt_world, goal, trajs, interp_per_seg).cpu().numpy()
    pt = np.broadcast_to(np.asarray(plan_time, dtype=np.float64), (m.shape[0],))
    out = []
    for s in range(m.shape[0]):
        cf = bool(m[s, 0] > 0.0)
        out.append(TrajectoryMetrics(success=success_flag(cf, float(m[s, 1]), float(m[s, 2]), delta_t, delta_r_deg),
                                     plan_time=float(pt[s]), max_jerk=float(m[s, 4]), motion_time=float(m[s, 3]),
                                     translation_error=float(m[s, 1]), angle_error_deg=float(m[s, 2]),
                                     collision_free=cf))
    return out


def metrics(arm, gt_world, goal, traj, plan_time: float = 0.0, delta_t: float = 0.005,
            delta_r_deg: float = 2.86, interp_per_seg: int = 4) -> TrajectoryMetrics:
    """src/trajopt.py:239-272: judge a trajectory against ground-truth geometry."""
    return metrics_batch(arm, gt_world, goal, np.asarray(traj, dtype=np.float64)[None], plan_time, delta_t,
                         delta_r_deg, interp_per_seg)[0]


def traj_min_clearance(arm, gt_world, traj, interp_per_seg: int = 4) -> float:
    """_kernels.traj_min_clearance (src/_kernels.py:144-162) for one trajectory."""
    return float(metrics_device(arm, gt_world, _ZeroPose(), np.asarray(traj, dtype=np.float64)[None],
                                interp_per_seg)[0, 0].item())
