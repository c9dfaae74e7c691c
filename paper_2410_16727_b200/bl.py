"""BASELINE-profile refinement API over the C-ABI (batched over problems).

Batched counterparts of the reference refiner / planner helpers:
  esdf_build      ~ geometry.build_esdf / pipeline.build_planner_esdf  (geometry.py:195-210)
  cost            ~ trajopt.evaluate_cost_batch                        (trajopt.py:105-119)
  refine          ~ trajopt.optimize + pipeline.planner_success        (trajopt.py:140-177,
                                                                        pipeline.py:139-157)
  select          ~ pipeline.select_best                               (pipeline.py:160-165)

  evaluate_cost_batch / optimize  the reference-semantics forms: raise ValueError naming the
                  seeds that leave the ESDF extent (trajopt.py:116-118, :157-163)

Inputs may be numpy arrays or torch CUDA tensors; outputs are torch CUDA tensors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .spec import BLCost, DHRobot, GridSpec


def _dev(x, dtype=None):
    torch = _lib.require_cuda()
    dtype = dtype or torch.float32
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.cuda()
        return t.to(dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda")


@dataclass
class RobotTables:
    """Host float32/int32 tables copied into each kernel's parameter block."""

    dh: np.ndarray
    base: np.ndarray
    sph: np.ndarray
    link: np.ndarray

    @classmethod
    def of(cls, robot: DHRobot) -> "RobotTables":
        return cls(dh=np.ascontiguousarray(robot.dh_table_f32()),
                   base=np.ascontiguousarray(robot.base, dtype=np.float32),
                   sph=np.ascontiguousarray(robot.sphere_table_f32()),
                   link=np.ascontiguousarray(robot.sphere_link, dtype=np.int32))


def _grid_args(grid: GridSpec):
    n = np.array(grid.n, dtype=np.int32)
    o = np.array(grid.origin, dtype=np.float32)
    return n, o


ESDF_C_ORDER, ESDF_BRICKED, ESDF_QUAD = 0, 1, 2


def esdf_build(boxes, grid: GridSpec = GridSpec(), stream=None, layout: int = ESDF_C_ORDER, out=None):
    """boxes (P, n_boxes, 6) -> ESDF values (P, nx, ny, nz) float32 on device.  With
    layout=ESDF_BRICKED the same values are stored in 4x4x4 bricks (the planner's layout;
    see ps_esdf_build_boxes_layout) and the tensor's index order is not (x, y, z)."""
    torch = _lib.require_cuda()
    b = _dev(boxes)
    if b.dim() != 3 or b.shape[2] != 6:
        raise ValueError("boxes must be (P, n_boxes, 6)")
    P = b.shape[0]
    n, o = _grid_args(grid)
    if layout == ESDF_QUAD:
        # quad bricks (4 floats per node, see ps_esdf_quad_expand): built as bricks, then expanded
        bricks = esdf_build(b, grid, stream, ESDF_BRICKED)
        if out is None:
            out = torch.empty((P,) + tuple(grid.n) + (4,), dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().ps_esdf_quad_expand(_lib.ptr(bricks), P, _lib.hptr(n), _lib.ptr(out),
                                                  _lib.stream_handle(stream)), "esdf_quad_expand")
        return out
    if out is None:
        out = torch.empty((P,) + tuple(grid.n), dtype=torch.float32, device="cuda")
    st = _lib.lib().ps_esdf_build_boxes_layout(_lib.ptr(b), P, b.shape[1], _lib.hptr(n), _lib.hptr(o),
                                               grid.h, grid.cap, _lib.ptr(out), int(layout),
                                               _lib.stream_handle(stream))
    _lib.check(st, "esdf_build")
    return out


def unbrick(esdf_bricked, grid: GridSpec = GridSpec()):
    """(P, nx, ny, nz)-shaped bricked storage -> C-order values (test / inspection helper)."""
    nx, ny, nz = grid.n
    P = esdf_bricked.shape[0]
    v = esdf_bricked.reshape(P, nx // 4, ny // 4, nz // 4, 4, 4, 4)
    return v.permute(0, 1, 4, 2, 5, 3, 6).reshape(P, nx, ny, nz)


def _esdf_stride(esdf, grid: GridSpec, n_problems: int) -> int:
    """Floats between consecutive problems' ESDFs (4 per node for quad bricks, (P, nx, ny, nz, 4))."""
    quad = esdf.dim() in (4, 5) and esdf.shape[-1] == 4 and tuple(esdf.shape[-4:-1]) == tuple(grid.n)
    if esdf.dim() == (4 if quad else 3):
        return 0                      # one ESDF shared by every problem
    if esdf.shape[0] == 1:
        return 0
    if esdf.shape[0] < n_problems:
        raise ValueError("need one ESDF per problem (or a single shared one)")
    return grid.n_nodes * (4 if quad else 1)


OUT_OF_GRID_MSG = "trajectory collision points leave the ESDF extent"


def _raise_out_of_grid(clamped):
    seeds = clamped.nonzero().flatten().cpu().tolist()
    raise ValueError(f"{OUT_OF_GRID_MSG} (seeds {seeds})")


def cost(q, esdf, S: int, robot: DHRobot, grid: GridSpec = GridSpec(), w: BLCost = BLCost(),
         stream=None, esdf_layout: int = ESDF_C_ORDER):
    """Batched cost (B,), gradient (B,T,7) (row 0 zero) and clamped flags (B,) -- the kernel-level
    form (cost_terms_batch, _kernels.py:165-312): never raises for out-of-grid points."""
    torch = _lib.require_cuda()
    qd = _dev(q)
    B, T, D = qd.shape
    if D != 7 or T not in (32, 64):
        raise ValueError("q must be (B, 32|64, 7)")
    e = _dev(esdf)
    rt = RobotTables.of(robot)
    n, o = _grid_args(grid)
    wts = w.as_f32()
    c = torch.empty(B, dtype=torch.float32, device="cuda")
    g = torch.empty_like(qd)
    cl = torch.empty(B, dtype=torch.uint8, device="cuda")
    st = _lib.lib().ps_bl_cost_layout(_lib.ptr(qd), B, T, S, _lib.ptr(e), _esdf_stride(e, grid, -(-B // S)),
                                      int(esdf_layout), _lib.hptr(n), _lib.hptr(o), grid.h, _lib.hptr(rt.dh),
                                      _lib.hptr(rt.base), _lib.hptr(rt.sph), _lib.hptr(rt.link),
                                      len(rt.link), _lib.hptr(wts), _lib.ptr(c), _lib.ptr(g), _lib.ptr(cl),
                                      _lib.stream_handle(stream))
    _lib.check(st, "bl_cost")
    return c, g, cl.bool()


def evaluate_cost_batch(q, esdf, S: int, robot: DHRobot, grid: GridSpec = GridSpec(), w: BLCost = BLCost(),
                        stream=None, esdf_layout: int = ESDF_C_ORDER):
    """trajopt.evaluate_cost_batch semantics (trajopt.py:104-119): (totals, grads); raises
    ValueError naming the seeds whose collision spheres leave the ESDF extent."""
    c, g, cl = cost(q, esdf, S, robot, grid, w, stream, esdf_layout)
    if bool(cl.any()):
        _raise_out_of_grid(cl)
    return c, g


def optimize(q, esdf, S: int, robot: DHRobot, grid: GridSpec = GridSpec(), w: BLCost = BLCost(),
             n_iters: int | None = None, stream=None, out=None, esdf_layout: int = ESDF_C_ORDER):
    """trajopt.optimize semantics (trajopt.py:140-177) for the fixed-step BL refinement: ValueError
    for n_iters < 1 or no seeds, and -- before any refinement -- for seeds that leave the ESDF
    extent (ps_bl_optimize).  Returns refine()'s (q_out, cost, feasible, clamped)."""
    torch = _lib.require_cuda()
    n_iters = w.n_iters if n_iters is None else int(n_iters)
    if n_iters < 1:
        raise ValueError("n_iters must be >= 1")
    qd = _dev(q)
    if qd.dim() != 3 or qd.shape[0] == 0:
        raise ValueError("need at least one seed")
    B, T, D = qd.shape
    if D != 7 or T not in (32, 64):
        raise ValueError("q must be (B, 32|64, 7)")
    e = _dev(esdf)
    rt = RobotTables.of(robot)
    n, o = _grid_args(grid)
    wts = w.as_f32()
    if out is None:
        out = (torch.empty_like(qd), torch.empty(B, dtype=torch.float32, device="cuda"),
               torch.empty(B, dtype=torch.uint8, device="cuda"),
               torch.empty(B, dtype=torch.uint8, device="cuda"))
    qo, c, f, cl = out
    cl0 = torch.empty(B, dtype=torch.uint8, device="cuda")
    st = _lib.lib().ps_bl_optimize(_lib.ptr(qd), B, T, S, _lib.ptr(e), _esdf_stride(e, grid, -(-B // S)),
                                   int(esdf_layout), _lib.hptr(n), _lib.hptr(o), grid.h, _lib.hptr(rt.dh),
                                   _lib.hptr(rt.base), _lib.hptr(rt.sph), _lib.hptr(rt.link), len(rt.link),
                                   _lib.hptr(wts), n_iters, _lib.ptr(qo), _lib.ptr(c), _lib.ptr(f), _lib.ptr(cl),
                                   _lib.ptr(cl0), _lib.stream_handle(stream))
    if st == _lib.PS_ERR_OUT_OF_GRID:
        _raise_out_of_grid(cl0.bool())
    _lib.check(st, "bl_optimize")
    return qo, c, f, cl


def refine(q, esdf, S: int, robot: DHRobot, grid: GridSpec = GridSpec(), w: BLCost = BLCost(),
           n_iters: int | None = None, stream=None, out=None, esdf_layout: int = ESDF_C_ORDER):
    """n_iters fixed steps + final cost, feasibility and clamped flags.

    Returns (q_out (B,T,7), cost (B,), feasible (B,) bool, clamped (B,) bool)."""
    torch = _lib.require_cuda()
    qd = _dev(q)
    B, T, D = qd.shape
    if D != 7 or T not in (32, 64):
        raise ValueError("q must be (B, 32|64, 7)")
    n_iters = w.n_iters if n_iters is None else n_iters
    e = _dev(esdf)
    rt = RobotTables.of(robot)
    n, o = _grid_args(grid)
    wts = w.as_f32()
    if out is None:
        out = (torch.empty_like(qd), torch.empty(B, dtype=torch.float32, device="cuda"),
               torch.empty(B, dtype=torch.uint8, device="cuda"),
               torch.empty(B, dtype=torch.uint8, device="cuda"))
    qo, c, f, cl = out
    st = _lib.lib().ps_bl_refine_layout(_lib.ptr(qd), B, T, S, _lib.ptr(e), _esdf_stride(e, grid, -(-B // S)),
                                        int(esdf_layout), _lib.hptr(n), _lib.hptr(o), grid.h, _lib.hptr(rt.dh),
                                        _lib.hptr(rt.base), _lib.hptr(rt.sph), _lib.hptr(rt.link),
                                        len(rt.link), _lib.hptr(wts), int(n_iters), _lib.ptr(qo),
                                        _lib.ptr(c), _lib.ptr(f), _lib.ptr(cl), _lib.stream_handle(stream))
    _lib.check(st, "bl_refine")
    return qo, c, f, cl


def guide(x0, esdf, S: int, robot: DHRobot, grid: GridSpec = GridSpec(), w: BLCost = BLCost(),
          lo=None, span=None, n_grad: int = 20, alpha: float = 1.0, max_halvings: int = 8, stream=None,
          esdf_layout: int = ESDF_C_ORDER):
    """guided_ddim_sample's guide() (planseed/diffusion.py:598-617) for the BL cost, in place on the
    normalised x0_hat (B,T,7) device tensor; returns the per-seed clamped flags (B,) (some
    evaluation left the ESDF extent)."""
    torch = _lib.require_cuda()
    B, T, D = x0.shape
    if D != 7 or T not in (32, 64) or not x0.is_cuda or x0.dtype != torch.float32 or not x0.is_contiguous():
        raise ValueError("x0 must be a contiguous float32 CUDA tensor (B, 32|64, 7)")
    e = _dev(esdf)
    rt = RobotTables.of(robot)
    n, o = _grid_args(grid)
    lo = np.ascontiguousarray(robot.lo if lo is None else lo, dtype=np.float32)
    span = np.ascontiguousarray((robot.hi - robot.lo) if span is None else span, dtype=np.float32)
    cl = torch.empty(B, dtype=torch.uint8, device="cuda")
    st = _lib.lib().ps_bl_guide(_lib.ptr(x0), B, T, S, _lib.ptr(e), _esdf_stride(e, grid, -(-B // S)),
                                int(esdf_layout), _lib.hptr(n), _lib.hptr(o), grid.h, _lib.hptr(rt.dh),
                                _lib.hptr(rt.base), _lib.hptr(rt.sph), _lib.hptr(rt.link), len(rt.link),
                                _lib.hptr(w.as_f32()), _lib.hptr(lo), _lib.hptr(span), int(n_grad), float(alpha),
                                int(max_halvings), _lib.ptr(cl), _lib.stream_handle(stream))
    _lib.check(st, "bl_guide")
    return cl.bool()


@dataclass
class BLMetrics:
    """trajopt.TrajectoryMetrics for a batch (device tensors, one entry per trajectory)."""

    success: object
    collision_free: object
    clearance: object
    translation_error: object
    angle_error_deg: object
    motion_time: object
    max_jerk: object


def metrics(traj, boxes, goal, S: int, robot: DHRobot, cap: float = GridSpec().cap,
            delta_t: float | None = None, delta_r_deg: float | None = None,
            interp_per_seg: int | None = None, limits=None, stream=None) -> BLMetrics:
    """Ground-truth evaluation of (B, T, 7) trajectories against each problem's analytic boxes
    (P, n_boxes, 6) and goal (P, 7) -- trajopt.metrics / retime / traj_min_clearance
    (trajopt.py:209-272, _kernels.py:144-162) in 3-D, one launch for the whole batch."""
    from . import spec
    torch = _lib.require_cuda()
    q = _dev(traj)
    B, T, D = q.shape
    if D != 7 or T not in (32, 64):
        raise ValueError("traj must be (B, 32|64, 7)")
    bx, g = _dev(boxes), _dev(goal)
    if bx.dim() != 3 or bx.shape[2] != 6 or g.shape != (bx.shape[0], 7) or bx.shape[0] * S < B:
        raise ValueError("boxes (P, n_boxes, 6) and goal (P, 7) for P = B / S problems")
    rt = RobotTables.of(robot)
    lim = np.asarray(limits if limits is not None else (spec.VEL_LIMIT, spec.ACC_LIMIT, spec.JERK_LIMIT),
                     dtype=np.float32)
    f = lambda: torch.empty(B, dtype=torch.float32, device="cuda")
    u = lambda: torch.empty(B, dtype=torch.uint8, device="cuda")
    out = BLMetrics(u(), u(), f(), f(), f(), f(), f())
    st = _lib.lib().ps_bl_metrics(
        _lib.ptr(q), B, T, S, _lib.ptr(bx), bx.shape[1], _lib.ptr(g), _lib.hptr(rt.dh), _lib.hptr(rt.base),
        _lib.hptr(rt.sph), _lib.hptr(rt.link), len(rt.link), _lib.hptr(lim), float(cap),
        spec.DELTA_T if delta_t is None else float(delta_t),
        spec.DELTA_R_DEG if delta_r_deg is None else float(delta_r_deg),
        spec.INTERP_PER_SEG if interp_per_seg is None else int(interp_per_seg),
        _lib.ptr(out.clearance), _lib.ptr(out.translation_error), _lib.ptr(out.angle_error_deg),
        _lib.ptr(out.motion_time), _lib.ptr(out.max_jerk), _lib.ptr(out.success), _lib.ptr(out.collision_free),
        _lib.stream_handle(stream))
    _lib.check(st, "bl_metrics")
    return out


def select(cost_, feasible, S: int, stream=None, out=None):
    """Best seed per problem (P,) int32: lowest-cost feasible, else lowest cost, ties low."""
    torch = _lib.require_cuda()
    c = _dev(cost_)
    f = _dev(feasible, torch.uint8)
    P = c.shape[0] // S
    best = out if out is not None else torch.empty(P, dtype=torch.int32, device="cuda")
    st = _lib.lib().ps_select(_lib.ptr(c), _lib.ptr(f), P, S, _lib.ptr(best),
                              _lib.stream_handle(stream))
    _lib.check(st, "select")
    return best
