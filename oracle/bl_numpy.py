"""ORACLE (test infrastructure only): float64 numpy restatement of the BASELINE-profile
refinement path, written independently of the canonical fp32 C oracle.

Formulation differs on purpose (4x4 homogeneous DH transforms, product-weight
trilinear interpolation, dense numpy.gradient operators) so that agreement between
this module, the C oracle and the CUDA kernels is evidence rather than a tautology.

Reference anchors (generalised from the planar planseed kernels):
  FK chain + points on links         planseed/arm.py:107-125
  bilinear value / in-cell gradient  planseed/_kernels.py:23-57  -> trilinear
  world hinge^2, gradient -2w h grad planseed/_kernels.py:206-228
  Jacobian^T accumulation            planseed/_kernels.py:277-289
  D = numpy.gradient stencil         planseed/trajopt.py:64-73
  row-0 gradient = 0                 planseed/_kernels.py:296-299
  planner_success dense check        planseed/pipeline.py:139-157
  select_best                        planseed/pipeline.py:160-165
"""

from __future__ import annotations

import numpy as np


def diff_matrix(n: int) -> np.ndarray:
    """numpy.gradient first-derivative stencil (planseed/trajopt.py:64-73)."""
    d = np.zeros((n, n))
    for i in range(1, n - 1):
        d[i, i - 1] = -0.5
        d[i, i + 1] = 0.5
    d[0, 0], d[0, 1] = -1.0, 1.0
    d[-1, -2], d[-1, -1] = -1.0, 1.0
    return d


def dh_frames(robot, q: np.ndarray):
    """q (..., 7) -> list of 8 homogeneous frames (..., 4, 4); frame 0 is the base."""
    q = np.asarray(q, dtype=np.float64)
    shp = q.shape[:-1]
    T = np.broadcast_to(np.eye(4), shp + (4, 4)).copy()
    T[..., :3, 3] = robot.base
    frames = [T]
    for k in range(robot.dof):
        c, s = np.cos(q[..., k]), np.sin(q[..., k])
        ca, sa = np.cos(robot.alpha[k]), np.sin(robot.alpha[k])
        A = np.zeros(shp + (4, 4))
        A[..., 0, 0] = c
        A[..., 0, 1] = -s * ca
        A[..., 0, 2] = s * sa
        A[..., 0, 3] = robot.a[k] * c
        A[..., 1, 0] = s
        A[..., 1, 1] = c * ca
        A[..., 1, 2] = -c * sa
        A[..., 1, 3] = robot.a[k] * s
        A[..., 2, 1] = sa
        A[..., 2, 2] = ca
        A[..., 2, 3] = robot.d[k]
        A[..., 3, 3] = 1.0
        T = T @ A
        frames.append(T)
    return frames


def sphere_centers(robot, q: np.ndarray):
    """(..., 7) -> sphere centres (..., S, 3) and the frames."""
    frames = dh_frames(robot, q)
    F = np.stack(frames[1:], axis=-3)                 # (..., 7, 4, 4)
    Fs = F[..., robot.sphere_link, :, :]              # (..., S, 4, 4)
    p = np.einsum("...ij,...j->...i", Fs[..., :3, :3], robot.sphere_offset) + Fs[..., :3, 3]
    return p, frames


def trilinear(values: np.ndarray, origin, h: float, pts: np.ndarray):
    """Product-weight trilinear value, in-cell gradient and clamp flag (N,3) points."""
    n = np.array(values.shape)
    u = (pts - np.asarray(origin)) / h
    clamped = np.any((u < 0) | (u > n - 1), axis=-1)
    idx = np.clip(np.floor(u).astype(np.int64), 0, n - 2)
    t = np.clip(u - idx, 0.0, 1.0)
    d = np.zeros(pts.shape[:-1])
    g = np.zeros(pts.shape)
    for cx in (0, 1):
        for cy in (0, 1):
            for cz in (0, 1):
                v = values[idx[..., 0] + cx, idx[..., 1] + cy, idx[..., 2] + cz]
                wx = t[..., 0] if cx else 1.0 - t[..., 0]
                wy = t[..., 1] if cy else 1.0 - t[..., 1]
                wz = t[..., 2] if cz else 1.0 - t[..., 2]
                d += v * wx * wy * wz
                g[..., 0] += v * (1 if cx else -1) * wy * wz
                g[..., 1] += v * wx * (1 if cy else -1) * wz
                g[..., 2] += v * wx * wy * (1 if cz else -1)
    return d, g / h, clamped


def esdf_boxes(boxes: np.ndarray, grid) -> np.ndarray:
    """Analytic signed distance to axis-aligned boxes (min over boxes), on the nodes."""
    n = grid.n
    axes = [grid.origin[a] + grid.h * np.arange(n[a]) for a in range(3)]
    P = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1)
    best = np.full(n, grid.cap)
    for b in boxes:
        c = 0.5 * (b[:3] + b[3:])
        hw = 0.5 * (b[3:] - b[:3])
        qd = np.abs(P - c) - hw
        outside = np.linalg.norm(np.maximum(qd, 0.0), axis=-1)
        inside = np.minimum(qd.max(axis=-1), 0.0)
        best = np.minimum(best, outside + inside)
    return best


def world_cost_grad(robot, values, origin, h, cost, q: np.ndarray):
    """World term per configuration and its joint gradient.  q (..., 7)."""
    p, frames = sphere_centers(robot, q)
    d, g, cl = trilinear(values, origin, h, p)
    r = robot.sphere_radius
    hinge = r + cost.margin - d
    act = hinge > 0
    wc = cost.w_coll * np.sum(np.where(act, hinge * hinge, 0.0), axis=-1)
    gp = np.where(act[..., None], -2.0 * cost.w_coll * hinge[..., None] * g, 0.0)  # (..., S, 3)
    gq = np.zeros(q.shape)
    for j in range(robot.dof):
        z = frames[j][..., :3, 2]
        o = frames[j][..., :3, 3]
        on = robot.sphere_link >= j
        lever = p - o[..., None, :]
        col = np.cross(z[..., None, :], lever)          # dp/dq_j
        gq[..., j] = np.sum(np.where(on[:, None], col * gp, 0.0), axis=(-1, -2))
    minclear = np.min(d - r, axis=-1)
    return wc, gq, minclear, np.any(cl, axis=-1)


def smooth_cost_grad(cost, x: np.ndarray):
    """x (B,T,7): w_v|Dq|^2 + w_a|D^2q|^2 + w_j|D^3q|^2 and its gradient."""
    T = x.shape[-2]
    D = diff_matrix(T)
    D2 = D @ D
    D3 = D2 @ D
    c = 0.0
    g = 0.0
    for w, M in ((cost.w_vel, D), (cost.w_acc, D2), (cost.w_jerk, D3)):
        y = np.einsum("rt,btk->brk", M, x)
        c = c + w * np.sum(y * y, axis=(1, 2))
        g = g + 2.0 * w * np.einsum("rt,brk->btk", M, y)
    return c, g


def bl_cost(robot, values_of, origin, h, cost, x: np.ndarray, S: int):
    """Total cost (B,), gradient (B,T,7) with row 0 zeroed, clamped (B,)."""
    x = np.asarray(x, dtype=np.float64)
    B = x.shape[0]
    wc = np.zeros(B)
    gw = np.zeros_like(x)
    cl = np.zeros(B, dtype=bool)
    for b in range(B):
        c, g, _, c_l = world_cost_grad(robot, values_of(b // S), origin, h, cost, x[b])
        wc[b] = c.sum()
        gw[b] = g
        cl[b] = c_l.any()
    sc, sg = smooth_cost_grad(cost, x)
    g = gw + sg
    g[:, 0, :] = 0.0
    return wc + sc, g, cl


def bl_refine(robot, values_of, origin, h, cost, x0: np.ndarray, S: int, n_iters: int):
    """Fixed-step refinement + final cost + dense feasibility (d - r > 0 at waypoints and
    4 interpolants per segment; out-of-grid points use clamped values, as
    planseed/pipeline.py:139-157 does through sample_esdf_many)."""
    x = np.asarray(x0, dtype=np.float64).copy()
    for _ in range(n_iters):
        _, g, _ = bl_cost(robot, values_of, origin, h, cost, x, S)
        x = x - cost.eta * g
    c, _, _ = bl_cost(robot, values_of, origin, h, cost, x, S)
    B, T, _ = x.shape
    feas = np.zeros(B, dtype=bool)
    minclear = np.zeros(B)
    fr = np.arange(1, 5) / 5.0
    for b in range(B):
        dense = [x[b]] + [x[b, :-1] + f * (x[b, 1:] - x[b, :-1]) for f in fr]
        cfg = np.concatenate(dense, axis=0)
        _, _, mc, cl = world_cost_grad(robot, values_of(b // S), origin, h, cost, cfg)
        minclear[b] = mc.min()
        feas[b] = mc.min() > 0.0
    return x, c, feas, minclear


def select_best(cost: np.ndarray, feasible: np.ndarray, S: int) -> np.ndarray:
    P = cost.shape[0] // S
    out = np.empty(P, dtype=np.int64)
    for p in range(P):
        c = cost[p * S:(p + 1) * S]
        f = feasible[p * S:(p + 1) * S]
        pool = [i for i in range(S) if f[i]] or list(range(S))
        out[p] = min(pool, key=lambda i: (c[i], i))
    return out


# ----------------------------------------------------------------------------
# Ground-truth evaluation (trajopt.metrics / retime / traj_min_clearance,
# planseed/trajopt.py:209-272, planseed/_kernels.py:144-162), 3-D BL form
# ----------------------------------------------------------------------------

def box_sdf(boxes: np.ndarray, pts: np.ndarray, cap: float) -> np.ndarray:
    """Analytic signed distance (..., 3) -> (...,) to the union of axis-aligned boxes (nb, 6),
    capped at `cap` (planseed/_kernels.py:60-83 in 3-D)."""
    b = np.asarray(boxes, dtype=np.float64)
    d = np.full(pts.shape[:-1], cap, dtype=np.float64)
    if b.shape[0] == 0:
        return d
    c = 0.5 * (b[:, :3] + b[:, 3:])
    hw = 0.5 * (b[:, 3:] - b[:, :3])
    q = np.abs(pts[..., None, :] - c) - hw                     # (..., nb, 3)
    out = np.linalg.norm(np.maximum(q, 0.0), axis=-1)
    ins = np.minimum(q.max(axis=-1), 0.0)
    return np.minimum(d, (out + ins).min(axis=-1))


def traj_min_clearance(robot, boxes, traj: np.ndarray, cap: float, interp_per_seg: int = 4) -> float:
    """Min over waypoints and interp_per_seg interpolants per segment of min over spheres of
    (box SDF at the centre - radius)."""
    traj = np.asarray(traj, dtype=np.float64)
    f = (np.arange(interp_per_seg) + 1.0) / (interp_per_seg + 1.0)
    qi = traj[:-1, None, :] + f[None, :, None] * (traj[1:, None, :] - traj[:-1, None, :])
    qs = np.concatenate([traj, qi.reshape(-1, traj.shape[1])], axis=0)
    p, _ = sphere_centers(robot, qs)
    return float((box_sdf(boxes, p, cap) - robot.sphere_radius).min())


def retime(traj: np.ndarray, vel=2.1, acc=15.0, jerk=7500.0):
    """(motion_time, max_jerk) -- planseed/trajopt.py:209-228 and metrics' max-jerk line."""
    traj = np.asarray(traj, dtype=np.float64)
    n = traj.shape[0]
    D = diff_matrix(n)
    v = D @ traj
    a = D @ v
    j = D @ a
    dt = max(float(np.max(np.abs(v).max(0) / vel)), float(np.sqrt(np.max(np.abs(a).max(0) / acc))),
             float(np.cbrt(np.max(np.abs(j).max(0) / jerk))))
    mt = dt * (n - 1)
    return mt, (float(np.abs(j).max()) / dt ** 3 if mt > 0.0 else 0.0)


def quat_matrix(qw, qx, qy, qz) -> np.ndarray:
    return np.array([[1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qz * qw), 2 * (qx * qz + qy * qw)],
                     [2 * (qx * qy + qz * qw), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qx * qw)],
                     [2 * (qx * qz - qy * qw), 2 * (qy * qz + qx * qw), 1 - 2 * (qx * qx + qy * qy)]])


def end_pose_errors(robot, q_last: np.ndarray, goal: np.ndarray):
    """(translation error m, rotation error deg) of the frame after joint 7 against the goal
    (xyz relative to the base, unit quaternion w, x, y, z)."""
    F = dh_frames(robot, np.asarray(q_last, dtype=np.float64))[-1]
    terr = float(np.linalg.norm(F[:3, 3] - robot.base - goal[:3]))
    G = quat_matrix(*goal[3:7])
    R = G.T @ F[:3, :3]
    v = np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])
    ang = np.arctan2(np.linalg.norm(v), np.trace(R) - 1.0)
    return terr, float(np.degrees(ang))


def bl_metrics(robot, boxes, goal, traj, cap, delta_t=0.005, delta_r_deg=2.86, interp_per_seg=4,
               limits=(2.1, 15.0, 7500.0)):
    """trajopt.metrics for one BL trajectory: dict of success, collision_free, clearance,
    translation_error, angle_error_deg, motion_time, max_jerk."""
    clr = traj_min_clearance(robot, boxes, traj, cap, interp_per_seg)
    terr, aerr = end_pose_errors(robot, traj[-1], np.asarray(goal, dtype=np.float64))
    mt, mj = retime(traj, *limits)
    free = clr > 0.0
    return {"success": bool(free and terr <= delta_t and aerr <= delta_r_deg), "collision_free": free,
            "clearance": clr, "translation_error": terr, "angle_error_deg": aerr, "motion_time": mt,
            "max_jerk": mj}
