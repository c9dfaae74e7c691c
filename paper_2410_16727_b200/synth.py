"""Seeded synthetic inputs for the BASELINE configs.

The paper evaluates on the MpiNet scenes, which are absent; BASELINE.json's synthetic
scenes stand in for them.  Every problem p is drawn from its own generator
`default_rng([seed, p, stream])`, so a shard of problems [p0, p1) is identical no
matter how many ranks split the batch (the world-size invariance the reference's
data generator guarantees for worker counts, planseed/data.py:391-394).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .spec import (BOX_SIDE, DOF, GOAL_EXTENT, JOINT_LIMIT, N_BOXES, GridSpec)

STREAM_PROBLEM = 11
STREAM_BOXES = 12
STREAM_IMAGE = 13
STREAM_REFINE = 14


def _rng(seed: int, p: int, stream: int) -> np.random.Generator:
    return np.random.default_rng([int(seed), int(p), int(stream)])


@dataclass
class ProblemBatch:
    """Problems [p0, p0+P) of a seeded batch, host arrays."""

    p0: int
    q_start: np.ndarray   # (P, 7) float32, radians
    goal: np.ndarray      # (P, 7) float32: xyz (m) + unit quaternion (w, x, y, z)
    boxes: np.ndarray     # (P, n_boxes, 6) float32: lo xyz, hi xyz
    images: Optional[np.ndarray] = None   # (P, n_img, H, W) float32 depth, m

    @property
    def P(self) -> int:
        return int(self.q_start.shape[0])


def sample_q_start(rng) -> np.ndarray:
    # U(-pi, pi)^7 clipped to the Franka-like limits (BASELINE config 0)
    return np.clip(rng.uniform(-math.pi, math.pi, size=DOF), -JOINT_LIMIT, JOINT_LIMIT)


def sample_goal(rng) -> np.ndarray:
    xyz = rng.uniform(-GOAL_EXTENT, GOAL_EXTENT, size=3)
    quat = rng.standard_normal(4)
    quat /= np.linalg.norm(quat)
    return np.concatenate([xyz, quat])


def sample_boxes(rng, n_boxes: int = N_BOXES, grid: GridSpec = GridSpec()) -> np.ndarray:
    side = rng.uniform(BOX_SIDE[0], BOX_SIDE[1], size=(n_boxes, 3))
    lo = rng.uniform(0.0, 1.0, size=(n_boxes, 3)) * (grid.cube - side)
    return np.concatenate([lo, lo + side], axis=1)


def depth_image_params(rng, h: int, w: int, n_rect: int) -> np.ndarray:
    """The draws of one synthetic depth image: [background, (y0, y1, x0, x1, depth) x n_rect]
    (float64; the corners are integers).  Background b ~ U(0.3, 2.0) m; n_rect axis-aligned
    pixel rectangles with random corners at depths ~ U(0.3, 2.0)."""
    out = np.empty(1 + 5 * n_rect)
    out[0] = rng.uniform(0.3, 2.0)
    for r in range(n_rect):
        ys = np.sort(rng.integers(0, h + 1, size=2))
        xs = np.sort(rng.integers(0, w + 1, size=2))
        out[1 + 5 * r:6 + 5 * r] = (ys[0], ys[1], xs[0], xs[1], rng.uniform(0.3, 2.0))
    return out


def render_depth_params(prm: np.ndarray, h: int, w: int) -> np.ndarray:
    """Host rasteriser of depth_image_params: each pixel keeps the nearest depth."""
    img = np.full((h, w), prm[0])
    for r in range((len(prm) - 1) // 5):
        y0, y1, x0, x1, depth = prm[1 + 5 * r:6 + 5 * r]
        sub = img[int(y0):int(y1), int(x0):int(x1)]
        np.minimum(sub, depth, out=sub)
    return img


def synth_depth_image(rng, h: int, w: int, n_rect: int) -> np.ndarray:
    """Uniform background b ~ U(0.3, 2.0) m; n_rect axis-aligned pixel rectangles
    with random corners at depths ~ U(0.3, 2.0); each pixel keeps the nearest depth."""
    return render_depth_params(depth_image_params(rng, h, w, n_rect), h, w)


def image_params(P: int, p0: int = 0, seed: int = 0, image_shape=(240, 320), n_images: int = 2,
                 n_rect: int = 8) -> np.ndarray:
    """(P, n_images, 1 + 5 n_rect) draws of make_problems' images (same per-problem streams)."""
    out = np.empty((P, n_images, 1 + 5 * n_rect))
    for i in range(P):
        ri = _rng(seed, p0 + i, STREAM_IMAGE)
        for m in range(n_images):
            out[i, m] = depth_image_params(ri, image_shape[0], image_shape[1], n_rect)
    return out


def render_images_device(params: np.ndarray, image_shape, stream=None):
    """Rasterise image_params on the GPU (ps_render_depth_rects) -> (P, n_images, H, W) float32
    CUDA tensor, bit-identical to the host rasteriser (min of float32-rounded depths)."""
    from . import _lib
    torch = _lib.require_cuda()
    prm = np.ascontiguousarray(params, dtype=np.float32)
    P, n_img, n_par = prm.shape
    H, W = image_shape
    d_prm = torch.as_tensor(prm, device="cuda")
    out = torch.empty((P, n_img, H, W), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().ps_render_depth_rects(_lib.ptr(d_prm), P * n_img, (n_par - 1) // 5, H, W, _lib.ptr(out),
                                                _lib.stream_handle(stream)), "render_depth_rects")
    return out


def make_problems(P: int, p0: int = 0, seed: int = 0, n_boxes: int = N_BOXES,
                  image_shape=None, n_images: int = 1, n_rect: int = 5) -> ProblemBatch:
    q = np.empty((P, DOF))
    g = np.empty((P, 7))
    boxes = np.empty((P, n_boxes, 6))
    imgs = None
    if image_shape is not None:
        imgs = np.empty((P, n_images) + tuple(image_shape), dtype=np.float32)
    for i in range(P):
        p = p0 + i
        r = _rng(seed, p, STREAM_PROBLEM)
        q[i] = sample_q_start(r)
        g[i] = sample_goal(r)
        boxes[i] = sample_boxes(_rng(seed, p, STREAM_BOXES), n_boxes)
        if imgs is not None:
            ri = _rng(seed, p, STREAM_IMAGE)
            for m in range(n_images):
                imgs[i, m] = synth_depth_image(ri, image_shape[0], image_shape[1], n_rect)
    return ProblemBatch(p0=p0, q_start=q.astype(np.float32), goal=g.astype(np.float32),
                        boxes=boxes.astype(np.float32), images=imgs)


def config0_problems(P: int = 1, p0: int = 0, seed: int = 0) -> ProblemBatch:
    return make_problems(P, p0, seed, image_shape=(128, 128), n_images=1, n_rect=5)


def config3_problems(P: int = 1024, p0: int = 0, seed: int = 0) -> ProblemBatch:
    return make_problems(P, p0, seed, image_shape=(240, 320), n_images=2, n_rect=8)


def config3_wide(P: int, p0: int = 0, seed: int = 0, h: float = 0.025):
    """Config-3 inputs in a 128^3 grid at 2.5 cm (a 3.2 m cube) with the robot base at its centre
    -> (ProblemBatch, GridSpec, DHRobot).  At config 3's own 1 cm / 1.28 m grid every seed of the
    random-init U-Net leaves the ESDF extent (the 7 links reach ~1.6 m from the centre) and no
    seed is feasible, so feasibility flags carry no information there; in this scene ~1 seed in 8
    is feasible and none leaves the grid (used by the flag-agreement tests and tools/agreement.py)."""
    import dataclasses

    from .spec import make_bl_robot
    grid = GridSpec(h=h, cube=128 * h)
    robot = dataclasses.replace(make_bl_robot(), base=np.full(3, 64 * h))
    pb = config3_problems(P, p0=p0, seed=seed)
    pb.boxes = np.stack([sample_boxes(_rng(seed, p0 + i, STREAM_BOXES), N_BOXES, grid)
                         for i in range(P)]).astype(np.float32)
    return pb, grid, robot


def refine_init(n_traj: int, t_len: int = 32, t0: int = 0, seed: int = 0,
                noise: float = 0.2) -> np.ndarray:
    """BASELINE config 2 seeds: straight line q_start -> q_goal (both uniform within the
    limits) plus N(0, noise^2) on rows 1..T-1; row 0 is the start (pinned)."""
    out = np.empty((n_traj, t_len, DOF))
    alphas = np.linspace(0.0, 1.0, t_len)[:, None]
    for i in range(n_traj):
        r = _rng(seed, t0 + i, STREAM_REFINE)
        qa = r.uniform(-JOINT_LIMIT, JOINT_LIMIT, size=DOF)
        qb = r.uniform(-JOINT_LIMIT, JOINT_LIMIT, size=DOF)
        tr = qa[None, :] + alphas * (qb - qa)[None, :]
        tr[1:] += noise * r.standard_normal((t_len - 1, DOF))
        out[i] = tr
    return out.astype(np.float32)
