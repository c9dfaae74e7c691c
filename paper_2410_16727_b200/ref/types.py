"""Host-side types of the reference-profile API, compatible field-for-field with
planseed's (src/arm.py:13-85, src/geometry.py:16-276) so that either package's
objects can be passed to the drop-in functions (duck typing on the attributes the
kernels read).  These are data containers and input adapters, not compute."""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Tuple

import numpy as np

DEFAULT_N_RAYS = 256
DEFAULT_FOV = np.pi / 2


def wrap_angle(theta):
    """Wrap to (-pi, pi] (src/geometry.py:16-18)."""
    return np.pi - np.mod(np.pi - np.asarray(theta), 2.0 * np.pi)


@dataclass(frozen=True)
class Rect:
    lo: Tuple[float, float]
    hi: Tuple[float, float]

    @property
    def extent(self) -> np.ndarray:
        return np.array(self.hi) - np.array(self.lo)

    @property
    def diagonal(self) -> float:
        return float(np.hypot(*self.extent))


WORKSPACE = Rect((-1.0, -1.0), (1.0, 1.0))


@dataclass(frozen=True)
class Pose2:
    position: Tuple[float, float]
    theta: float

    def __post_init__(self):
        object.__setattr__(self, "theta", float(wrap_angle(self.theta)))

    @property
    def pos(self) -> np.ndarray:
        return np.asarray(self.position, dtype=np.float64)


@dataclass(frozen=True)
class ArmModel:
    """Planar revolute chain with cumulative joint angles (src/arm.py:28-76)."""

    lengths: np.ndarray
    lo: np.ndarray
    hi: np.ndarray
    base: np.ndarray = field(default_factory=lambda: np.zeros(2))
    points_per_link: int = 4
    vel_limit: np.ndarray = None
    acc_limit: np.ndarray = None
    jerk_limit: np.ndarray = None

    def __post_init__(self):
        for n in ("lengths", "lo", "hi", "base"):
            object.__setattr__(self, n, np.asarray(getattr(self, n), dtype=np.float64))
        d = self.lengths.shape[0]
        for n, v in (("vel_limit", 2.1), ("acc_limit", 15.0), ("jerk_limit", 7500.0)):   # src/arm.py:48-53
            cur = getattr(self, n)
            object.__setattr__(self, n, np.full(d, v) if cur is None else np.asarray(cur, dtype=np.float64))
        if np.any(self.lengths <= 0):
            raise ValueError("link lengths must be positive")
        if np.any(self.lo >= self.hi):
            raise ValueError("joint limits must satisfy lo < hi")

    @property
    def dof(self) -> int:
        return int(self.lengths.shape[0])

    def point_fractions(self) -> np.ndarray:
        m = self.points_per_link
        return (np.arange(m) + 0.5) / m


def default_arm(dof: int = 7) -> ArmModel:
    if dof > 7:
        raise ValueError("default arm supports up to 7 joints")
    lengths = np.array([0.16, 0.14, 0.13, 0.12, 0.11, 0.10, 0.09])[:dof]
    lim = 2.8973
    return ArmModel(lengths=lengths, lo=np.full(dof, -lim), hi=np.full(dof, lim))


def fk_pose(arm, q) -> Pose2:
    th = np.cumsum(np.asarray(q, dtype=np.float64))
    x = arm.base[0] + float(np.dot(arm.lengths, np.cos(th)))
    y = arm.base[1] + float(np.dot(arm.lengths, np.sin(th)))
    return Pose2(position=(x, y), theta=float(th[-1]))


def normalize(arm, q):
    return (np.asarray(q, dtype=np.float64) - arm.lo) / (arm.hi - arm.lo)


def denormalize(arm, u):
    return arm.lo + np.asarray(u, dtype=np.float64) * (arm.hi - arm.lo)


def nonadjacent_point_pairs(arm):
    """Point index pairs on links at least two apart (src/arm.py:204-214)."""
    m = arm.points_per_link
    ii, jj = [], []
    for a in range(arm.dof):
        for b in range(a + 2, arm.dof):
            for pa in range(m):
                for pb in range(m):
                    ii.append(a * m + pa)
                    jj.append(b * m + pb)
    return np.array(ii, dtype=np.int64), np.array(jj, dtype=np.int64)


@dataclass
class SdfGrid:
    """Node (i, j) at origin + (i*h, j*h) (src/geometry.py:176-192)."""

    origin: np.ndarray
    h: float
    nx: int
    ny: int
    values: np.ndarray


@dataclass(frozen=True)
class SensorPose:
    position: Tuple[float, float]
    heading: float
    fov: float = DEFAULT_FOV
    n_rays: int = DEFAULT_N_RAYS
    max_range: float = 2.0 * WORKSPACE.diagonal


@dataclass(frozen=True)
class DepthScan:
    pose: SensorPose
    depths: np.ndarray


@dataclass(frozen=True)
class Circle:
    center: Tuple[float, float]
    radius: float


@dataclass(frozen=True)
class Box:
    lo: Tuple[float, float]
    hi: Tuple[float, float]


class World:
    """Ground-truth obstacle world (src/geometry.py:72-99): the flat circle / box arrays
    and the empty-world distance cap the metric kernels read."""

    def __init__(self, obstacles=(), bounds: Rect = WORKSPACE):
        self.obstacles = tuple(obstacles)
        self.bounds = bounds
        cs = [o for o in self.obstacles if isinstance(o, Circle)]
        bs = [o for o in self.obstacles if isinstance(o, Box)]
        self.circle_arr = (np.array([[c.center[0], c.center[1], c.radius] for c in cs], dtype=np.float64)
                           if cs else np.zeros((0, 3)))
        self.box_arr = (np.array([[b.lo[0], b.lo[1], b.hi[0], b.hi[1]] for b in bs], dtype=np.float64)
                        if bs else np.zeros((0, 4)))

    @property
    def sdf_cap(self) -> float:
        return self.bounds.diagonal


def render_depth_scan(world, pose):
    """geometry.render_depth_scan (src/geometry.py:326-329): the sensor's fan of rays cast
    against the world on the GPU (`ps_ref_render_scan`, fp64); depth = first hit, max_range
    otherwise.  Accepts planseed's World / SensorPose or this module's."""
    from .. import _lib
    torch = _lib.require_cuda()
    dev = lambda a, w: torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1, w)),
                                       device="cuda")
    circ, box = dev(world.circle_arr, 3), dev(world.box_arr, 4)
    n = int(pose.n_rays)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    st = _lib.lib().ps_ref_render_scan(_lib.ptr(circ), circ.shape[0], _lib.ptr(box), box.shape[0],
                                       float(pose.position[0]), float(pose.position[1]), float(pose.heading),
                                       float(pose.fov), n, float(pose.max_range), _lib.ptr(out),
                                       _lib.stream_handle())
    _lib.check(st, "render_depth_scan")
    return DepthScan(pose=pose, depths=out.cpu().numpy())
