"""Pinned choices for the BASELINE ("BL") profile of the seeding hot path.

The reference package (`planseed`, /root/reference/pkg/src/planseed) implements a
planar arm, a fully connected denoiser and 5-step DDIM.  BASELINE.json asks for the
3-D variant: a 7-joint DH chain with 50 collision spheres, a 128^3 ESDF, a depth-image
CNN encoder, a 1-D temporal U-Net and 100-step squared-cosine DDPM.  Everything the
configs leave open is pinned here, once, and cited by the kernels, the host layer
and the oracle.  SURVEY.md §8(d) lists the same choices.

Reference anchors for the generalisations:
  * joint limits +-2.8973              planseed/arm.py:79-85
  * normalisation u=(q-lo)/(hi-lo)     planseed/arm.py:195-201
  * numpy.gradient stencil D           planseed/trajopt.py:64-73
  * grid convention + clamp semantics  planseed/_kernels.py:23-57, geometry.py:176-240
  * hinge^2 world cost, row-0 pin      planseed/_kernels.py:206-228, :296-299
  * 1-based step index, x0 clip        planseed/diffusion.py:32-51, :529-556
  * sinusoid with (half-1) denominator planseed/diffusion.py:228-234
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

JOINT_LIMIT = 2.8973          # planseed/arm.py:84
DOF = 7
T_DEFAULT = 32
X0_CLIP = (-0.1, 1.1)         # planseed/diffusion.py:532

# ----------------------------------------------------------------------------
# Robot: 7 revolute standard-DH joints + 50 collision spheres
# ----------------------------------------------------------------------------

ROBOT_SEED = 7
N_SPHERES = 50


@dataclass(frozen=True)
class DHRobot:
    """Standard DH chain: frame_k = frame_{k-1} * Rz(q_k) Tz(d_k) Tx(a_k) Rx(alpha_k).

    Spheres are rigidly attached to the frame after joint `sphere_link[i]` (0-based
    link index k => frame k+1) at `sphere_offset[i]` in that frame.  The sphere table
    is sorted by link (stable), which fixes the canonical accumulation order.
    """

    a: np.ndarray            # (7,) link lengths, m
    d: np.ndarray            # (7,) link offsets, m
    alpha: np.ndarray        # (7,) link twists, rad
    base: np.ndarray         # (3,) base position in the ESDF frame
    lo: np.ndarray           # (7,) joint limits
    hi: np.ndarray
    sphere_link: np.ndarray  # (S,) int32, sorted ascending
    sphere_offset: np.ndarray  # (S,3)
    sphere_radius: np.ndarray  # (S,)

    @property
    def dof(self) -> int:
        return int(self.a.shape[0])

    @property
    def n_spheres(self) -> int:
        return int(self.sphere_radius.shape[0])

    def dh_table_f32(self) -> np.ndarray:
        """(7,4) float32 rows (a, d, cos alpha, sin alpha) -- the device layout."""
        return np.stack([self.a, self.d, np.cos(self.alpha), np.sin(self.alpha)],
                        axis=1).astype(np.float32)

    def sphere_table_f32(self) -> np.ndarray:
        """(S,4) float32 rows (x, y, z, r) in the link frame; link ids separately."""
        return np.concatenate([self.sphere_offset, self.sphere_radius[:, None]],
                              axis=1).astype(np.float32)


def make_bl_robot(seed: int = ROBOT_SEED, n_spheres: int = N_SPHERES) -> DHRobot:
    """The BASELINE robot: a ~ U(0.1, 0.35), d ~ U(0, 0.08), a fixed Franka-like twist
    table alpha = (-pi/2, pi/2, pi/2, -pi/2, pi/2, pi/2, 0);
    sphere i sits on link i % 7 at fraction f ~ U(0,1) back along x_k with a +-2 cm
    lateral jitter, radius ~ U(0.03, 0.08)."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.1, 0.35, size=DOF)
    d = rng.uniform(0.0, 0.08, size=DOF)
    h = math.pi / 2
    alpha = np.array([-h, h, h, -h, h, h, 0.0])[:DOF]
    link = np.arange(n_spheres) % DOF
    frac = rng.uniform(0.0, 1.0, size=n_spheres)
    jitter = rng.uniform(-0.02, 0.02, size=(n_spheres, 2))
    radius = rng.uniform(0.03, 0.08, size=n_spheres)
    # In frame k the link-k segment runs from (-a_k, 0, 0) (joint k axis foot, up to
    # the d_k offset along the previous z) to the origin.
    offset = np.column_stack([-frac * a[link], jitter[:, 0], jitter[:, 1]])
    order = np.argsort(link, kind="stable")
    lim = JOINT_LIMIT
    return DHRobot(
        a=a, d=d, alpha=alpha, base=np.array([0.64, 0.64, 0.64]),
        lo=np.full(DOF, -lim), hi=np.full(DOF, lim),
        sphere_link=link[order].astype(np.int32),
        sphere_offset=offset[order], sphere_radius=radius[order],
    )


# ----------------------------------------------------------------------------
# ESDF grid: 128^3 nodes at 1 cm, node (i,j,k) at origin + h*(i,j,k), C-order
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class GridSpec:
    n: Tuple[int, int, int] = (128, 128, 128)
    h: float = 0.01
    origin: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    cube: float = 1.28

    @property
    def n_nodes(self) -> int:
        return self.n[0] * self.n[1] * self.n[2]

    @property
    def cap(self) -> float:
        """Distance reported when a scene has no obstacles (planseed geometry.py:98-101
        uses the bounds diagonal)."""
        return float(self.cube * math.sqrt(3.0))


N_BOXES = 20
BOX_SIDE = (0.05, 0.4)

# ----------------------------------------------------------------------------
# Refinement cost and fixed-step optimiser
# ----------------------------------------------------------------------------


@dataclass(frozen=True)
class BLCost:
    """world: w_coll * sum hinge(r + margin - d)^2 ;
    smooth: w_vel |Dq|^2 + w_acc |D^2 q|^2 + w_jerk |D^3 q|^2 per joint;
    update: q <- q - eta * grad, row 0 pinned (gradient zeroed)."""

    w_coll: float = 50.0
    w_vel: float = 0.5
    w_acc: float = 1.0
    w_jerk: float = 1.0
    margin: float = 0.01
    eta: float = 1e-3
    n_iters: int = 10

    def as_f32(self) -> np.ndarray:
        return np.array([self.w_coll, self.w_vel, self.w_acc, self.w_jerk,
                         self.margin, self.eta], dtype=np.float32)


INTERP_PER_SEG = 4  # planseed/pipeline.py:139-157 dense check

# Ground-truth evaluation (trajopt.metrics / retime, planseed/trajopt.py:209-272): planseed's
# per-joint limits (arm.py:48-53) and the PlanRequest success thresholds (pipeline.py:37-60).
# BL end pose: the frame after joint 7; goal xyz is relative to the robot base, the goal
# quaternion (w, x, y, z) is the end-effector orientation in the base (= world) axes.
VEL_LIMIT, ACC_LIMIT, JERK_LIMIT = 2.1, 15.0, 7500.0
DELTA_T, DELTA_R_DEG = 0.005, 2.86

# ----------------------------------------------------------------------------
# Observation encoder (depth CNN) and condition vector
# ----------------------------------------------------------------------------

DEPTH_SCALE = 2.0        # background depth ~ U(0.3, 2.0) -> features depth / 2.0
GOAL_EXTENT = 0.6        # goal xyz ~ U[-0.6, 0.6]^3 -> features xyz / 0.6


@dataclass(frozen=True)
class EncoderArch:
    channels: Tuple[int, ...] = (32, 64, 128, 256)   # conv3x3 stride 2 pad 1, ReLU
    in_channels: int = 1

    @property
    def embed(self) -> int:
        return self.channels[-1]


ENCODER_CFG0 = EncoderArch()
ENCODER_CFG3 = EncoderArch(channels=(32, 64, 128, 256, 256))

COND_DIM = 256 + DOF + 7   # image embedding + normalised q_start + (goal xyz/0.6, quat)

# ----------------------------------------------------------------------------
# 1-D temporal U-Net noise predictor
# ----------------------------------------------------------------------------

T_EMB = 128
T_HIDDEN = 512
GN_GROUPS = 8
GN_EPS = 1e-5
KSIZE = 5


@dataclass(frozen=True)
class ResBlockSpec:
    name: str
    c_in: int
    c_out: int
    level: int          # time resolution T >> level


@dataclass(frozen=True)
class UNetArch:
    """Down (64,128,256) x 2 residual blocks, 2 mid blocks, up path with skip concat,
    conv3 s2 downsampling, transposed conv4 s2 upsampling, final conv5+GN+Mish and a
    1x1 projection to 7 joints.  FiLM (scale, shift) per residual block from
    Linear(Mish([t_emb 128 ; cond 270])).  72.8 MFLOP per trajectory-step at T=32."""

    dof: int = DOF
    dims: Tuple[int, ...] = (64, 128, 256)
    cond_dim: int = COND_DIM

    @property
    def film_in(self) -> int:
        return T_EMB + self.cond_dim

    def blocks(self) -> List[ResBlockSpec]:
        d = self.dims
        return [
            ResBlockSpec("d0r0", self.dof, d[0], 0), ResBlockSpec("d0r1", d[0], d[0], 0),
            ResBlockSpec("d1r0", d[0], d[1], 1), ResBlockSpec("d1r1", d[1], d[1], 1),
            ResBlockSpec("d2r0", d[1], d[2], 2), ResBlockSpec("d2r1", d[2], d[2], 2),
            ResBlockSpec("m0", d[2], d[2], 2), ResBlockSpec("m1", d[2], d[2], 2),
            ResBlockSpec("u0r0", 2 * d[2], d[1], 2), ResBlockSpec("u0r1", d[1], d[1], 2),
            ResBlockSpec("u1r0", 2 * d[1], d[0], 1), ResBlockSpec("u1r1", d[0], d[0], 1),
        ]

    def film_channels(self) -> int:
        return sum(b.c_out for b in self.blocks())

    def param_shapes(self) -> List[Tuple[str, Tuple[int, ...]]]:
        d = self.dims
        s: List[Tuple[str, Tuple[int, ...]]] = [
            ("t_fc1_w", (T_EMB, T_HIDDEN)), ("t_fc1_b", (T_HIDDEN,)),
            ("t_fc2_w", (T_HIDDEN, T_EMB)), ("t_fc2_b", (T_EMB,)),
        ]

        def res(b: ResBlockSpec):
            n, ci, co = b.name, b.c_in, b.c_out
            out = [(f"{n}_c0_w", (co, ci, KSIZE)), (f"{n}_c0_b", (co,)),
                   (f"{n}_gn0_g", (co,)), (f"{n}_gn0_b", (co,)),
                   (f"{n}_c1_w", (co, co, KSIZE)), (f"{n}_c1_b", (co,)),
                   (f"{n}_gn1_g", (co,)), (f"{n}_gn1_b", (co,)),
                   (f"{n}_film_w", (self.film_in, 2 * co)), (f"{n}_film_b", (2 * co,))]
            if ci != co:
                out += [(f"{n}_res_w", (co, ci, 1)), (f"{n}_res_b", (co,))]
            return out

        blocks = {b.name: b for b in self.blocks()}
        for n in ("d0r0", "d0r1"):
            s += res(blocks[n])
        s += [("down0_w", (d[0], d[0], 3)), ("down0_b", (d[0],))]
        for n in ("d1r0", "d1r1"):
            s += res(blocks[n])
        s += [("down1_w", (d[1], d[1], 3)), ("down1_b", (d[1],))]
        for n in ("d2r0", "d2r1", "m0", "m1", "u0r0", "u0r1"):
            s += res(blocks[n])
        # ConvTranspose1d weight layout (C_in, C_out, K) as in torch
        s += [("up0_w", (d[1], d[1], 4)), ("up0_b", (d[1],))]
        for n in ("u1r0", "u1r1"):
            s += res(blocks[n])
        s += [("up1_w", (d[0], d[0], 4)), ("up1_b", (d[0],))]
        s += [("fin_c_w", (d[0], d[0], KSIZE)), ("fin_c_b", (d[0],)),
              ("fin_gn_g", (d[0],)), ("fin_gn_b", (d[0],)),
              ("out_w", (self.dof, d[0], 1)), ("out_b", (self.dof,))]
        return s

    def n_params(self) -> int:
        return int(sum(np.prod(sh) for _, sh in self.param_shapes()))

    def flops_per_traj_step(self, t_len: int = T_DEFAULT) -> int:
        """Algorithmic FLOPs (2 x MAC) of one noise prediction for one trajectory,
        FiLM and the step MLP excluded (they are per (problem, step))."""
        mac = 0
        for name, sh in self.param_shapes():
            if not name.endswith("_w") or name.startswith("t_fc") or "_film_" in name:
                continue
            lvl = _level_of(name)
            t_out = t_len >> lvl
            if name.startswith("down"):
                t_out = t_len >> (lvl + 1)
                mac += sh[0] * sh[1] * sh[2] * t_out
            elif name.startswith("up"):
                t_in = t_len >> lvl
                mac += sh[0] * sh[1] * sh[2] * t_in
            else:
                mac += sh[0] * sh[1] * sh[2] * t_out
        return 2 * mac

    def film_flops(self) -> int:
        return 2 * self.film_in * 2 * self.film_channels()


def _level_of(pname: str) -> int:
    p = pname.split("_")[0]
    table = {"d0r0": 0, "d0r1": 0, "down0": 0, "d1r0": 1, "d1r1": 1, "down1": 1,
             "d2r0": 2, "d2r1": 2, "m0": 2, "m1": 2, "u0r0": 2, "u0r1": 2, "up0": 2,
             "u1r0": 1, "u1r1": 1, "up1": 1, "fin": 0, "out": 0}
    return table[p]


def encoder_param_shapes(enc: EncoderArch) -> List[Tuple[str, Tuple[int, ...]]]:
    s = []
    c_prev = enc.in_channels
    for i, c in enumerate(enc.channels):
        s += [(f"enc{i}_w", (c, c_prev, 3, 3)), (f"enc{i}_b", (c,))]
        c_prev = c
    return s


def init_params(shapes, seed: int = 0) -> dict:
    """Seeded uniform fan-in init, drawn in table order from default_rng(seed)
    (the planseed convention, diffusion.py:185-200).  Unlike planseed, biases,
    GroupNorm affines and FiLM are NOT zero: with random weights a zero FiLM would
    leave the condition path untested."""
    rng = np.random.default_rng(seed)
    fan = {}
    out = {}
    for name, sh in shapes:
        stem = name.rsplit("_", 1)[0]
        if name.endswith("_w"):
            if name.startswith(("t_fc", )) or "_film_" in name:
                fan_in = sh[0]                       # Linear (in, out)
            elif name.startswith("up"):
                fan_in = sh[0] * sh[2]               # ConvTranspose (C_in, C_out, K)
            else:
                fan_in = int(np.prod(sh[1:]))        # Conv (C_out, C_in, K...)
            fan[stem] = fan_in
            b = 1.0 / math.sqrt(fan_in)
            out[name] = rng.uniform(-b, b, size=sh)
        elif "_gn" in name and name.endswith("_g"):
            out[name] = 1.0 + rng.uniform(-0.1, 0.1, size=sh)
        elif "_gn" in name:
            out[name] = rng.uniform(-0.1, 0.1, size=sh)
        else:  # bias
            b = 1.0 / math.sqrt(fan.get(stem, sh[0]))
            out[name] = rng.uniform(-b, b, size=sh)
    return out


# ----------------------------------------------------------------------------
# Noise schedule and sampler
# ----------------------------------------------------------------------------

K_STEPS = 100
COSINE_S = 0.008
NOISE_SEED = 1
WEIGHT_SEED = 0


def cosine_betas(K: int = K_STEPS, s: float = COSINE_S, max_beta: float = 0.999) -> np.ndarray:
    """Squared-cosine schedule: abar(t) = f(t)/f(0), f(t) = cos^2(((t/K)+s)/(1+s) pi/2),
    beta_t = min(1 - abar(t)/abar(t-1), max_beta), t = 1..K (float64)."""
    def f(t):
        return math.cos(((t / K) + s) / (1.0 + s) * math.pi / 2.0) ** 2
    betas = [min(1.0 - f(t) / f(t - 1), max_beta) for t in range(1, K + 1)]
    return np.array(betas, dtype=np.float64)


# Strided DDIM in bf16 (mode 1).  The x0 reconstruction multiplies the noise prediction by
# 1/sqrt(abar_k): 2029 at k = 100, 5.9 at k = 89, 3.0 at k = 78 in the 10-step schedule, and the
# deterministic update carries every error forward, so bf16-level noise-prediction differences end
# ~0.37 rad RMS from the float64 oracle (fp32: 6e-5).  A schedule whose first x0 factor exceeds
# DDIM_BF16_MAX_RSQ is numerically unqualified in bf16 (SeedSampler warns).  SeedSampler(hp_rsq=h)
# runs the leading steps with factor > h on the fp32 network: h = 4 (2 fp32 steps) measured 0.068
# rad RMS, h = 2.5 (3 steps) 0.037, at 6-9x the sampler time at 1024 x 32.
DDIM_BF16_MAX_RSQ = 50.0
HP_RSQ = 4.0


def strided_steps(K: int, n_steps: int) -> np.ndarray:
    """round-half-even(linspace(K, 1, n)) -- planseed/diffusion.py:520-526."""
    if n_steps > K:
        raise ValueError("n_steps cannot exceed K")
    if n_steps == 1:
        return np.array([K], dtype=np.int64)
    return np.round(np.linspace(K, 1, n_steps)).astype(np.int64)


@dataclass(frozen=True)
class SamplerTables:
    """Per-step float32 coefficient tables, indexed by the 1-based step k (row 0 unused).

    x0  = clip((x - sq1m[k] * eps) * rsq[k], clip)
    DDPM: x' = c0[k] * x0 + c1[k] * x + sig[k] * z     (k > 1)
    DDIM: x' = sq[k'] * x0 + sq1m[k'] * eps             (next index k')
    """

    sq: np.ndarray
    sq1m: np.ndarray
    rsq: np.ndarray
    c0: np.ndarray
    c1: np.ndarray
    sig: np.ndarray


def sampler_tables(betas: np.ndarray, dtype=np.float32) -> SamplerTables:
    """float32 by default (the device tables); dtype=np.float64 keeps the exact coefficients
    (used by the oracle's bridge to planseed's float64 sampler)."""
    K = betas.shape[0]
    ab = np.cumprod(1.0 - betas)
    ab_prev = np.concatenate([[1.0], ab[:-1]])
    al = 1.0 - betas
    z = np.zeros(1)
    c0 = np.sqrt(ab_prev) * betas / (1.0 - ab)
    c1 = np.sqrt(al) * (1.0 - ab_prev) / (1.0 - ab)
    var = betas * (1.0 - ab_prev) / (1.0 - ab)
    f = lambda a: np.concatenate([z, a]).astype(dtype)
    return SamplerTables(sq=f(np.sqrt(ab)), sq1m=f(np.sqrt(1.0 - ab)), rsq=f(1.0 / np.sqrt(ab)),
                         c0=f(c0), c1=f(c1), sig=f(np.sqrt(var)))


def timestep_sinusoid(k, dim: int = T_EMB) -> np.ndarray:
    """[sin(k w_i), cos(k w_i)], w_i = exp(-ln(1e4) i / (half-1)) -- diffusion.py:228-234."""
    k = np.atleast_1d(np.asarray(k, dtype=np.float64))
    half = dim // 2
    freqs = np.exp(-np.log(10000.0) * np.arange(half) / max(half - 1, 1))
    ang = k[:, None] * freqs[None, :]
    return np.concatenate([np.sin(ang), np.cos(ang)], axis=1)


# ----------------------------------------------------------------------------
# Counter-based noise: Philox4x32-10 + Box-Muller
# ----------------------------------------------------------------------------
# counter = (block, step, global_problem, seed_index), key = (noise_seed, KEY_HI)
# block b yields elements 4b..4b+3 of the (T, D) trajectory noise, row-major.
# step = 0 draws x_K; step = k draws the posterior noise of the k -> k-1 update.
# u1 = ((r0 >> 8) + 1) * 2^-24 in (0,1], u2 = (r1 >> 8) * 2^-24 in [0,1)
# z0 = sqrt(-2 ln u1) cos(2 pi u2), z1 = sqrt(-2 ln u1) sin(2 pi u2); same for r2,r3.
PHILOX_KEY_HI = 0x5EED5EED


def model_param_shapes(enc: EncoderArch = ENCODER_CFG0, arch: UNetArch = UNetArch()):
    """Encoder table followed by the U-Net table; the PSCK blob order."""
    return encoder_param_shapes(enc) + arch.param_shapes()


def random_model(enc: EncoderArch = ENCODER_CFG0, arch: UNetArch = UNetArch(),
                 seed: int = WEIGHT_SEED) -> dict:
    """BASELINE random-init weights ("weights seed 0"), float64 host arrays."""
    return init_params(model_param_shapes(enc, arch), seed)
