"""Drop-in for planseed.diffusion's sampler API on the GPU (src/diffusion.py).

Weights are the reference's own: `create_net` draws them exactly like planseed
(same rng, same order, same fan-in rule, zero biases and FiLM) and the PSCK
checkpoint format is read/written byte-compatibly, so a planseed checkpoint loads
here and vice versa.  The forward passes run in float64 CUDA kernels
(`ps_ref_linear`, `ps_ref_conv1d_silu`, `ps_ref_film`, `ps_ref_ddim_update`, ...);
input feature vectors (11 + 4 scalars) are formed on the host as the reference does.
"""

from __future__ import annotations

import json
import struct
from dataclasses import asdict, dataclass
from pathlib import Path
from typing import Dict, List, Optional, Tuple

import numpy as np

from .. import _lib
from .types import WORKSPACE, Rect

CKPT_MAGIC = b"PSCK"
X0_CLIP = (-0.1, 1.1)


@dataclass(frozen=True)
class NoiseSchedule:
    betas: np.ndarray

    @property
    def K(self) -> int:
        return self.betas.shape[0]

    @property
    def alpha_bars(self) -> np.ndarray:
        return np.cumprod(1.0 - self.betas)

    def alpha_bar(self, k):
        return self.alpha_bars[np.asarray(k) - 1]


def make_schedule(K: int = 100, beta_start: float = 1e-3, beta_end: float = 8e-2) -> NoiseSchedule:
    if K < 2:
        raise ValueError("need at least 2 diffusion steps")
    if not (0.0 < beta_start < beta_end < 1.0):
        raise ValueError("betas must satisfy 0 < beta_start < beta_end < 1")
    return NoiseSchedule(betas=np.linspace(beta_start, beta_end, K))


@dataclass(frozen=True)
class ArchConfig:
    """src/diffusion.py:84-120."""

    t_len: int = 32
    dof: int = 7
    n_rays: int = 256
    scan_channels: Tuple[int, ...] = (8, 16, 16)
    scan_kernels: Tuple[int, ...] = (5, 5, 3)
    scan_strides: Tuple[int, ...] = (2, 2, 2)
    scan_embed: int = 64
    problem_embed: int = 32
    pose_embed: int = 32
    t_embed: int = 32
    embed_hidden: int = 64
    hidden: int = 512
    n_hidden: int = 3
    joint_lo: Tuple[float, ...] = (-2.8973,) * 7
    joint_hi: Tuple[float, ...] = (2.8973,) * 7
    bounds_lo: Tuple[float, float] = WORKSPACE.lo
    bounds_hi: Tuple[float, float] = WORKSPACE.hi
    max_range: float = 2.0 * WORKSPACE.diagonal

    @property
    def cond_dim(self) -> int:
        return self.scan_embed + self.problem_embed + self.pose_embed

    @property
    def x_dim(self) -> int:
        return self.t_len * self.dof

    def conv_out_len(self) -> int:
        n = self.n_rays
        for kk, ss in zip(self.scan_kernels, self.scan_strides):
            n = (n - kk) // ss + 1
        return n

    def lo_hi(self):
        return np.array(self.joint_lo), np.array(self.joint_hi)


def arch_for_arm(arm, bounds: Rect = WORKSPACE, **overrides) -> ArchConfig:
    base = dict(dof=arm.dof, joint_lo=tuple(arm.lo.tolist()), joint_hi=tuple(arm.hi.tolist()),
                bounds_lo=tuple(bounds.lo), bounds_hi=tuple(bounds.hi), max_range=2.0 * bounds.diagonal)
    base.update(overrides)
    return ArchConfig(**base)


@dataclass
class DenoiserNet:
    config: ArchConfig
    params: Dict[str, np.ndarray]
    init_seed: int = 0


def _param_shapes(cfg) -> List[Tuple[str, Tuple[int, ...]]]:
    """Parameter table in planseed's order (src/diffusion.py:146-182)."""
    shapes = []
    c_prev = 1
    for i, (c, k) in enumerate(zip(cfg.scan_channels, cfg.scan_kernels)):
        shapes += [(f"scan_conv{i}_w", (c, c_prev, k)), (f"scan_conv{i}_b", (c,))]
        c_prev = c
    flat = cfg.scan_channels[-1] * cfg.conv_out_len()
    shapes += [("scan_fc_w", (flat, cfg.scan_embed)), ("scan_fc_b", (cfg.scan_embed,)),
               ("prob_fc1_w", (cfg.dof + 4, cfg.embed_hidden)), ("prob_fc1_b", (cfg.embed_hidden,)),
               ("prob_fc2_w", (cfg.embed_hidden, cfg.problem_embed)), ("prob_fc2_b", (cfg.problem_embed,)),
               ("pose_fc1_w", (4, cfg.embed_hidden)), ("pose_fc1_b", (cfg.embed_hidden,)),
               ("pose_fc2_w", (cfg.embed_hidden, cfg.pose_embed)), ("pose_fc2_b", (cfg.pose_embed,)),
               ("t_fc1_w", (cfg.t_embed, cfg.embed_hidden)), ("t_fc1_b", (cfg.embed_hidden,)),
               ("t_fc2_w", (cfg.embed_hidden, cfg.t_embed)), ("t_fc2_b", (cfg.t_embed,))]
    d_in = cfg.x_dim + cfg.cond_dim + cfg.t_embed
    mod_in = cfg.cond_dim + cfg.t_embed
    for i in range(cfg.n_hidden):
        shapes += [(f"trunk{i}_w", (d_in, cfg.hidden)), (f"trunk{i}_b", (cfg.hidden,)),
                   (f"trunk{i}_scale_w", (mod_in, cfg.hidden)), (f"trunk{i}_scale_b", (cfg.hidden,)),
                   (f"trunk{i}_shift_w", (mod_in, cfg.hidden)), (f"trunk{i}_shift_b", (cfg.hidden,))]
        d_in = cfg.hidden
    shapes += [("trunk_out_w", (d_in, cfg.x_dim)), ("trunk_out_b", (cfg.x_dim,))]
    return shapes


def create_net(cfg: ArchConfig, seed: int = 0) -> DenoiserNet:
    """Uniform fan-in init, identical draws to planseed (src/diffusion.py:185-200)."""
    rng = np.random.default_rng(seed)
    params = {}
    for name, shape in _param_shapes(cfg):
        if name.endswith("_b") or "_scale_" in name or "_shift_" in name:
            params[name] = np.zeros(shape)
        else:
            fan_in = int(np.prod(shape[:-1])) if name.endswith("fc_w") or "trunk" in name \
                or "fc1" in name or "fc2" in name else int(np.prod(shape[1:]))
            bound = 1.0 / np.sqrt(max(fan_in, 1))
            params[name] = rng.uniform(-bound, bound, size=shape)
    return DenoiserNet(config=cfg, params=params, init_seed=seed)


def _host_params(net) -> Dict[str, np.ndarray]:
    return {k: np.asarray(getattr(v, "data", v), dtype=np.float64) for k, v in net.params.items()}


# scalar type of the device path: "fp64" is planseed's parity mode, "fp32" the fast mode
_DTN = {"fp64": 0, "fp32": 1}


def _tdt(dtype: str):
    torch = _lib.require_cuda()
    if dtype not in _DTN:
        raise ValueError("dtype must be 'fp64' or 'fp32'")
    return torch.float64 if dtype == "fp64" else torch.float32


def _dt_of(t) -> int:
    torch = _lib.require_cuda()
    return 0 if t.dtype == torch.float64 else 1


def _dev_params(net, dtype: str = "fp64"):
    """Device copies of the weights in `dtype` (rounded once from float64), cached on the net object."""
    torch = _lib.require_cuda()
    tdt = _tdt(dtype)
    cache = getattr(net, "_ps_dev", None)
    if cache is None:
        cache = {}
        try:
            object.__setattr__(net, "_ps_dev", cache)
        except Exception:
            pass
    if dtype not in cache:
        cache[dtype] = {k: torch.as_tensor(np.ascontiguousarray(v), device="cuda").to(tdt)
                        for k, v in _host_params(net).items()}
    return cache[dtype]


# ----------------------------------------------------------------------------- features
def _norm_pos(cfg, p):
    lo = np.array(cfg.bounds_lo)
    return (np.asarray(p, dtype=np.float64) - lo) / (np.array(cfg.bounds_hi) - lo)


def problem_features(cfg, q0, goal) -> np.ndarray:
    lo, hi = cfg.lo_hi()
    q0n = (np.asarray(q0, dtype=np.float64) - lo) / (hi - lo)
    g = _norm_pos(cfg, goal.pos)
    return np.concatenate([q0n, [g[0], g[1], np.cos(goal.theta), np.sin(goal.theta)]])


def pose_features(cfg, pose) -> np.ndarray:
    p = _norm_pos(cfg, pose.position)
    return np.array([p[0], p[1], np.cos(pose.heading), np.sin(pose.heading)])


def ddim_steps(K: int, n_steps: int) -> np.ndarray:
    """src/diffusion.py:520-526 (numpy round-half-even)."""
    if n_steps > K:
        raise ValueError("n_steps cannot exceed K")
    if n_steps == 1:
        return np.array([K], dtype=np.int64)
    return np.round(np.linspace(K, 1, n_steps)).astype(np.int64)


# ----------------------------------------------------------------------------- forward
def _linear(x, W, b, act: int, out=None):
    torch = _lib.require_cuda()
    R, K = x.shape
    N = W.shape[1]
    y = out if out is not None else torch.empty((R, N), dtype=x.dtype, device="cuda")
    _lib.check(_lib.lib().ps_ref_linear_dt(_dt_of(x), _lib.ptr(x), x.stride(0), _lib.ptr(W), _lib.ptr(b), R, K, N,
                                           act, _lib.ptr(y), y.stride(0), _lib.stream_handle()), "linear")
    return y


def _mlp2(p, prefix, x):
    return _linear(_linear(x, p[f"{prefix}_fc1_w"], p[f"{prefix}_fc1_b"], 1),
                   p[f"{prefix}_fc2_w"], p[f"{prefix}_fc2_b"], 0)


def condition_device(net, depths, prob_feats, pose_feats, dtype: str = "fp64"):
    """condition_graph (src/diffusion.py:246-257) for one observation -> (1, cond_dim) device."""
    torch = _lib.require_cuda()
    tdt = _tdt(dtype)
    cfg, p = net.config, _dev_params(net, dtype)
    L = _lib.lib()
    dt = _DTN[dtype]
    d = torch.as_tensor(np.asarray(depths, dtype=np.float64), device="cuda").to(tdt).contiguous()
    h = torch.empty_like(d)
    _lib.check(L.ps_ref_div_dt(dt, _lib.ptr(d), d.numel(), float(cfg.max_range), _lib.ptr(h),
                               _lib.stream_handle()), "scan_features")
    C, Ln = 1, cfg.n_rays
    for i, (c, kk, ss) in enumerate(zip(cfg.scan_channels, cfg.scan_kernels, cfg.scan_strides)):
        lo = (Ln - kk) // ss + 1
        y = torch.empty(c * lo, dtype=tdt, device="cuda")
        _lib.check(L.ps_ref_conv1d_silu_dt(dt, _lib.ptr(h), C, Ln, _lib.ptr(p[f"scan_conv{i}_w"]),
                                           _lib.ptr(p[f"scan_conv{i}_b"]), c, kk, ss, _lib.ptr(y),
                                           _lib.stream_handle()), "conv1d")
        h, C, Ln = y, c, lo
    scan_emb = _linear(h.view(1, -1), p["scan_fc_w"], p["scan_fc_b"], 0)
    pf = torch.as_tensor(np.asarray(prob_feats, dtype=np.float64)[None], device="cuda").to(tdt)
    qf = torch.as_tensor(np.asarray(pose_feats, dtype=np.float64)[None], device="cuda").to(tdt)
    return torch.cat([scan_emb, _mlp2(p, "prob", pf), _mlp2(p, "pose", qf)], dim=1)


def encode_condition(net, scan, q0, goal, dtype: str = "fp64") -> np.ndarray:
    """src/diffusion.py:260-269 (float64 result; dtype="fp32" runs the fast mode)."""
    cfg = net.config
    c = condition_device(net, scan.depths, problem_features(cfg, q0, goal), pose_features(cfg, scan.pose), dtype)
    return c.cpu().numpy().astype(np.float64)[0]


def predict_noise_device(net, x, k: int, cond):
    """predict_noise_graph (src/diffusion.py:272-285); x (B,T,D) and cond (1,C) device tensors of
    one scalar type (float64 parity mode or float32 fast mode)."""
    torch = _lib.require_cuda()
    dtype = "fp64" if x.dtype == torch.float64 else "fp32"
    cfg, p = net.config, _dev_params(net, dtype)
    L = _lib.lib()
    B = x.shape[0]
    half = cfg.t_embed // 2
    tf = torch.empty((1, cfg.t_embed), dtype=x.dtype, device="cuda")
    _lib.check(L.ps_ref_sinusoid_dt(_DTN[dtype], float(k), half, _lib.ptr(tf), _lib.stream_handle()), "sinusoid")
    t_emb = _mlp2(p, "t", tf)
    cond = cond.to(x.dtype)
    mod = torch.cat([cond, t_emb], dim=1)
    h = torch.cat([x.reshape(B, cfg.x_dim), cond.expand(B, -1), t_emb.expand(B, -1)], dim=1).contiguous()
    for i in range(cfg.n_hidden):
        h = _linear(h, p[f"trunk{i}_w"], p[f"trunk{i}_b"], 1)
        sc = _linear(mod, p[f"trunk{i}_scale_w"], p[f"trunk{i}_scale_b"], 0)
        sh = _linear(mod, p[f"trunk{i}_shift_w"], p[f"trunk{i}_shift_b"], 0)
        _lib.check(L.ps_ref_film_dt(_DTN[dtype], _lib.ptr(h), _lib.ptr(sc), _lib.ptr(sh), B, h.shape[1],
                                    _lib.stream_handle()), "film")
    return _linear(h, p["trunk_out_w"], p["trunk_out_b"], 0).view(B, cfg.t_len, cfg.dof)


def predict_noise(net, x_k, k, cond, K: int = 100, dtype: str = "fp64") -> np.ndarray:
    """src/diffusion.py:288-300: x_k (T,D) or (B,T,D), one cond row broadcast."""
    torch = _lib.require_cuda()
    x = np.asarray(x_k, dtype=np.float64)
    single = x.ndim == 2
    if single:
        x = x[None]
    if np.ndim(k) != 0:
        raise ValueError("per-row step indices are not supported by the drop-in sampler")
    c = np.atleast_2d(np.asarray(cond, dtype=np.float64))
    if c.shape[0] != 1:
        raise ValueError("one condition row per call (the reference broadcasts a single row)")
    tdt = _tdt(dtype)
    xd = torch.as_tensor(x, device="cuda").to(tdt)
    cd = torch.as_tensor(c, device="cuda").to(tdt)
    out = predict_noise_device(net, xd, int(k), cd).cpu().numpy().astype(np.float64)
    return out[0] if single else out


def ddim_sample_device(net, schedule, cond, x_K, q0, arm, n_steps: int = 5, dtype: str = "fp64"):
    """_ddim_core + ddim_sample (src/diffusion.py:535-569) on the device, in float64 (parity mode)
    or float32 (fast mode); the schedule coefficients are formed in float64 either way."""
    torch = _lib.require_cuda()
    tdt = _tdt(dtype)
    dt = _DTN[dtype]
    L = _lib.lib()
    ks = ddim_steps(schedule.K, n_steps)
    x = torch.as_tensor(np.array(x_K, dtype=np.float64), device="cuda").to(tdt)
    single = x.dim() == 2
    if single:
        x = x[None]
    x = x.contiguous()
    cd = torch.as_tensor(np.atleast_2d(np.asarray(cond, dtype=np.float64)), device="cuda").to(tdt)
    x0 = torch.empty_like(x)
    n = x.numel()
    for i, k in enumerate(ks):
        ab = float(schedule.alpha_bar(int(k)))
        eps = predict_noise_device(net, x, int(k), cd)
        has_next = i + 1 < len(ks)
        ab_next = float(schedule.alpha_bar(int(ks[i + 1]))) if has_next else 1.0
        _lib.check(L.ps_ref_ddim_update_dt(dt, _lib.ptr(x), _lib.ptr(eps), n, ab, ab_next, int(has_next),
                                           X0_CLIP[0], X0_CLIP[1], _lib.ptr(x0), _lib.stream_handle()),
                   "ddim_update")
    B, T, D = x0.shape
    lo = torch.as_tensor(np.asarray(arm.lo, dtype=np.float64), device="cuda").to(tdt)
    hi = torch.as_tensor(np.asarray(arm.hi, dtype=np.float64), device="cuda").to(tdt)
    q = torch.as_tensor(np.asarray(q0, dtype=np.float64), device="cuda").to(tdt)
    traj = torch.empty_like(x0)
    _lib.check(L.ps_ref_denorm_pin_dt(dt, _lib.ptr(x0), B, T, D, _lib.ptr(lo), _lib.ptr(hi), _lib.ptr(q),
                                      _lib.ptr(traj), _lib.stream_handle()), "denormalize")
    return traj[0] if single else traj


def ddim_sample(net, schedule, cond, x_K, q0, arm, n_steps: int = 5, dtype: str = "fp64") -> np.ndarray:
    """src/diffusion.py:559-569: denoise x_K (T,D) or (B,T,D); row 0 pinned to q0 (float64 result;
    dtype="fp32" runs the fast mode; its row 0 is re-pinned to the float64 q0)."""
    out = ddim_sample_device(net, schedule, cond, x_K, q0, arm, n_steps, dtype).cpu().numpy().astype(np.float64)
    out[..., 0, :] = np.asarray(q0, dtype=np.float64)
    return out


class PlannerCost:
    """The planner's guidance cost, `evaluate_cost_batch(arm, esdf, goal, trajs, w)` ->
    (totals, grads) (src/pipeline.py:190-192).  Callable on host arrays exactly like the
    reference's closure; `guided_ddim_sample` recognises it and runs the whole guidance
    (n_grad descent steps x halvings over all seeds) as one fused GPU launch per sub-step."""

    def __init__(self, arm, esdf, goal, w=None, dtype: str = "fp64"):
        from .trajopt import CostWeights
        self.arm, self.esdf, self.goal = arm, esdf, goal
        self.w = w if w is not None else CostWeights()
        self.dtype = dtype

    def __call__(self, trajs):
        from .trajopt import evaluate_cost_batch
        totals, grads, _ = evaluate_cost_batch(self.arm, self.esdf, self.goal, trajs, self.w, dtype=self.dtype)
        return totals, grads


def _guide_device(cost: PlannerCost, arm, net, x0, n_grad, alpha_guide, max_halvings, ws):
    """One fused `ps_ref_guide` launch on x0 (B,T,D) device f64, in place; raises the
    reference's ValueError when an evaluation leaves the ESDF (src/trajopt.py:116-118)."""
    torch = _lib.require_cuda()
    from .trajopt import _DT, _ArmArgs
    B, T, D = x0.shape
    A = _ArmArgs(cost.arm, cost.esdf, cost.goal, cost.w, T, "fp64")
    lo, hi = net.config.lo_hi()
    arm_lo = ws["arm_lo"]
    flags = torch.empty(2 * B, dtype=torch.int32, device="cuda")
    err = torch.zeros(2 + B, dtype=torch.int32, device="cuda")
    st = _lib.lib().ps_ref_guide(_DT["fp64"], _lib.ptr(x0), B, T, D, *A.args, _lib.ptr(arm_lo),
                                 _lib.ptr(ws["arm_span"]), _lib.ptr(ws["net_span"]), int(n_grad),
                                 float(alpha_guide), int(max_halvings), _lib.ptr(flags), _lib.ptr(err),
                                 _lib.stream_handle())
    _lib.check(st, "guide")
    e = err.cpu().numpy()
    if e[0]:
        raise ValueError("trajectory collision points leave the ESDF extent "
                         f"(seeds {np.nonzero(e[2:])[0].tolist()})")


def _guide_host(cost_fn, arm, span, x0_hat, n_grad, alpha_guide, max_halvings):
    """guide() of src/diffusion.py:598-617 for an arbitrary user cost_fn (a host callable):
    the same loop, with the user's function evaluated on host arrays."""
    from .types import denormalize
    batched = x0_hat.ndim == 3
    x = x0_hat if batched else x0_hat[None]
    for _ in range(n_grad):
        costs, grads = cost_fn(denormalize(arm, x))
        g_norm = grads * span
        step = np.full(x.shape[0], alpha_guide)
        remaining = np.ones(x.shape[0], dtype=bool)
        for _ in range(max_halvings):
            if not remaining.any():
                break
            cand = x - step[:, None, None] * g_norm
            new_costs, _ = cost_fn(denormalize(arm, cand))
            improved = remaining & (new_costs < costs)
            x = np.where(improved[:, None, None], cand, x)
            remaining = remaining & ~improved
            step = np.where(remaining, step * 0.5, step)
    return x if batched else x[0]


def guided_ddim_sample_device(net, schedule, cond, x_K, q0, arm, cost_fn, n_steps: int = 5,
                              k_guide_frac: float = 0.6, n_grad: int = 20, alpha_guide: float = 1.0,
                              max_halvings: int = 8):
    """guided_ddim_sample (src/diffusion.py:572-628) -> (device traj, log)."""
    torch = _lib.require_cuda()
    L = _lib.lib()
    ks = ddim_steps(schedule.K, n_steps)
    xin = np.array(x_K, dtype=np.float64)
    single = xin.ndim == 2
    x = torch.as_tensor(xin[None] if single else xin, device="cuda").contiguous()
    cd = torch.as_tensor(np.atleast_2d(np.asarray(cond, dtype=np.float64)), device="cuda")
    lo, hi = net.config.lo_hi()
    span = hi - lo
    k_guide = k_guide_frac * schedule.K
    fused = isinstance(cost_fn, PlannerCost)
    ws = {"arm_lo": torch.as_tensor(np.asarray(arm.lo, dtype=np.float64), device="cuda"),
          "arm_span": torch.as_tensor(np.asarray(arm.hi - arm.lo, dtype=np.float64), device="cuda"),
          "net_span": torch.as_tensor(np.asarray(span, dtype=np.float64), device="cuda")}
    log: List[Tuple[int, bool]] = []
    x0 = torch.empty_like(x)
    n = x.numel()
    for i, k in enumerate(ks):
        ab = float(schedule.alpha_bar(int(k)))
        eps = predict_noise_device(net, x, int(k), cd)
        has_next = i + 1 < len(ks)
        ab_next = float(schedule.alpha_bar(int(ks[i + 1]))) if has_next else 1.0
        guided = False
        if has_next:
            guided = bool(k < k_guide and alpha_guide != 0.0)
            log.append((int(k), guided))
        if not guided:
            _lib.check(L.ps_ref_ddim_update(_lib.ptr(x), _lib.ptr(eps), n, ab, ab_next, int(has_next),
                                            X0_CLIP[0], X0_CLIP[1], _lib.ptr(x0), _lib.stream_handle()),
                       "ddim_update")
            continue
        _lib.check(L.ps_ref_ddim_update(_lib.ptr(x), _lib.ptr(eps), n, ab, ab_next, 0, X0_CLIP[0],
                                        X0_CLIP[1], _lib.ptr(x0), _lib.stream_handle()), "ddim_update")
        if fused:
            _guide_device(cost_fn, arm, net, x0, n_grad, alpha_guide, max_halvings, ws)
        else:
            xh = _guide_host(cost_fn, arm, span, x0.cpu().numpy(), n_grad, alpha_guide, max_halvings)
            x0.copy_(torch.as_tensor(np.ascontiguousarray(xh), device="cuda"))
        _lib.check(L.ps_ref_ddim_next(_lib.ptr(x), _lib.ptr(x0), _lib.ptr(eps), n, ab_next,
                                      _lib.stream_handle()), "ddim_next")
    log.append((int(ks[-1]), False))
    B, T, D = x0.shape
    hi_t = torch.as_tensor(np.asarray(arm.hi, dtype=np.float64), device="cuda")
    q = torch.as_tensor(np.asarray(q0, dtype=np.float64), device="cuda")
    traj = torch.empty_like(x0)
    _lib.check(L.ps_ref_denorm_pin(_lib.ptr(x0), B, T, D, _lib.ptr(ws["arm_lo"]), _lib.ptr(hi_t), _lib.ptr(q),
                                   _lib.ptr(traj), _lib.stream_handle()), "denormalize")
    return (traj[0] if single else traj), log


def guided_ddim_sample(net, schedule, cond, x_K, q0, arm, cost_fn, n_steps: int = 5,
                       k_guide_frac: float = 0.6, n_grad: int = 20, alpha_guide: float = 1.0,
                       max_halvings: int = 8):
    """src/diffusion.py:572-628: DDIM with cost-gradient descent on the intermediate x0_hat
    for sub-steps with k < k_guide_frac*K (never the last).  Returns (trajectories, log).
    With a `PlannerCost` the guidance is one fused GPU launch per guided sub-step; any other
    callable is evaluated on host arrays, as the reference does."""
    traj, log = guided_ddim_sample_device(net, schedule, cond, x_K, q0, arm, cost_fn, n_steps,
                                          k_guide_frac, n_grad, alpha_guide, max_halvings)
    return traj.cpu().numpy(), log


# ----------------------------------------------------------------------------- checkpoints
def save_checkpoint(path, net, schedule, meta: Optional[dict] = None):
    """PSCK: magic, u64 header length, sorted-key JSON, little-endian f64 blob (src/diffusion.py:635-651)."""
    names = [n for n, _ in _param_shapes(net.config)]
    hp = _host_params(net)
    header = {"format": 1, "arch": asdict(net.config), "init_seed": net.init_seed,
              "schedule": {"betas": [float(x) for x in np.asarray(schedule.betas).ravel()]},
              "meta": meta or {},
              "params": [{"name": n, "shape": list(hp[n].shape)} for n in names]}
    blob = b"".join(np.ascontiguousarray(hp[n], dtype="<f8").tobytes() for n in names)
    head = json.dumps(header, sort_keys=True).encode()
    with open(path, "wb") as f:
        f.write(CKPT_MAGIC)
        f.write(struct.pack("<Q", len(head)))
        f.write(head)
        f.write(blob)


def load_checkpoint(path):
    """src/diffusion.py:657-687."""
    path = Path(path)
    if not path.exists():
        raise FileNotFoundError(f"checkpoint not found: {path}")
    with open(path, "rb") as f:
        if f.read(4) != CKPT_MAGIC:
            raise ValueError(f"{path} is not a checkpoint file")
        (hlen,) = struct.unpack("<Q", f.read(8))
        header = json.loads(f.read(hlen).decode())
        blob = f.read()
    arch = header["arch"]
    for key in ("scan_channels", "scan_kernels", "scan_strides", "joint_lo", "joint_hi", "bounds_lo",
                "bounds_hi"):
        arch[key] = tuple(arch[key])
    cfg = ArchConfig(**arch)
    params, off = {}, 0
    for spec_ in header["params"]:
        shape = tuple(spec_["shape"])
        n = int(np.prod(shape))
        params[spec_["name"]] = np.frombuffer(blob, dtype="<f8", count=n, offset=off).reshape(shape).copy()
        off += n * 8
    if off != len(blob):
        raise ValueError(f"checkpoint blob size mismatch in {path}")
    net = DenoiserNet(config=cfg, params=params, init_seed=header.get("init_seed", 0))
    return net, NoiseSchedule(betas=np.array(header["schedule"]["betas"])), header.get("meta", {})
