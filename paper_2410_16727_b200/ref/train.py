"""Training of planseed's denoiser on the GPU (src/diffusion.py:357-508): `loss_eq2` (one record's
loss and parameter gradients) and `train` (Adam over iid minibatches), same signatures, same host
random draws and the same float64 arithmetic as the reference, with the forward pass, the backward
pass through every layer and the Adam update as float64 CUDA kernels (csrc/ref_train.cu).

The layers are the reference graph's (condition_graph + predict_noise_graph, :240-285): a strided
conv1d scan encoder with SiLU, three small MLPs, the 3-layer FiLM trunk; the loss is
fk_weighted_mse(noise) + mse_stabilizer * plain_weighted_mse (:304-349).  Host-side input
preparation (feature vectors, forward noising of the normalised expert, timestep features) follows
the reference line for line, as the sampler drop-in does."""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import numpy as np

from .. import _lib
from .diffusion import ArchConfig, _param_shapes, make_schedule, pose_features, problem_features
from .types import fk_pose, normalize


@dataclass
class TrainConfig:
    """src/diffusion.py:357-379."""

    batch_size: int = 256
    lr: float = 3e-4
    lr_final: Optional[float] = None
    epochs: int = 400
    alpha_loss: float = 4.0
    seed: int = 0
    fk_points_per_link: Optional[int] = None
    augment_reversal: bool = True
    fk_loss_target: str = "noise"
    mse_stabilizer: float = 1.0

    def __post_init__(self):
        if self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.alpha_loss < 0:
            raise ValueError("alpha_loss must be >= 0")
        if self.fk_loss_target not in ("noise", "x0_reconstruction"):
            raise ValueError(f"unknown fk_loss_target {self.fk_loss_target!r}")


@dataclass
class _Sample:
    traj_fwd: np.ndarray
    prob_fwd: np.ndarray
    prob_rev: np.ndarray
    scans: np.ndarray
    poses: np.ndarray
    weight: float


def prepare_samples(cfg: ArchConfig, arm, records: Sequence, alpha_loss: float) -> List[_Sample]:
    """src/diffusion.py:395-412."""
    out = []
    for rec in records:
        traj = np.asarray(rec.expert, dtype=np.float64)
        q0 = rec.problem.q_start
        goal = rec.problem.goal
        start_pose = fk_pose(arm, q0)
        out.append(_Sample(
            traj_fwd=normalize(arm, traj),
            prob_fwd=problem_features(cfg, q0, goal),
            prob_rev=problem_features(cfg, traj[-1], start_pose),
            scans=np.stack([np.asarray(s.depths, dtype=np.float64) / cfg.max_range for s in rec.scans]),
            poses=np.stack([pose_features(cfg, s.pose) for s in rec.scans]),
            weight=1.0 + alpha_loss * float(rec.graph_used),
        ))
    return out


def _timestep_features(cfg: ArchConfig, k: np.ndarray) -> np.ndarray:
    """src/diffusion.py:228-234 for a vector of steps."""
    k = np.atleast_1d(np.asarray(k, dtype=np.float64))
    half = cfg.t_embed // 2
    freqs = np.exp(-np.log(10000.0) * np.arange(half) / max(half - 1, 1))
    ang = k[:, None] * freqs[None, :]
    return np.concatenate([np.sin(ang), np.cos(ang)], axis=1)


class _Trainer:
    """Device float64 parameters, gradients and Adam moments of one DenoiserNet."""

    def __init__(self, net, arm):
        self.torch = _lib.require_cuda()
        self.L = _lib.lib()
        self.net, self.cfg, self.arm = net, net.config, arm
        t = self.torch
        host = {k: np.asarray(getattr(v, "data", v), dtype=np.float64) for k, v in net.params.items()}
        self.names = [n for n, _ in _param_shapes(self.cfg)]
        self.p = {n: t.as_tensor(np.ascontiguousarray(host[n]), device="cuda") for n in self.names}
        self.g = {n: t.zeros_like(self.p[n]) for n in self.names}
        self.m = {n: t.zeros_like(self.p[n]) for n in self.names}
        self.v = {n: t.zeros_like(self.p[n]) for n in self.names}
        self.t = 0
        lo, hi = self.cfg.lo_hi()
        self.lo = t.as_tensor(lo, device="cuda")
        self.span = t.as_tensor(hi - lo, device="cuda")
        self.len = t.as_tensor(np.asarray(arm.lengths, dtype=np.float64), device="cuda")

    # -- layer helpers -------------------------------------------------------------------------
    def _s(self):
        return _lib.stream_handle()

    def _gemm(self, A, lda, ta, B, ldb, tb, C, ldc, M, N, K, acc=0):
        _lib.check(self.L.ps_train_gemm(A, lda, ta, B, ldb, tb, C, ldc, M, N, K, acc, self._s()), "train_gemm")

    def _linear(self, x, ldx, R, W, b, out, ldo, act, pre=None):
        K, N = W.shape
        self._gemm(x, ldx, 0, _lib.ptr(W), N, 0, out, ldo, R, N, K)
        _lib.check(self.L.ps_train_bias_act(out, ldo, _lib.ptr(b), R, N, act, _lib.ptr(pre) if pre is not None else None,
                                            self._s()), "bias_act")

    def _linear_bwd(self, gy, ldg, x, ldx, R, name, gx=None, ldgx=0, acc_gx=0):
        """dW = x^T gy, db = colsum gy, gx (+)= gy W^T."""
        W = self.p[f"{name}_w"]
        K, N = W.shape
        self._gemm(x, ldx, 1, gy, ldg, 0, _lib.ptr(self.g[f"{name}_w"]), N, K, N, R)
        _lib.check(self.L.ps_train_colsum(gy, ldg, R, N, _lib.ptr(self.g[f"{name}_b"]), 0, self._s()), "colsum")
        if gx is not None:
            self._gemm(gy, ldg, 0, _lib.ptr(W), N, 1, gx, ldgx, R, K, N, acc_gx)

    # -- one minibatch ---------------------------------------------------------------------------
    def loss_and_grads(self, schedule, tcfg: TrainConfig, trajs, probs, scans, poses, weights, ks, eps) -> float:
        """_batch_loss (src/diffusion.py:415-432) forward + backward; gradients into self.g."""
        if tcfg.fk_loss_target != "noise":
            raise NotImplementedError("fk_loss_target='x0_reconstruction' is not built on the GPU path")
        t, cfg, p = self.torch, self.cfg, self.p
        dev = lambda a: t.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")
        B = trajs.shape[0]
        ab = schedule.alpha_bar(np.asarray(ks)).reshape(-1, 1, 1)
        x_k = np.sqrt(ab) * trajs + np.sqrt(1.0 - ab) * eps                  # forward_noise (:66-77)
        D_x, C = cfg.x_dim, cfg.cond_dim
        E = lambda *s: t.empty(s, dtype=t.float64, device="cuda")
        P = _lib.ptr
        # ---- condition_graph: scan conv stack
        h = dev(scans.reshape(B, 1, cfg.n_rays))
        conv_io = []
        c_in, L_in = 1, cfg.n_rays
        for i, (co, kk, ss) in enumerate(zip(cfg.scan_channels, cfg.scan_kernels, cfg.scan_strides)):
            lo_ = (L_in - kk) // ss + 1
            pre, y = E(B, co, lo_), E(B, co, lo_)
            _lib.check(self.L.ps_train_conv1d(P(h), B, c_in, L_in, P(p[f"scan_conv{i}_w"]), P(p[f"scan_conv{i}_b"]),
                                              co, kk, ss, P(pre), P(y), self._s()), "conv1d")
            conv_io.append((h, c_in, L_in, co, kk, ss, pre))
            h, c_in, L_in = y, co, lo_
        flat = h.reshape(B, -1)
        nflat = flat.shape[1]
        ct = E(B, C + cfg.t_embed)                                      # [scan | prob | pose | t_emb]
        ldc = C + cfg.t_embed
        self._linear(P(flat), nflat, B, p["scan_fc_w"], p["scan_fc_b"], P(ct), ldc, 0)
        mlp_io = {}
        off = cfg.scan_embed
        for name, feats, width in (("prob", probs, cfg.problem_embed), ("pose", poses, cfg.pose_embed),
                                   ("t", _timestep_features(cfg, ks), cfg.t_embed)):
            xin = dev(feats)
            hid, pre = E(B, cfg.embed_hidden), E(B, cfg.embed_hidden)
            self._linear(P(xin), xin.shape[1], B, p[f"{name}_fc1_w"], p[f"{name}_fc1_b"], P(hid), cfg.embed_hidden, 1, pre)
            out_off = C if name == "t" else off
            self._linear(P(hid), cfg.embed_hidden, B, p[f"{name}_fc2_w"], p[f"{name}_fc2_b"], P(ct) + 8 * out_off, ldc, 0)
            mlp_io[name] = (xin, hid, pre, out_off, width)
            if name != "t":
                off += width
        # ---- predict_noise_graph: trunk with FiLM
        hin = t.cat([dev(x_k.reshape(B, D_x)), ct], dim=1).contiguous()   # [x | cond | t_emb]
        mod = ct                                                          # [cond | t_emb]
        trunk = []
        h_prev, w_prev = hin, hin.shape[1]
        H = cfg.hidden
        for i in range(cfg.n_hidden):
            a, pre, sc, sh, hn = E(B, H), E(B, H), E(B, H), E(B, H), E(B, H)
            self._linear(P(h_prev), w_prev, B, p[f"trunk{i}_w"], p[f"trunk{i}_b"], P(a), H, 1, pre)
            self._linear(P(mod), ldc, B, p[f"trunk{i}_scale_w"], p[f"trunk{i}_scale_b"], P(sc), H, 0)
            self._linear(P(mod), ldc, B, p[f"trunk{i}_shift_w"], p[f"trunk{i}_shift_b"], P(sh), H, 0)
            _lib.check(self.L.ps_train_film(P(a), P(sc), P(sh), B * H, P(hn), self._s()), "film")
            trunk.append((h_prev, w_prev, a, pre, sc))
            h_prev, w_prev = hn, H
        eps_hat = E(B, D_x)
        self._linear(P(h_prev), H, B, p["trunk_out_w"], p["trunk_out_b"], P(eps_hat), D_x, 0)
        # ---- loss: fk_weighted_mse(noise) + mse_stabilizer * plain_weighted_mse
        m = tcfg.fk_points_per_link or self.arm.points_per_link
        fr = dev((np.arange(m) + 0.5) / m)
        w = dev(weights)
        row_fk, row_mse, g_out = E(B * cfg.t_len), E(B * cfg.t_len), E(B, D_x)
        eps_d = dev(eps.reshape(B, D_x))
        base = np.asarray(self.arm.base, dtype=np.float64)
        _lib.check(self.L.ps_train_fk_loss(P(eps_d), P(eps_hat), B, cfg.t_len, cfg.dof, m, P(w), P(self.lo),
                                           P(self.span), P(self.len), P(fr), float(base[0]), float(base[1]),
                                           float(tcfg.mse_stabilizer), P(row_fk), P(row_mse), P(g_out), self._s()),
                   "fk_loss")
        # ---- backward
        g_h = E(B, H)
        self._linear_bwd(P(g_out), D_x, P(h_prev), H, B, "trunk_out", P(g_h), H)
        g_mod = t.zeros((B, ldc), dtype=t.float64, device="cuda")
        g_hin = E(B, hin.shape[1])
        for i in reversed(range(cfg.n_hidden)):
            h_in, w_in, a, pre, sc = trunk[i]
            g_a, g_sc = E(B, H), E(B, H)
            _lib.check(self.L.ps_train_film_bwd(P(g_h), P(a), P(sc), B * H, P(g_a), P(g_sc), self._s()), "film_bwd")
            self._linear_bwd(P(g_sc), H, P(mod), ldc, B, f"trunk{i}_scale", P(g_mod), ldc, 1)
            self._linear_bwd(P(g_h), H, P(mod), ldc, B, f"trunk{i}_shift", P(g_mod), ldc, 1)   # g_sh = g_h
            _lib.check(self.L.ps_train_silu_bwd(P(g_a), H, P(pre), B, H, self._s()), "silu_bwd")
            if i > 0:
                g_h = E(B, H)
                self._linear_bwd(P(g_a), H, P(h_in), w_in, B, f"trunk{i}", P(g_h), H)
            else:
                self._linear_bwd(P(g_a), H, P(h_in), w_in, B, f"trunk{i}", P(g_hin), hin.shape[1])
        g_ct = g_mod + g_hin[:, D_x:]                                     # concat backward (plumbing)
        for name in ("t", "pose", "prob"):
            xin, hid, pre, out_off, width = mlp_io[name]
            g_o = g_ct[:, out_off:out_off + width].contiguous()
            g_hid = E(B, cfg.embed_hidden)
            self._linear_bwd(P(g_o), width, P(hid), cfg.embed_hidden, B, f"{name}_fc2", P(g_hid), cfg.embed_hidden)
            _lib.check(self.L.ps_train_silu_bwd(P(g_hid), cfg.embed_hidden, P(pre), B, cfg.embed_hidden, self._s()),
                       "silu_bwd")
            self._linear_bwd(P(g_hid), cfg.embed_hidden, P(xin), xin.shape[1], B, f"{name}_fc1")
        g_scan = g_ct[:, :cfg.scan_embed].contiguous()
        g_flat = E(B, nflat)
        self._linear_bwd(P(g_scan), cfg.scan_embed, P(flat), nflat, B, "scan_fc", P(g_flat), nflat)
        g_y = g_flat
        for i in reversed(range(len(conv_io))):
            x_in, c_in, L_in, co, kk, ss, pre = conv_io[i]
            lo_ = (L_in - kk) // ss + 1
            _lib.check(self.L.ps_train_silu_bwd(P(g_y), co * lo_, P(pre), B, co * lo_, self._s()), "silu_bwd")
            g_x = E(B, c_in, L_in) if i > 0 else None
            _lib.check(self.L.ps_train_conv1d_bwd(P(g_y), P(x_in), P(p[f"scan_conv{i}_w"]), B, c_in, L_in, co, kk, ss,
                                                  P(self.g[f"scan_conv{i}_w"]), P(self.g[f"scan_conv{i}_b"]),
                                                  P(g_x) if g_x is not None else None, self._s()), "conv1d_bwd")
            g_y = g_x
        n_pts = cfg.t_len * cfg.dof * m
        fk = row_fk.view(B, cfg.t_len).sum(1).cpu().numpy() / n_pts
        ms = row_mse.view(B, cfg.t_len).sum(1).cpu().numpy() / (cfg.t_len * cfg.dof)
        wts = np.asarray(weights, dtype=np.float64)
        loss = float(np.mean(fk * wts))
        if tcfg.mse_stabilizer > 0.0:
            loss = loss + float(np.mean(ms * wts)) * tcfg.mse_stabilizer
        return loss

    def adam_step(self, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        """Adam.step (src/autodiff.py:272-284)."""
        self.t += 1
        b1t = 1.0 - beta1 ** self.t
        b2t = 1.0 - beta2 ** self.t
        for n in self.names:
            _lib.check(self.L.ps_train_adam(_lib.ptr(self.p[n]), _lib.ptr(self.g[n]), _lib.ptr(self.m[n]),
                                            _lib.ptr(self.v[n]), self.p[n].numel(), lr, beta1, beta2, b1t, b2t, eps,
                                            self._s()), "adam")

    def write_back(self):
        """Copy the trained weights into net.params (and drop the sampler's device cache)."""
        for n in self.names:
            arr = self.p[n].cpu().numpy()
            cur = self.net.params[n]
            if hasattr(cur, "data") and not isinstance(cur, np.ndarray):
                cur.data = arr
            else:
                self.net.params[n] = arr
        if hasattr(self.net, "_ps_dev"):
            try:
                object.__delattr__(self.net, "_ps_dev")
            except Exception:
                pass


def loss_eq2(arm, net, record, k: int, eps: np.ndarray, alpha_loss: float = 4.0, schedule=None,
             scan_index: int = 0):
    """src/diffusion.py:435-458: single-record training loss and its parameter gradients."""
    if len(record.scans) < 1:
        raise ValueError("record carries no depth scan")
    schedule = schedule or make_schedule()
    cfg = TrainConfig(batch_size=1, alpha_loss=alpha_loss)
    sample = prepare_samples(net.config, arm, [record], alpha_loss)[0]
    tr = _Trainer(net, arm)
    loss = tr.loss_and_grads(schedule, cfg, sample.traj_fwd[None], sample.prob_fwd[None],
                             sample.scans[scan_index][None], sample.poses[scan_index][None],
                             np.array([sample.weight]), np.array([k]), np.asarray(eps, dtype=np.float64)[None])
    return loss, {n: tr.g[n].cpu().numpy() for n in tr.names}


def train(net, records: Sequence, schedule, arm, cfg: TrainConfig, log_every: int = 0,
          callback: Optional[Callable[[int, float], None]] = None) -> List[float]:
    """src/diffusion.py:461-508: Adam over iid minibatches with the reference's host draws;
    the trained weights are written back into net.params."""
    if len(records) == 0:
        raise ValueError("training needs a nonempty dataset")
    samples = prepare_samples(net.config, arm, records, cfg.alpha_loss)
    rng = np.random.default_rng(cfg.seed)
    tr = _Trainer(net, arm)
    t_len, dof = net.config.t_len, net.config.dof
    steps_per_epoch = max(1, len(samples) // cfg.batch_size)
    curve = []
    step = 0
    lr = cfg.lr
    for epoch in range(cfg.epochs):
        if cfg.lr_final is not None and cfg.epochs > 1:
            lr = cfg.lr * (cfg.lr_final / cfg.lr) ** (epoch / (cfg.epochs - 1))
        epoch_losses = []
        for _ in range(steps_per_epoch):
            idx = rng.integers(0, len(samples), size=cfg.batch_size)
            trajs = np.empty((cfg.batch_size, t_len, dof))
            probs = np.empty((cfg.batch_size, dof + 4))
            scans = np.empty((cfg.batch_size, net.config.n_rays))
            poses = np.empty((cfg.batch_size, 4))
            weights = np.empty(cfg.batch_size)
            for i, j in enumerate(idx):
                s = samples[j]
                si = rng.integers(0, s.scans.shape[0])
                reverse = cfg.augment_reversal and rng.random() < 0.5
                trajs[i] = s.traj_fwd[::-1] if reverse else s.traj_fwd
                probs[i] = s.prob_rev if reverse else s.prob_fwd
                scans[i] = s.scans[si]
                poses[i] = s.poses[si]
                weights[i] = s.weight
            ks = rng.integers(1, schedule.K + 1, size=cfg.batch_size)
            eps = rng.standard_normal((cfg.batch_size, t_len, dof))
            loss = tr.loss_and_grads(schedule, cfg, trajs, probs, scans, poses, weights, ks, eps)
            tr.adam_step(lr)
            epoch_losses.append(loss)
            step += 1
            if log_every and step % log_every == 0:
                print(f"step {step}: loss {epoch_losses[-1]:.6f}")
        curve.append(float(np.mean(epoch_losses)))
        if callback is not None:
            callback(epoch, curve[-1])
    tr.write_back()
    return curve
