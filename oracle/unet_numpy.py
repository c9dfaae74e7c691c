"""ORACLE (test infrastructure only): numpy restatement of the BASELINE-profile seed
sampler -- depth-image encoder, 1-D temporal U-Net noise predictor with GroupNorm /
Mish / FiLM, squared-cosine DDPM and the Philox + Box-Muller noise stream.

Architecture and every pinned choice: paper_2410_16727_b200/spec.py (UNetArch).
Reference anchors generalised here:
  condition encoder -> cond vector          planseed/diffusion.py:246-269
  1-based k, sinusoid with (half-1)         planseed/diffusion.py:32-51, :228-234
  FiLM h*(1+scale)+shift                    planseed/diffusion.py:272-285
  x0 clip [-0.1, 1.1], returns last x0_hat  planseed/diffusion.py:529-556
  denormalise, row 0 := q0                  planseed/diffusion.py:559-569, arm.py:195-201

Layout is channels-last (B, T, C) throughout, as on the device.  Computations run in
float64 unless `dtype=np.float32` is requested (the CPU baseline uses float32).
"""

from __future__ import annotations

import math

import numpy as np

from paper_2410_16727_b200 import spec


# ----------------------------------------------------------------------------
# elementwise
# ----------------------------------------------------------------------------

def softplus(x):
    return np.where(x > 20.0, x, np.log1p(np.exp(np.minimum(x, 20.0))))


def mish(x):
    return x * np.tanh(softplus(x))


# ----------------------------------------------------------------------------
# convolutions, channels-last
# ----------------------------------------------------------------------------

def conv1d(x, w, b, stride=1, pad=None):
    """x (B,T,C), w (O,C,K) -> (B,T',O); zero padding (K-1)//2 by default."""
    B, T, C = x.shape
    O, C2, K = w.shape
    assert C == C2
    pad = (K - 1) // 2 if pad is None else pad
    xp = np.zeros((B, T + 2 * pad, C), dtype=x.dtype)
    xp[:, pad:pad + T] = x
    T_out = (T + 2 * pad - K) // stride + 1
    cols = np.stack([xp[:, k:k + stride * (T_out - 1) + 1:stride] for k in range(K)], axis=2)
    # cols (B, T_out, K, C) @ w (K, C, O)
    wk = np.transpose(w, (2, 1, 0)).reshape(K * C, O).astype(x.dtype)
    y = cols.reshape(B * T_out, K * C) @ wk
    return y.reshape(B, T_out, O) + b.astype(x.dtype)


def conv_transpose1d(x, w, b):
    """ConvTranspose1d(k=4, s=2, p=1): x (B,T,C), w (C,O,4) -> (B,2T,O).
    out[t] = sum_{s,k: t = 2s - 1 + k} x[s] w[:, :, k]."""
    B, T, C = x.shape
    _, O, K = w.shape
    out = np.zeros((B, 2 * T + 2, O), dtype=x.dtype)  # index t+1
    xf = x.reshape(B * T, C)
    for k in range(K):
        y = (xf @ w[:, :, k].astype(x.dtype)).reshape(B, T, O)
        # t = 2s - 1 + k  ->  stored at t+1 = 2s + k
        out[:, k:k + 2 * T:2] += y
    return out[:, 1:2 * T + 1] + b.astype(x.dtype)


def group_norm(x, gamma, beta, groups=spec.GN_GROUPS, eps=spec.GN_EPS):
    B, T, C = x.shape
    xg = x.reshape(B, T, groups, C // groups)
    mean = xg.mean(axis=(1, 3), keepdims=True)
    var = ((xg - mean) ** 2).mean(axis=(1, 3), keepdims=True)
    y = (xg - mean) / np.sqrt(var + eps)
    return y.reshape(B, T, C) * gamma.astype(x.dtype) + beta.astype(x.dtype)


def conv2d_s2(x, w, b):
    """x (C,H,W), w (O,C,3,3), stride 2, pad 1 -> (O, ceil(H/2), ceil(W/2))."""
    C, H, W = x.shape
    O = w.shape[0]
    Ho, Wo = (H - 1) // 2 + 1, (W - 1) // 2 + 1
    xp = np.zeros((C, H + 2, W + 2), dtype=x.dtype)
    xp[:, 1:H + 1, 1:W + 1] = x
    cols = np.empty((C, 3, 3, Ho, Wo), dtype=x.dtype)
    for dy in range(3):
        for dx in range(3):
            cols[:, dy, dx] = xp[:, dy:dy + 2 * Ho - 1:2, dx:dx + 2 * Wo - 1:2]
    y = w.reshape(O, C * 9).astype(x.dtype) @ cols.reshape(C * 9, Ho * Wo)
    return y.reshape(O, Ho, Wo) + b.astype(x.dtype)[:, None, None]


# ----------------------------------------------------------------------------
# encoder and condition
# ----------------------------------------------------------------------------

def encode_image(enc_params, enc: spec.EncoderArch, img, dtype=np.float64):
    """depth (H,W) metres -> 256-d embedding (conv3x3 s2 + ReLU stack, global mean)."""
    h = (np.asarray(img, dtype=dtype) / spec.DEPTH_SCALE)[None]
    for i in range(len(enc.channels)):
        h = np.maximum(conv2d_s2(h, enc_params[f"enc{i}_w"], enc_params[f"enc{i}_b"]), 0.0)
    return h.mean(axis=(1, 2))


def make_cond(img_emb, q_start, goal, robot_lo=None, robot_hi=None):
    lo = -spec.JOINT_LIMIT if robot_lo is None else robot_lo
    hi = spec.JOINT_LIMIT if robot_hi is None else robot_hi
    qn = (np.asarray(q_start, dtype=np.float64) - lo) / (hi - lo)
    g = np.asarray(goal, dtype=np.float64)
    return np.concatenate([img_emb, qn, g[:3] / spec.GOAL_EXTENT, g[3:7]])


def encode_problems(enc_params, enc, images, q_start, goal, dtype=np.float64):
    """images (P, n_img, H, W) -> cond (P, 270); multiple images are averaged."""
    P = images.shape[0]
    out = np.empty((P, spec.COND_DIM))
    for p in range(P):
        embs = [encode_image(enc_params, enc, images[p, m], dtype) for m in range(images.shape[1])]
        out[p] = make_cond(np.mean(embs, axis=0), q_start[p], goal[p])
    return out


# ----------------------------------------------------------------------------
# U-Net
# ----------------------------------------------------------------------------

def time_embedding(params, k):
    s = spec.timestep_sinusoid(k)
    h = mish(s @ params["t_fc1_w"] + params["t_fc1_b"])
    return h @ params["t_fc2_w"] + params["t_fc2_b"]


def film_vectors(params, arch: spec.UNetArch, cond, k):
    """cond (P,270), scalar k -> {block: (scale (P,C), shift (P,C))}.
    e = mish([t_emb(k) ; cond]); (scale, shift) = e @ W + b."""
    temb = time_embedding(params, k)                  # (1,128)
    P = cond.shape[0]
    e = mish(np.concatenate([np.repeat(temb, P, axis=0), cond], axis=1))
    out = {}
    for blk in arch.blocks():
        f = e @ params[f"{blk.name}_film_w"] + params[f"{blk.name}_film_b"]
        out[blk.name] = (f[:, :blk.c_out], f[:, blk.c_out:])
    return out


def _expand(v, S, T):
    """(P,C) per-problem vector -> broadcastable (P*S, 1, C)."""
    return np.repeat(v, S, axis=0)[:, None, :]


def res_block(params, name, x, film, S, dtype):
    p = lambda s: params[f"{name}_{s}"]
    T = x.shape[1]
    h = mish(group_norm(conv1d(x, p("c0_w"), p("c0_b")), p("gn0_g"), p("gn0_b")))
    sc, sh = film[name]
    h = h * (1.0 + _expand(sc, S, T).astype(dtype)) + _expand(sh, S, T).astype(dtype)
    h = mish(group_norm(conv1d(h, p("c1_w"), p("c1_b")), p("gn1_g"), p("gn1_b")))
    res = conv1d(x, p("res_w"), p("res_b")) if f"{name}_res_w" in params else x
    return h + res


def unet_forward(params, arch: spec.UNetArch, x, k, cond, S, dtype=np.float64):
    """x (B,T,7) normalised trajectories, scalar step k (1-based), cond (P,270), B=P*S."""
    x = np.asarray(x, dtype=dtype)
    film = film_vectors(params, arch, np.asarray(cond, dtype=np.float64), k)
    P = lambda n: params[n]
    h = res_block(params, "d0r0", x, film, S, dtype)
    h = res_block(params, "d0r1", h, film, S, dtype)
    h = conv1d(h, P("down0_w"), P("down0_b"), stride=2, pad=1)
    h = res_block(params, "d1r0", h, film, S, dtype)
    h = res_block(params, "d1r1", h, film, S, dtype)
    skip1 = h
    h = conv1d(h, P("down1_w"), P("down1_b"), stride=2, pad=1)
    h = res_block(params, "d2r0", h, film, S, dtype)
    h = res_block(params, "d2r1", h, film, S, dtype)
    skip2 = h
    h = res_block(params, "m0", h, film, S, dtype)
    h = res_block(params, "m1", h, film, S, dtype)
    h = res_block(params, "u0r0", np.concatenate([h, skip2], axis=2), film, S, dtype)
    h = res_block(params, "u0r1", h, film, S, dtype)
    h = conv_transpose1d(h, P("up0_w"), P("up0_b"))
    h = res_block(params, "u1r0", np.concatenate([h, skip1], axis=2), film, S, dtype)
    h = res_block(params, "u1r1", h, film, S, dtype)
    h = conv_transpose1d(h, P("up1_w"), P("up1_b"))
    h = mish(group_norm(conv1d(h, P("fin_c_w"), P("fin_c_b")), P("fin_gn_g"), P("fin_gn_b")))
    return conv1d(h, P("out_w"), P("out_b"))


# ----------------------------------------------------------------------------
# noise stream: Philox4x32-10 + Box-Muller (spec.py, "Counter-based noise")
# ----------------------------------------------------------------------------

_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)


def philox4x32(c0, c1, c2, c3, k0, k1):
    c = [np.asarray(v, dtype=np.uint64) & _MASK for v in (c0, c1, c2, c3)]
    k0 = np.uint64(k0) & _MASK
    k1 = np.uint64(k1) & _MASK
    c0, c1, c2, c3 = np.broadcast_arrays(*c)
    c0, c1, c2, c3 = (a.copy() for a in (c0, c1, c2, c3))
    for _ in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & _MASK, lo1, (hi0 ^ c3 ^ k1) & _MASK, lo0
        k0 = (k0 + _W0) & _MASK
        k1 = (k1 + _W1) & _MASK
    return [a.astype(np.uint32) for a in (c0, c1, c2, c3)]


def noise(step: int, problems: np.ndarray, seeds: np.ndarray, T: int, D: int = spec.DOF,
          noise_seed: int = spec.NOISE_SEED) -> np.ndarray:
    """Standard normals (len(problems), T, D) float32 for global (problem, seed) pairs."""
    n = T * D
    nb = (n + 3) // 4
    blk = np.arange(nb, dtype=np.uint64)[None, :]
    pr = np.asarray(problems, dtype=np.uint64)[:, None]
    sd = np.asarray(seeds, dtype=np.uint64)[:, None]
    r0, r1, r2, r3 = philox4x32(blk, np.uint64(step), pr, sd, noise_seed, spec.PHILOX_KEY_HI)
    two24 = np.float32(1.0 / 16777216.0)
    out = np.empty((len(problems), nb, 4), dtype=np.float32)
    for (a, b), (i, j) in (((r0, r1), (0, 1)), ((r2, r3), (2, 3))):
        u1 = ((a >> np.uint32(8)).astype(np.float32) + np.float32(1.0)) * two24
        u2 = (b >> np.uint32(8)).astype(np.float32) * two24
        rad = np.sqrt(np.float32(-2.0) * np.log(u1))
        ang = np.float32(2.0 * math.pi) * u2
        out[:, :, i] = rad * np.cos(ang)
        out[:, :, j] = rad * np.sin(ang)
    return out.reshape(len(problems), nb * 4)[:, :n].reshape(len(problems), T, D)


# ----------------------------------------------------------------------------
# samplers
# ----------------------------------------------------------------------------

def sample(params, arch, cond, q_start, S, p0=0, T=spec.T_DEFAULT, betas=None, steps=None,
           dtype=np.float64, x_init=None, return_eps=False, problems=None, table_dtype=np.float32,
           guide_fn=None):
    """Seed generation for P problems x S seeds.

    steps=None: full K-step stochastic DDPM (posterior mean + sigma z).
    steps=[...]: deterministic DDIM (eta=0) over the given 1-based indices, as
    planseed's _ddim_core (diffusion.py:535-556).
    problems: explicit global problem indices of the rows of cond (default p0 .. p0+P-1), so a
    subset of a large batch can be checked (problems are independent: per-sample GroupNorm,
    per-problem FiLM, noise keyed by the global index).
    table_dtype: float32 = the device's coefficient tables; float64 = exact (planseed bridge).
    guide_fn(i, k, x0_hat) -> x0_hat: guided_ddim_sample's hook (diffusion.py:540-552), DDIM only,
    never on the last step.
    Returns physical trajectories (P*S, T, 7) with row 0 := q_start."""
    betas = spec.cosine_betas() if betas is None else betas
    K = betas.shape[0]
    tab = spec.sampler_tables(betas, dtype=table_dtype)
    P = cond.shape[0]
    gp = np.arange(p0, p0 + P) if problems is None else np.asarray(problems)
    assert gp.shape == (P,)
    prob = np.repeat(gp, S)
    sidx = np.tile(np.arange(S), P)
    x = noise(0, prob, sidx, T) if x_init is None else np.asarray(x_init)
    x = x.astype(dtype)
    lo, hi = -spec.JOINT_LIMIT, spec.JOINT_LIMIT
    ks = list(range(K, 0, -1)) if steps is None else [int(k) for k in steps]
    x0 = x
    for i, k in enumerate(ks):
        eps = unet_forward(params, arch, x, k, cond, S, dtype)
        x0 = np.clip((x - tab.sq1m[k] * eps) * tab.rsq[k], spec.X0_CLIP[0], spec.X0_CLIP[1])
        if steps is None:
            if k > 1:
                z = noise(k, prob, sidx, T).astype(dtype)
                x = tab.c0[k] * x0 + tab.c1[k] * x + tab.sig[k] * z
        elif i + 1 < len(ks):
            if guide_fn is not None:
                x0 = guide_fn(i, k, x0)
            kn = ks[i + 1]
            x = tab.sq[kn] * x0 + tab.sq1m[kn] * eps
    traj = lo + x0 * (hi - lo)
    traj[:, 0, :] = np.repeat(np.asarray(q_start, dtype=np.float64), S, axis=0)
    return traj
