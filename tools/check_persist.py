"""Persistent small-batch sampler (unet_small.cu) vs the layered tcgen05 kernels vs fp32 SIMT:
noise predictions, full DDPM-100 sampling, and per-call timing.
    python tools/check_persist.py"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2410_16727_b200 import spec, synth
from paper_2410_16727_b200.sampler import SeedSampler

params = spec.random_model()
s0 = SeedSampler(params, mode=0)
s1 = SeedSampler(params, mode=1)
rng = np.random.default_rng(0)


def cond_of(P):
    return np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)


def with_mode(m, f):
    os.environ["PS_PERSIST"] = m
    try:
        r = f()
        torch.cuda.synchronize()
        return r
    finally:
        os.environ.pop("PS_PERSIST", None)


for (P, S, T, k) in [(1, 32, 32, 50), (1, 3, 32, 10), (4, 32, 32, 99), (2, 4, 64, 20), (8, 32, 32, 5), (3, 40, 64, 70)]:
    cond = cond_of(P)
    x = rng.standard_normal((P * S, T, 7)).astype(np.float32)
    e0 = s0.predict_noise(x, k, s0.film(cond), S).cpu().numpy()
    ep = with_mode("1", lambda: s1.predict_noise(x, k, s1.film(cond), S).cpu().numpy())
    el = with_mode("0", lambda: s1.predict_noise(x, k, s1.film(cond), S).cpu().numpy())
    ref = np.sqrt((e0 ** 2).mean())
    f = lambda d: f"max {np.abs(d).max():.2e} rel-rms {np.sqrt((d ** 2).mean()) / ref:.2e}"
    print(f"P{P} S{S} T{T} k{k}: persist-vs-fp32 {f(ep - e0)} | layered-vs-fp32 {f(el - e0)} | "
          f"persist-vs-layered {f(ep - el)} finite {np.isfinite(ep).all()}", flush=True)

for (P, S, T) in [(1, 32, 32), (2, 8, 32), (4, 32, 64)]:
    cond = cond_of(P)
    q0 = synth.make_problems(P, seed=3).q_start
    fa = s1.film(cond)
    tp = with_mode("1", lambda: s1.sample(fa, q0, S, T=T).cpu().numpy())
    tl = with_mode("0", lambda: s1.sample(fa, q0, S, T=T).cpu().numpy())
    t0 = s0.sample(s0.film(cond), q0, S, T=T).cpu().numpy()
    d, dl = tp - t0, tl - t0
    print(f"sample P{P} S{S} T{T}: persist-vs-fp32 max {np.abs(d).max():.3e} rms {np.sqrt((d ** 2).mean()):.3e} | "
          f"layered-vs-fp32 max {np.abs(dl).max():.3e} rms {np.sqrt((dl ** 2).mean()):.3e} | "
          f"row0 pinned {np.array_equal(tp[:, 0], np.repeat(q0, S, axis=0))}", flush=True)

# timing: one planning call's sampler (100 DDPM steps) per batch size
for (P, S) in [(1, 8), (1, 32), (1, 128), (16, 8), (4, 32), (8, 32), (16, 32), (64, 32)]:
    cond = cond_of(P)
    q0 = synth.make_problems(P, seed=3).q_start
    fa = s1.film(cond)
    res = {}
    for m in ("1", "0"):
        os.environ["PS_PERSIST"] = m
        for _ in range(3):
            s1.sample(fa, q0, S)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0_.record()
            s1.sample(fa, q0, S)
            e1_.record()
            torch.cuda.synchronize()
            ts.append(e0_.elapsed_time(e1_))
        res[m] = float(np.median(ts))
    os.environ.pop("PS_PERSIST", None)
    print(f"time P{P} S{S} (B={P * S}): persistent {res['1']:.2f} ms | layered {res['0']:.2f} ms | "
          f"x{res['0'] / res['1']:.2f}", flush=True)
