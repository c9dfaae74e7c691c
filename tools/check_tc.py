"""Debug/validation: bf16 tcgen05 U-Net (mode 1) vs fp32 SIMT (mode 0) vs numpy oracle."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import unet_numpy as un
from paper_2410_16727_b200 import spec
from paper_2410_16727_b200.sampler import SeedSampler

arch = spec.UNetArch()
params = spec.random_model()
s0 = SeedSampler(params, mode=0)
s1 = SeedSampler(params, mode=1)
rng = np.random.default_rng(0)
for (P, S, T, k) in [(1, 16, 32, 50), (2, 8, 32, 100), (4, 32, 32, 3), (2, 4, 64, 20)]:
    cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
    x = rng.standard_normal((P * S, T, 7)).astype(np.float32)
    e0 = s0.predict_noise(x, k, s0.film(cond), S).cpu().numpy()
    e1 = s1.predict_noise(x, k, s1.film(cond), S)
    torch.cuda.synchronize()
    e1 = e1.cpu().numpy()
    want = un.unet_forward(params, arch, x, k, cond, S)
    d1 = e1 - want
    print(f"P{P} S{S} T{T} k{k}: fp32 max {np.abs(e0-want).max():.2e} | bf16 max {np.abs(d1).max():.3e} "
          f"rms {np.sqrt((d1**2).mean()):.3e} ref rms {np.sqrt((want**2).mean()):.3e}", flush=True)

# multi-tile-per-CTA persistence check: bf16 vs fp32 SIMT at B=4096 (>148 tiles per layer)
for P, S in [(128, 32), (1024, 32)]:
    cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
    x = rng.standard_normal((P * S, 32, 7)).astype(np.float32)
    e0 = s0.predict_noise(x, 40, s0.film(cond), S).cpu().numpy()
    e1 = s1.predict_noise(x, 40, s1.film(cond), S).cpu().numpy()
    d = e1 - e0
    print(f"P{P}: bf16 vs fp32 max {np.abs(d).max():.3e} rms {np.sqrt((d**2).mean()):.3e}", flush=True)

# tcgen05 encoder vs fp32 SIMT encoder vs oracle
from paper_2410_16727_b200 import synth
for enc, maker in ((spec.ENCODER_CFG0, synth.config0_problems), (spec.ENCODER_CFG3, synth.config3_problems)):
    pe = spec.random_model(enc)
    a0, a1 = SeedSampler(pe, enc, mode=0), SeedSampler(pe, enc, mode=1)
    pb = maker(3, seed=1)
    c0 = a0.encode(pb.images, pb.q_start, pb.goal).cpu().numpy()
    c1 = a1.encode(pb.images, pb.q_start, pb.goal).cpu().numpy()
    want = un.encode_problems(pe, enc, pb.images, pb.q_start, pb.goal)
    print(f"encoder {len(enc.channels)}L: fp32 max {np.abs(c0-want).max():.2e} | bf16 max {np.abs(c1-want).max():.3e}"
          f" rel {np.abs(c1-want)[:, :256].max() / np.abs(want[:, :256]).max():.3e}", flush=True)
