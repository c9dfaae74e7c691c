import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import unet_numpy as un
from paper_2410_16727_b200 import spec
from paper_2410_16727_b200.sampler import SeedSampler
P, S, T = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
arch = spec.UNetArch(); params = spec.random_model()
s1 = SeedSampler(params, mode=1)
rng = np.random.default_rng(0)
cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
x = rng.standard_normal((P * S, T, 7)).astype(np.float32)
e1 = s1.predict_noise(x, 50, s1.film(cond), S).cpu().numpy()
if P * S <= 64:
    want = un.unet_forward(params, arch, x, 50, cond, S)
else:
    want = SeedSampler(params, mode=0).predict_noise(x, 50, SeedSampler(params, mode=0).film(cond), S).cpu().numpy()
d = e1 - want
print(f"P{P} S{S} T{T}: max {np.abs(d).max():.3e} rms {np.sqrt((d**2).mean()):.3e}", flush=True)
