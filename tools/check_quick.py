import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import unet_numpy as un
from paper_2410_16727_b200 import spec
from paper_2410_16727_b200.sampler import SeedSampler
arch = spec.UNetArch(); params = spec.random_model()
s1 = SeedSampler(params, mode=1)
rng = np.random.default_rng(0)
for (P, S, T, k) in [(1, 16, 32, 50), (2, 8, 64, 20)]:
    cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
    x = rng.standard_normal((P * S, T, 7)).astype(np.float32)
    e1 = s1.predict_noise(x, k, s1.film(cond), S).cpu().numpy()
    want = un.unet_forward(params, arch, x, k, cond, S)
    d = e1 - want
    print(f"T{T}: bf16 max {np.abs(d).max():.3e} rms {np.sqrt((d**2).mean()):.3e}", flush=True)
