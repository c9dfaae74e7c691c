"""Debug: bf16 predict_noise at P problems vs fp32 SIMT mode; NaN count and error."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2410_16727_b200 import spec
from paper_2410_16727_b200.sampler import SeedSampler
P = int(sys.argv[1]) if len(sys.argv) > 1 else 128
params = spec.random_model()
s0, s1 = SeedSampler(params, mode=0), SeedSampler(params, mode=1)
rng = np.random.default_rng(5)
cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
x = np.random.default_rng(P).standard_normal((P * 32, 32, 7)).astype(np.float32)
e0 = s0.predict_noise(x, 40, s0.film(cond), 32).cpu().numpy()
e1 = s1.predict_noise(x, 40, s1.film(cond), 32).cpu().numpy()
bad = ~np.isfinite(e1)
print("P", P, "PDL off" if os.environ.get("PS_NO_PDL") else "PDL on", "nonfinite", bad.sum(),
      "first bad traj", np.nonzero(bad.any(axis=(1, 2)))[0][:10])
d = np.where(bad, 0, e1 - e0)
print("rel rms (finite)", np.sqrt((d ** 2).mean()) / np.sqrt((e0 ** 2).mean()))
