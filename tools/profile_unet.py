"""Small, repeatable U-Net workload for ncu: mode-1 predict_noise at P problems x 32 seeds."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2410_16727_b200 import spec
from paper_2410_16727_b200.sampler import SeedSampler
P = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
smp = SeedSampler(spec.random_model(), mode=1)
rng = np.random.default_rng(0)
cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
fa = smp.film(cond)
x = torch.randn(P * 32, 32, 7, device="cuda")
for _ in range(reps):
    smp.predict_noise(x, 50, fa, 32)
torch.cuda.synchronize()
print("ok")
