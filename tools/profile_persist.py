"""One persistent-sampler launch (1 problem x 32 seeds, 10-step DDIM) for ncu."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2410_16727_b200 import spec, synth
from paper_2410_16727_b200.sampler import SeedSampler

s1 = SeedSampler(spec.random_model(), mode=1)
rng = np.random.default_rng(0)
cond = np.concatenate([np.abs(rng.standard_normal((1, 256))) * 0.3, rng.uniform(0, 1, (1, 14))], 1)
q0 = synth.make_problems(1, seed=3).q_start
s1.sample(s1.film(cond), q0, 32, steps=spec.strided_steps(100, 10))
torch.cuda.synchronize()
print("ok")
