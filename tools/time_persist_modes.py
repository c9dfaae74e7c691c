"""100-step DDPM sampler time per call for a few batch sizes under the current env (A/B
helper for the persistent kernel's knobs).   python tools/time_persist_modes.py"""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2410_16727_b200 import spec, synth
from paper_2410_16727_b200.sampler import SeedSampler

s1 = SeedSampler(spec.random_model(), mode=1)
rng = np.random.default_rng(0)
res = []
for (P, S) in [(1, 32), (8, 32), (16, 32), (32, 32)]:
    cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
    q0 = synth.make_problems(P, seed=3).q_start
    fa = s1.film(cond)
    for _ in range(2):
        s1.sample(fa, q0, S)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.sample(fa, q0, S)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res.append(f"B={P * S}: {np.median(ts):.2f} ms")
print(os.environ.get("PS_PERSIST", "-"), os.environ.get("PS_PERSIST_WIDE_UNITS", "-"), " | ".join(res), flush=True)
