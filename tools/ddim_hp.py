"""bf16 strided DDIM from k = 100 with an fp32 prefix: accuracy against the float64 oracle and the
sampler's cost at 1024 x 32 for n_hp = 0 / 1 / 2 fp32 steps (hp_rsq None / 100 / 4)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import unet_numpy as un  # noqa: E402
from paper_2410_16727_b200 import spec, synth  # noqa: E402
from paper_2410_16727_b200.sampler import SeedSampler  # noqa: E402

params = spec.random_model()
ARCH = spec.UNetArch()
steps = spec.strided_steps(100, 10)
rng = np.random.default_rng(23)
P, S = 2, 16
cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
q0 = synth.make_problems(P, seed=29).q_start
want = un.sample(params, ARCH, cond, q0, S, steps=steps)
PB = 1024
condb = np.concatenate([np.abs(rng.standard_normal((PB, 256))) * 0.3, rng.uniform(0, 1, (PB, 14))], 1)
qb = synth.make_problems(PB, seed=5).q_start
for hp in (None, 100.0, 4.0, 2.5):
    smp = SeedSampler(params, mode=1, hp_rsq=hp)
    got = smp.sample(smp.film(cond), q0, S, steps=steps).cpu().numpy()
    d = got - want
    fa = smp.film(condb)
    qd = torch.as_tensor(qb).cuda()
    out = torch.empty((PB * 32, 32, 7), device="cuda")
    for _ in range(2):
        smp.sample(fa, qd, 32, steps=steps, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        smp.sample(fa, qd, 32, steps=steps, out=out)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"hp_rsq": hp, "n_hp": smp.hp_steps(steps), "rms": float(np.sqrt((d ** 2).mean())),
                      "max": float(np.abs(d).max()), "ms_1024x32": e0.elapsed_time(e1) / 5}), flush=True)
