"""Stage breakdown of one small planning call (device events around each planner stage).
    python tools/time_small_plan.py [P] [S] [T]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2410_16727_b200 import bl, spec, synth
from paper_2410_16727_b200.planner import BLPlanner

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1
S = int(sys.argv[2]) if len(sys.argv) > 2 else 32
T = int(sys.argv[3]) if len(sys.argv) > 3 else 32
params = spec.random_model(spec.ENCODER_CFG3)
pl = BLPlanner(params, spec.ENCODER_CFG3, mode=1, S=S, T=T, steps=spec.strided_steps(100, 10), max_problems=P)
pb = synth.config3_problems(P, p0=0, seed=0)
dev = torch.device("cuda")
imgs, q, g, bx = (torch.as_tensor(a, device=dev) for a in (pb.images, pb.q_start, pb.goal, pb.boxes))
names = ["esdf", "encode", "film", "sample", "refine", "select"]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
acc = {n: [] for n in names}
for it in range(25):
    ev[0].record()
    esdf = pl.esdf[:P]
    pl._esdf_build(bx, esdf); ev[1].record()
    cond = pl.sampler.encode(imgs, q, g); ev[2].record()
    fa = pl.sampler.film(cond, out=pl.film_a[:P]); ev[3].record()
    seeds = pl.sampler.sample(fa, q, S, T, steps=pl.steps, out=pl.seeds[:P * S]); ev[4].record()
    out = tuple(o[:P * S] for o in pl.out)
    bl.refine(seeds, esdf, S, pl.robot, pl.grid, pl.cost, out=out, esdf_layout=pl.esdf_layout); ev[5].record()
    bl.select(out[1], out[2], S, out=pl.best[:P]); ev[6].record()
    torch.cuda.synchronize()
    if it >= 5:
        for i, n in enumerate(names):
            acc[n].append(ev[i].elapsed_time(ev[i + 1]))
print({n: round(float(np.median(v)), 3) for n, v in acc.items()}, "total", round(sum(float(np.median(v)) for v in acc.values()), 3))
