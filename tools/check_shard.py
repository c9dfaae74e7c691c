"""Which stage of the planner breaks shard invariance?  Plans problems [0, 5) in one call and as
[0, 2) + [2, 5), comparing cond, FiLM, seeds and refined trajectories stage by stage."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_16727_b200 import spec, synth  # noqa: E402
from paper_2410_16727_b200.planner import BLPlanner  # noqa: E402

params = spec.random_model(spec.ENCODER_CFG3)
S = 32
out = {}
for name, parts in (("one", [(0, 5)]), ("two", [(0, 2), (2, 5)])):
    res = {k: [] for k in ("cond", "fa", "seeds", "traj")}
    for a, b in parts:
        pl = BLPlanner(params, spec.ENCODER_CFG3, mode=1, S=S, max_problems=5)
        pb = synth.config3_problems(b - a, p0=a, seed=0)
        d = [torch.as_tensor(x).cuda() for x in (pb.images, pb.q_start, pb.goal, pb.boxes)]
        cond = pl.sampler.encode(d[0], d[1], d[2])
        fa = pl.sampler.film(cond)
        r = pl.plan_batch_device(*d, p0=a)
        res["cond"].append(cond.cpu().numpy())
        res["fa"].append(fa.cpu().numpy())
        res["seeds"].append(r.seeds.cpu().numpy())
        res["traj"].append(r.trajectories.cpu().numpy())
    out[name] = {k: np.concatenate(v) for k, v in res.items()}
for k in ("cond", "fa", "seeds", "traj"):
    x, y = out["one"][k], out["two"][k]
    print(k, "equal" if np.array_equal(x, y) else f"maxdiff {np.abs(x - y).max():.3e}",
          "rows differing:", np.unique(np.nonzero((x != y).reshape(len(x), -1).any(1))[0] // (S if k in ("seeds", "traj") else 1)))
