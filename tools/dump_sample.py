"""Dump sampler outputs of the layered tcgen05 path (and the noise prediction) to an npz, for
bitwise A/B of two builds (PS_LIB_OVERRIDE): python tools/dump_sample.py out.npz"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_16727_b200 import spec  # noqa: E402
from paper_2410_16727_b200.sampler import SeedSampler  # noqa: E402

os.environ["PS_PERSIST"] = "0"
params = spec.random_model()
smp = SeedSampler(params, mode=1)
rng = np.random.default_rng(0)
res = {}
for P, S, steps in [(64, 32, None), (8, 32, [100, 89, 78, 67, 56, 45, 34, 23, 12, 1]), (1200, 32, None)]:
    cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
    q = rng.uniform(-1, 1, (P, 7)).astype(np.float32)
    fa = smp.film(cond)
    out = smp.sample(fa, q, S, steps=steps)
    torch.cuda.synchronize()
    res[f"traj_P{P}"] = out.cpu().numpy()
    if P == 64:
        x = rng.standard_normal((P * S, 32, 7)).astype(np.float32)
        res["eps_P64"] = smp.predict_noise(x, 50, fa, S).cpu().numpy()
np.savez(sys.argv[1], **res)
print({k: (v.shape, bool(np.isfinite(v).all())) for k, v in res.items()})
