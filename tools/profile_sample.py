"""DDPM-100 sampler call at P problems x 32 seeds (layered tcgen05 path), for ncu captures of
the bench's own kernels (final-layer DDPM epilogue included)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_16727_b200 import spec  # noqa: E402
from paper_2410_16727_b200.sampler import SeedSampler  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
smp = SeedSampler(spec.random_model(), mode=1)
rng = np.random.default_rng(0)
cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
q = rng.uniform(-1, 1, (P, 7)).astype(np.float32)
out = smp.sample(smp.film(cond), q, 32)
torch.cuda.synchronize()
print("ok", bool(torch.isfinite(out).all()))
