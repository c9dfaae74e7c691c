"""eps of the layered U-Net at P problems (layered path) -> npy: python tools/mb2_check.py out.npy [P]"""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_16727_b200 import spec  # noqa: E402
from paper_2410_16727_b200.sampler import SeedSampler  # noqa: E402

os.environ["PS_PERSIST"] = "0"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 40
smp = SeedSampler(spec.random_model(), mode=1)
rng = np.random.default_rng(0)
cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
x = rng.standard_normal((P * 32, 32, 7)).astype(np.float32)
eps = smp.predict_noise(x, 50, smp.film(cond), 32).cpu().numpy()
np.save(sys.argv[1], eps)
if len(sys.argv) > 3:
    from oracle import unet_numpy as un
    want = un.unet_forward(spec.random_model(), spec.UNetArch(), x[:64], 50, cond[:2], 32)
    d = eps[:64] - want
    print("vs oracle rel RMS", np.sqrt((d ** 2).mean() / (want ** 2).mean()))
