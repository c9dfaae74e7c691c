"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
the persistent sampler (2 DDPM steps), the layered tcgen05 U-Net incl. CTA-pair layers (PS_PERSIST=0),
the tcgen05 encoder, ESDF build, refinement and select."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_16727_b200 import bl, spec, synth  # noqa: E402
from paper_2410_16727_b200.sampler import SeedSampler  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
params = spec.random_model(spec.ENCODER_CFG3)
smp = SeedSampler(params, spec.ENCODER_CFG3, mode=1)
P, S = 1, 8
pb = synth.make_problems(P, seed=0, n_boxes=4, image_shape=(32, 48), n_images=2, n_rect=3)
if what in ("all", "encoder"):
    cond = smp.encode(pb.images, pb.q_start, pb.goal)
else:
    cond = torch.rand((P, spec.COND_DIM), device="cuda")
fa = smp.film(cond)
steps = np.array([100, 99])
if what in ("all", "persist"):
    os.environ["PS_PERSIST"] = "1"
    smp.sample(fa, pb.q_start, S, steps=None if False else steps)
if what in ("all", "layered"):
    os.environ["PS_PERSIST"] = "0"
    os.environ["PS_NO_GRAPH"] = "1"
    smp.predict_noise(torch.randn((P * S, 32, 7), device="cuda"), 50, fa, S)
if what in ("all", "refine"):
    grid = spec.GridSpec(n=(32, 32, 32), h=0.04, cube=1.28)
    esdf = bl.esdf_build(pb.boxes, grid, layout=bl.ESDF_BRICKED)
    q = synth.refine_init(P * S, seed=1)
    out = bl.refine(q, esdf, S, spec.make_bl_robot(), grid, spec.BLCost(), esdf_layout=bl.ESDF_BRICKED)
    bl.select(out[1], out[2], S)
torch.cuda.synchronize()
print("sanitize run ok", what)
