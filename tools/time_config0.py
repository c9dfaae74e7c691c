"""BASELINE config 0 (1 problem x 32 seeds, 1x128x128 image, 4-layer encoder, 100 DDPM steps): sampler
call time in fp32 mode (the config's precision, SIMT) and bf16 mode (persistent tcgen05 kernel)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_16727_b200 import spec, synth  # noqa: E402
from paper_2410_16727_b200.sampler import SeedSampler  # noqa: E402

params = spec.random_model(spec.ENCODER_CFG0)
pb = synth.config0_problems(1, seed=0)
res = {}
for mode in (0, 1):
    smp = SeedSampler(params, spec.ENCODER_CFG0, mode=mode)
    q = torch.as_tensor(pb.q_start).cuda()
    im = torch.as_tensor(pb.images).cuda()
    g = torch.as_tensor(pb.goal).cuda()
    out = torch.empty((32, 32, 7), device="cuda")

    def call():
        fa = smp.film(smp.encode(im, q, g))
        smp.sample(fa, q, 32, out=out)

    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        call()
    e1.record()
    torch.cuda.synchronize()
    res["fp32" if mode == 0 else "bf16"] = {"ms_per_call": e0.elapsed_time(e1) / 10}
print(json.dumps({"config": "0: 1 problem x 32 seeds, encode + 100 DDPM steps", **res}))
