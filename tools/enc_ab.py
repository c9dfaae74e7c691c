"""Encoder output + timing of the working build (or PS_LIB_OVERRIDE): python tools/enc_ab.py out.npy"""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_16727_b200 import spec, synth  # noqa: E402
from paper_2410_16727_b200.sampler import SeedSampler  # noqa: E402

P = 1024
smp = SeedSampler(spec.random_model(spec.ENCODER_CFG3), spec.ENCODER_CFG3, mode=1)
pb = synth.config3_problems(P, seed=0)
im = torch.as_tensor(pb.images, device="cuda")
q = torch.as_tensor(pb.q_start, device="cuda")
g = torch.as_tensor(pb.goal, device="cuda")
out = torch.empty((P, spec.COND_DIM), device="cuda")
for _ in range(3):
    smp.encode(im, q, g, out=out)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    smp.encode(im, q, g, out=out)
e.record()
torch.cuda.synchronize()
np.save(sys.argv[1], out.cpu().numpy())
print(json.dumps({"encode_ms": s.elapsed_time(e) / 10}))
