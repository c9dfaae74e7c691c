"""Device timing of the sampler at config-1/config-3 sizes."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2410_16727_b200 import spec, synth
from paper_2410_16727_b200.sampler import SeedSampler

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
S = 32
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 1
params = spec.random_model(spec.ENCODER_CFG3)
smp = SeedSampler(params, spec.ENCODER_CFG3, mode=mode)
rng = np.random.default_rng(0)
cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
fa = smp.film(cond)
x = torch.randn(P * S, 32, 7, device="cuda")
def ev(fn, reps):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
ms_fwd = ev(lambda: smp.predict_noise(x, 50, fa, S), 5)
flops = P * S * spec.UNetArch().flops_per_traj_step(32)
res = {"P": P, "mode": mode, "fwd_ms": ms_fwd, "fwd_TFLOPs": flops / ms_fwd / 1e9}
q0 = torch.zeros(P, 7, device="cuda")
ms_s = ev(lambda: smp.sample(fa, q0, S, steps=spec.strided_steps(100, 10)), 2)
res["ddim10_ms"] = ms_s
pb = synth.config3_problems(min(P, 64), seed=0)
imgs = torch.as_tensor(pb.images, device="cuda")
ms_enc = ev(lambda: smp.encode(imgs, pb.q_start, pb.goal), 3)
res["encode_ms_per_64_problems"] = ms_enc
print(json.dumps(res))
