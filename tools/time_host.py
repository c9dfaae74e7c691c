import sys, json, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2410_16727_b200 import spec
from paper_2410_16727_b200.sampler import SeedSampler
P = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
smp = SeedSampler(spec.random_model(), mode=1)
rng = np.random.default_rng(0)
cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
fa = smp.film(cond); x = torch.randn(P * 32, 32, 7, device="cuda")
for _ in range(3): smp.predict_noise(x, 50, fa, 32)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10): smp.predict_noise(x, 50, fa, 32)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
q0 = torch.zeros(P, 7, device="cuda")
smp.sample(fa, q0, 32, steps=spec.strided_steps(100, 10)); torch.cuda.synchronize()
t3 = time.perf_counter()
smp.sample(fa, q0, 32, steps=spec.strided_steps(100, 10))
t4 = time.perf_counter(); torch.cuda.synchronize(); t5 = time.perf_counter()
print(json.dumps({"host_ms_per_fwd": (t1 - t0) * 100, "wall_ms_per_fwd": (t2 - t0) * 100,
                  "sample10_host_ms": (t4 - t3) * 1e3, "sample10_wall_ms": (t5 - t3) * 1e3}))
