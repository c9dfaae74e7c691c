import sys, json
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
for _ in range(2): smp.predict_noise(x, 50, fa, 32)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): smp.predict_noise(x, 50, fa, 32)
e.record(); torch.cuda.synchronize()
print(json.dumps({"P": P, "fwd_ms": s.elapsed_time(e) / 10}))
