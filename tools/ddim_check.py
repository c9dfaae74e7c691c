"""bf16 DDIM conditioning check: persistent / layered / fp32 paths against the fp64 oracle\n(python tools/ddim_check.py [comma-separated 1-based steps])."""
import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from oracle import unet_numpy as un
from paper_2410_16727_b200 import spec, synth
from paper_2410_16727_b200.sampler import SeedSampler
params = spec.random_model(); ARCH = spec.UNetArch()
s0 = SeedSampler(params, mode=0); s1 = SeedSampler(params, mode=1)
rng = np.random.default_rng(23)
P, S = 2, 16
cond = np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)
q0 = synth.make_problems(P, seed=29).q_start
steps = np.array([int(v) for v in sys.argv[1].split(",")]) if len(sys.argv) > 1 else spec.strided_steps(100, 10)
fa = s1.film(cond)
def run(m):
    os.environ["PS_PERSIST"] = m
    r = s1.sample(fa, q0, S, steps=steps).cpu().numpy(); os.environ.pop("PS_PERSIST"); return r
tp, tl = run("1"), run("0")
t0 = s0.sample(s0.film(cond), q0, S, steps=steps).cpu().numpy()
want = un.sample(params, ARCH, cond, q0, S, steps=steps)
f = lambda d: f"rms {np.sqrt((d**2).mean()):.3e} max {np.abs(d).max():.3e}"
print("persist-oracle", f(tp - want)); print("layered-oracle", f(tl - want)); print("fp32-oracle", f(t0 - want)); print("persist-layered", f(tp - tl))
for st in [1, 2, 5]:
    sts = steps[:st]
    os.environ["PS_PERSIST"]="1"; a = s1.sample(fa, q0, S, steps=sts).cpu().numpy()
    os.environ["PS_PERSIST"]="0"; b = s1.sample(fa, q0, S, steps=sts).cpu().numpy(); os.environ.pop("PS_PERSIST")
    print(st, "steps: persist-layered", f(a - b))
