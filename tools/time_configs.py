"""BASELINE configs 0-2 on one B200 (the bench line is config 3): device time per call with CUDA
events after warm-up.  python tools/time_configs.py > profiles/r02_configs012.json
  config 0: 1 problem x 32 seeds, 1x128x128 image, 4-layer encoder, 100 DDPM steps -- encode +
            sample in fp32 (the config's precision) and bf16, and the whole planning call
            (ESDF + encode + sample + 10 refinement iterations + flags + select) in bf16;
  config 1: 64 problems x 32 seeds, batched sampling only (encode + 100 DDPM steps), bf16;
  config 2: refinement only, 2048 trajectories against one 128^3 ESDF, fp32 (bricked and quad
            layouts), with the algorithmic-bytes rate against the measured HBM peak."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_16727_b200 import bl, spec, synth  # noqa: E402
from paper_2410_16727_b200.planner import BLPlanner  # noqa: E402
from paper_2410_16727_b200.sampler import SeedSampler  # noqa: E402

peaks = json.load(open(Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"))


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


res = {}
params0 = spec.random_model(spec.ENCODER_CFG0)
# config 0
pb0 = synth.config0_problems(1, seed=0)
c0 = {}
for mode, name in ((0, "fp32"), (1, "bf16")):
    smp = SeedSampler(params0, spec.ENCODER_CFG0, mode=mode)
    q, im, g = (torch.as_tensor(a).cuda() for a in (pb0.q_start, pb0.images, pb0.goal))
    out = torch.empty((32, 32, 7), device="cuda")
    ms = timeit(lambda: smp.sample(smp.film(smp.encode(im, q, g)), q, 32, out=out))
    c0[name + "_encode_sample_ms"] = ms
pl0 = BLPlanner(params0, spec.ENCODER_CFG0, mode=1, S=32, max_problems=1, n_images=1, image_shape=(128, 128))
d0 = [torch.as_tensor(a).cuda() for a in (pb0.images, pb0.q_start, pb0.goal, pb0.boxes)]
c0["bf16_plan_call_ms"] = timeit(lambda: pl0.plan_batch_device(*d0))
c0["note"] = "1 problem x 32 seeds; small batch: the persistent single-launch sampler"
res["config0"] = c0
# config 1
P1 = 64
pb1 = synth.config0_problems(P1, seed=1)
smp1 = SeedSampler(params0, spec.ENCODER_CFG0, mode=1)
q1, im1, g1 = (torch.as_tensor(a).cuda() for a in (pb1.q_start, pb1.images, pb1.goal))
out1 = torch.empty((P1 * 32, 32, 7), device="cuda")
fa1 = smp1.film(smp1.encode(im1, q1, g1))
ms_s = timeit(lambda: smp1.sample(fa1, q1, 32, out=out1))
ms_all = timeit(lambda: smp1.sample(smp1.film(smp1.encode(im1, q1, g1)), q1, 32, out=out1))
res["config1"] = {"problems": P1, "seeds": 32, "encode_sample_ms": ms_all, "sample_ms": ms_s,
                  "ms_per_denoising_step": ms_s / 100, "trajectories_per_s": P1 * 32 / (ms_all * 1e-3),
                  "note": "B*T = 65,536 > 8,192: the layered tcgen05 kernels in a CUDA graph"}
# config 2
robot, grid, cost = spec.make_bl_robot(), spec.GridSpec(), spec.BLCost()
boxes = synth.make_problems(1, seed=0).boxes
q2 = torch.as_tensor(synth.refine_init(2048, seed=1), device="cuda")
outs = (torch.empty_like(q2), torch.empty(2048, device="cuda"), torch.empty(2048, dtype=torch.uint8, device="cuda"),
        torch.empty(2048, dtype=torch.uint8, device="cuda"))
alg = 2048 * 10 * 52992
c2 = {"trajectories": 2048, "algorithmic_bytes": alg}
for lay, name in ((bl.ESDF_BRICKED, "bricked"), (bl.ESDF_QUAD, "quad")):
    e = bl.esdf_build(boxes, grid, layout=lay)
    ms = timeit(lambda: bl.refine(q2, e[0], 2048, robot, grid, cost, out=outs, esdf_layout=lay))
    c2[name] = {"refine_ms": ms, "GBps_algorithmic": alg / (ms * 1e-3) / 1e9,
                "frac_of_hbm_peak": alg / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"]}
res["config2"] = c2
print(json.dumps(res, indent=1))
