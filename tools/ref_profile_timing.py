"""Literal-reference timing of the ref profile: one `plan_diffusion`
call at planseed's shapes with 32 seeds x 10 refinement iterations, through
  --impl planseed : the reference itself (CPU, numpy + numba; importable only in the dev
                    container, where /root/reference exists), or
  --impl b200     : the drop-in ref profile (paper_2410_16727_b200.ref) on the GPU,
on the golden fixture's problem (tests/golden/ref_plan.npz).  Reports the reference's own
PlanResult timers: plan_time (encode + sample + refine + select, ESDF excluded) and esdf_time.

    python tools/ref_profile_timing.py --impl planseed --out profiles/r01_ref_profile_planseed_cpu.json
    python tools/ref_profile_timing.py --impl b200 --out gpurun_out/ref_profile_b200.json
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def modules(impl):
    if impl == "planseed":
        sys.path.insert(0, "/root/reference/pkg/src")
        from planseed import arm as arm_m, diffusion, geometry, pipeline
        return dict(default_arm=arm_m.default_arm, Pose2=arm_m.Pose2, SensorPose=geometry.SensorPose,
                    DepthScan=geometry.DepthScan, diffusion=diffusion, pipeline=pipeline)
    from paper_2410_16727_b200.ref import diffusion, pipeline, types
    return dict(default_arm=types.default_arm, Pose2=types.Pose2, SensorPose=types.SensorPose,
                DepthScan=types.DepthScan, diffusion=diffusion, pipeline=pipeline)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", choices=["planseed", "b200"], required=True)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--seeds", type=int, default=32)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    m = modules(args.impl)
    z = np.load(ROOT / "tests" / "golden" / "ref_plan.npz")
    arm = m["default_arm"]()
    net = m["diffusion"].create_net(m["diffusion"].arch_for_arm(arm), seed=3)
    p = z["pose"]
    pose = m["SensorPose"](position=(p[0], p[1]), heading=p[2], fov=p[3], max_range=p[4], n_rays=int(p[5]))
    scan = m["DepthScan"](pose=pose, depths=z["depths"])
    goal = m["Pose2"]((z["goal"][0], z["goal"][1]), z["goal"][2])
    sched = m["diffusion"].make_schedule()
    req = m["pipeline"].PlanRequest(q_start=z["q0"], goal=goal, scan=scan, n_trajs=args.seeds, n_iters=args.iters,
                                    n_denoising=5, seed=int(z["seed"]))
    m["pipeline"].plan_diffusion(arm, net, sched, req)          # warm-up (numba JIT / CUDA init)
    plan, esdf = [], []
    for _ in range(args.reps):
        r = m["pipeline"].plan_diffusion(arm, net, sched, req)
        plan.append(r.plan_time)
        esdf.append(r.esdf_time)
    out = {"impl": args.impl, "seeds": args.seeds, "refine_iters": args.iters, "denoising_steps": 5,
           "reps": args.reps, "plan_time_ms_p50": 1e3 * statistics.median(plan),
           "esdf_time_ms_p50": 1e3 * statistics.median(esdf), "cpu_count": os.cpu_count(),
           "note": "planseed.plan_diffusion timers (ESDF excluded from plan_time); single process as shipped"
           if args.impl == "planseed" else "drop-in ref profile on the GPU, same timers"}
    if args.impl == "b200":
        import torch
        out["device"] = torch.cuda.get_device_name(0)
    print(json.dumps(out))
    if args.out:
        Path(args.out).parent.mkdir(parents=True, exist_ok=True)
        Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
