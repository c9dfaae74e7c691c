#!/usr/bin/env python
"""Flag / best-index agreement of the bf16 GPU planner (BLPlanner.plan_batch, config-3 shapes) with
the oracle pipeline (oracle/pipeline_cpu.plan_problem: C ESDF, numpy encoder + U-Net + DDPM, C
refinement, select) over a batch of problems.  The oracle runs one problem per host process.

  python tools/agreement.py [--problems 64] [--check 32] [--dtype float32|float64] [--mode 1]

Prints one JSON line: per-trajectory flag agreement, per-problem best-index agreement, the rate at
which the GPU's chosen seed is feasible vs the oracle's, and the seed / refined-trajectory
deviation statistics of the checked problems.
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problems", type=int, default=64)
    ap.add_argument("--check", type=int, default=32)
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--mode", type=int, default=1)
    ap.add_argument("--p0", type=int, default=0)
    ap.add_argument("--wide", action="store_true", help="synth.config3_wide scene (mixed flags)")
    a = ap.parse_args()
    import torch

    import oracle
    from oracle import pipeline_cpu as pc
    from paper_2410_16727_b200 import spec, synth
    from paper_2410_16727_b200.planner import BLPlanner

    oracle.build()
    S = 32
    params = spec.random_model(spec.ENCODER_CFG3)
    kw = {}
    if a.wide:
        pb, kw["grid"], kw["robot"] = synth.config3_wide(a.problems, p0=a.p0, seed=0)
    else:
        pb = synth.config3_problems(a.problems, p0=a.p0, seed=0)
    pl = BLPlanner(params, spec.ENCODER_CFG3, mode=a.mode, S=S, max_problems=a.problems, **kw)
    r = pl.plan_batch(pb.images, pb.q_start, pb.goal, pb.boxes, p0=pb.p0)
    gq = np.asarray(r.trajectories).reshape(a.problems, S, 32, 7)
    gf = np.asarray(r.feasible).astype(bool).reshape(a.problems, S)
    gb = np.asarray(r.best_index)
    idx = np.linspace(0, a.problems - 1, a.check).round().astype(int)
    dt = np.float32 if a.dtype == "float32" else np.float64
    t0 = time.perf_counter()
    workers = min(len(idx), os.cpu_count() or 1)
    with ProcessPoolExecutor(max_workers=workers, initializer=pc._init_worker, initargs=(5,)) as ex:
        futs = [ex.submit(pc.plan_problem, a.p0 + int(i), full=True, dtype=dt, wide=a.wide) for i in idx]
        res = [f.result() for f in futs]
    wall = time.perf_counter() - t0
    of = np.stack([x[3] for x in res])
    ob = np.array([x[0] for x in res])
    oq = np.stack([x[1] for x in res])
    d = np.abs(gq[idx] - oq).reshape(len(idx) * S, -1).max(1)
    line = {
        "problems_gpu": a.problems, "problems_checked": int(len(idx)), "trajectories_checked": int(len(idx) * S),
        "gpu_mode": "bf16" if a.mode == 1 else "fp32", "oracle_dtype": a.dtype,
        "scene": "config3_wide (2.5 cm grid, base at centre)" if a.wide else "config 3",
        "clamped_rate_gpu": float(np.asarray(r.clamped).astype(bool).mean()),
        "flag_agreement": float(np.mean(gf[idx] == of)),
        "best_index_agreement": float(np.mean(gb[idx] == ob)),
        "gpu_best_feasible": float(np.mean(gf[idx][np.arange(len(idx)), gb[idx]])),
        "oracle_best_feasible": float(np.mean(of[np.arange(len(idx)), ob])),
        "feasible_rate_gpu": float(gf[idx].mean()), "feasible_rate_oracle": float(of.mean()),
        "refined_maxabs_p50": float(np.median(d)), "refined_maxabs_p99": float(np.quantile(d, 0.99)),
        "oracle_wall_s": wall, "oracle_workers": workers,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
