"""ORACLE (test infrastructure / CPU baseline only): the BASELINE-profile planning
pipeline on host cores -- canonical-fp32 C ESDF build, numpy encoder + U-Net + DDPM
(float32), C refinement, flags and best-seed selection -- one problem per process.

bench.py times this as `cpu_baseline` and as the `--impl reference` arm: the reference
package (planseed) is pure Python and cannot run the BASELINE shapes, so this port of
its algorithm to those shapes is the CPU reference (SURVEY.md §8(d) "CPU baseline").
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

_STATE = {}


def _init_worker(enc_layers: int):
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    from paper_2410_16727_b200 import spec
    enc = spec.ENCODER_CFG3 if enc_layers == 5 else spec.ENCODER_CFG0
    _STATE["params"] = spec.random_model(enc)
    _STATE["enc"] = enc


def plan_problem(p: int, seed: int = 0, S: int = 32, T: int = 32, steps=None, n_iters: int = 10,
                 enc_layers: int = 5, full: bool = False, dtype=np.float32, wide: bool = False):
    """Plan one synthetic config-3 problem on one core; returns (best, traj_best, seconds), or with
    full=True (best, refined (S,T,7), cost (S,), feasible (S,), seconds)."""
    import oracle
    from oracle import unet_numpy as un
    from paper_2410_16727_b200 import spec, synth

    if "params" not in _STATE:
        _init_worker(enc_layers)
    t0 = time.perf_counter()
    grid, cost, robot = spec.GridSpec(), spec.BLCost(), spec.make_bl_robot()
    if wide:
        pb, grid, robot = synth.config3_wide(1, p0=p, seed=seed)
    else:
        pb = synth.config3_problems(1, p0=p, seed=seed) if enc_layers == 5 else synth.config0_problems(1, p0=p, seed=seed)
    esdf = oracle.esdf_build(pb.boxes[0], grid)
    cond = un.encode_problems(_STATE["params"], _STATE["enc"], pb.images, pb.q_start, pb.goal,
                              dtype=dtype)
    seeds = un.sample(_STATE["params"], spec.UNetArch(), cond, pb.q_start, S, p0=p, T=T, steps=steps,
                      dtype=dtype)
    ps = oracle.BLProblemSet(robot, grid, cost, esdf[None], grid.n_nodes)
    q, c, f, _ = oracle.bl_refine(ps, seeds.astype(np.float32), S, n_iters)
    best = int(oracle.select(c, f, S)[0])
    if full:
        return best, q, c, f, time.perf_counter() - t0
    return best, q[best], time.perf_counter() - t0


def run_parallel(n_problems: int, workers: int, p0: int = 0, **kw):
    """Plan problems [p0, p0+n) on `workers` processes; returns (wall seconds, results)."""
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=workers, initializer=_init_worker,
                             initargs=(kw.get("enc_layers", 5),)) as ex:
        futs = [ex.submit(plan_problem, p0 + i, **kw) for i in range(n_problems)]
        res = [f.result() for f in futs]
    return time.perf_counter() - t0, res
