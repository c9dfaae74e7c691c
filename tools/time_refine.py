"""Quick device timing of the fused refine kernel (config 2 and config-3-like)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2410_16727_b200 import bl, spec, synth

robot, grid, cost = spec.make_bl_robot(), spec.GridSpec(), spec.BLCost()
def timeit(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
res = {}
# config 2
boxes = synth.make_problems(1, seed=0).boxes
esdf = bl.esdf_build(boxes, grid)
q = torch.as_tensor(synth.refine_init(2048, seed=1), device="cuda")
outs = (torch.empty_like(q), torch.empty(2048, device="cuda"), torch.empty(2048, dtype=torch.uint8, device="cuda"), torch.empty(2048, dtype=torch.uint8, device="cuda"))
ms = timeit(lambda: bl.refine(q, esdf[0], 2048, robot, grid, cost, out=outs))
res["cfg2_refine_ms"] = ms
res["cfg2_GBps_alg"] = 2048 * 10 * 52992 / (ms * 1e-3) / 1e9
esdf_b = bl.esdf_build(boxes, grid, layout=bl.ESDF_BRICKED)
ms_b = timeit(lambda: bl.refine(q, esdf_b[0], 2048, robot, grid, cost, out=outs, esdf_layout=bl.ESDF_BRICKED))
res["cfg2_bricked_refine_ms"] = ms_b
esdf_q = bl.esdf_build(boxes, grid, layout=bl.ESDF_QUAD)
ms_q = timeit(lambda: bl.refine(q, esdf_q[0], 2048, robot, grid, cost, out=outs, esdf_layout=bl.ESDF_QUAD))
res["cfg2_quad_refine_ms"] = ms_q
res["cfg2_quad_GBps_alg"] = 2048 * 10 * 52992 / (ms_q * 1e-3) / 1e9
# config 3-like: 1024 problems x 32 seeds, per-problem ESDF
P = 1024
pb = synth.make_problems(P, seed=0)
bx = torch.as_tensor(pb.boxes, device="cuda")
ms_e = timeit(lambda: bl.esdf_build(bx, grid), reps=3)
res["cfg3_esdf_ms"] = ms_e
esdf3 = bl.esdf_build(bx, grid)
q3 = torch.as_tensor(synth.refine_init(P * 32, seed=2), device="cuda")
outs3 = (torch.empty_like(q3), torch.empty(P*32, device="cuda"), torch.empty(P*32, dtype=torch.uint8, device="cuda"), torch.empty(P*32, dtype=torch.uint8, device="cuda"))
ms3 = timeit(lambda: bl.refine(q3, esdf3, 32, robot, grid, cost, out=outs3), reps=5)
res["cfg3_refine_ms"] = ms3
res["cfg3_GBps_alg"] = P * 32 * 10 * 52992 / (ms3 * 1e-3) / 1e9
print(json.dumps(res))
# the planner's layout: 4^3 bricks
esdf3b = bl.esdf_build(bx, grid, layout=bl.ESDF_BRICKED)
ms3b = timeit(lambda: bl.refine(q3, esdf3b, 32, robot, grid, cost, out=outs3, esdf_layout=bl.ESDF_BRICKED), reps=5)
print(json.dumps({"cfg3_refine_bricked_ms": ms3b, "cfg3_bricked_GBps_alg": P * 32 * 10 * 52992 / (ms3b * 1e-3) / 1e9}))
