"""Config-3 refinement on per-problem quad-brick ESDFs (34 GB for 1024 problems) against the
bricked layout: is the refine L1-wavefront bound at config 3 too?  python tools/time_refine_quad3.py"""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2410_16727_b200 import bl, spec, synth  # noqa: E402

robot, grid, cost = spec.make_bl_robot(), spec.GridSpec(), spec.BLCost()


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


P = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
pb = synth.make_problems(P, seed=0)
bx = torch.as_tensor(pb.boxes, device="cuda")
q = torch.as_tensor(synth.refine_init(P * 32, seed=2), device="cuda")
outs = (torch.empty_like(q), torch.empty(P * 32, device="cuda"), torch.empty(P * 32, dtype=torch.uint8, device="cuda"),
        torch.empty(P * 32, dtype=torch.uint8, device="cuda"))
res = {"P": P}
eb = bl.esdf_build(bx, grid, layout=bl.ESDF_BRICKED)
res["build_bricked_ms"] = timeit(lambda: bl.esdf_build(bx, grid, layout=bl.ESDF_BRICKED, out=eb), 3)
res["refine_bricked_ms"] = timeit(lambda: bl.refine(q, eb, 32, robot, grid, cost, out=outs, esdf_layout=bl.ESDF_BRICKED))
ref_out = [o.clone() for o in outs]
del eb
torch.cuda.empty_cache()
eq = bl.esdf_build(bx, grid, layout=bl.ESDF_QUAD)
res["build_quad_ms"] = timeit(lambda: bl.esdf_build(bx, grid, layout=bl.ESDF_QUAD, out=eq), 3)
res["refine_quad_ms"] = timeit(lambda: bl.refine(q, eq, 32, robot, grid, cost, out=outs, esdf_layout=bl.ESDF_QUAD))
res["bitwise_equal"] = all(bool(torch.equal(a, b)) for a, b in zip(outs, ref_out))
alg = P * 32 * 10 * 52992
res["quad_GBps_alg"] = alg / (res["refine_quad_ms"] * 1e-3) / 1e9
res["bricked_GBps_alg"] = alg / (res["refine_bricked_ms"] * 1e-3) / 1e9
print(json.dumps(res))
