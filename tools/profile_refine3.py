"""Config-3 refinement workload for ncu: 1024 problems' ESDFs built in the planner's 4^3-brick
layout, then one fused refinement of 1024 x 32 trajectories (one launch of each kernel)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2410_16727_b200 import bl, spec, synth

robot, grid, cost = spec.make_bl_robot(), spec.GridSpec(), spec.BLCost()
P = 1024
pb = synth.make_problems(P, seed=0)
bx = torch.as_tensor(pb.boxes, device="cuda")
esdf = bl.esdf_build(bx, grid, layout=bl.ESDF_BRICKED)
q = torch.as_tensor(synth.refine_init(P * 32, seed=2), device="cuda")
bl.refine(q, esdf, 32, robot, grid, cost, esdf_layout=bl.ESDF_BRICKED)
torch.cuda.synchronize()
print("ok")
