"""Config-2 refinement (one shared ESDF, 2048 trajectories) in C-order and quad-brick layouts, for ncu."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_16727_b200 import bl, spec, synth  # noqa: E402

robot, grid, cost = spec.make_bl_robot(), spec.GridSpec(), spec.BLCost()
boxes = synth.make_problems(1, seed=0).boxes
q = torch.as_tensor(synth.refine_init(2048, seed=1), device="cuda")
for layout in (bl.ESDF_C_ORDER, bl.ESDF_QUAD):
    e = bl.esdf_build(boxes, grid, layout=layout)[0]
    for _ in range(2):
        bl.refine(q, e, 2048, robot, grid, cost, esdf_layout=layout)
torch.cuda.synchronize()
print("ok")
