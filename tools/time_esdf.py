"""ESDF build time for P config-3 problems (bricked layout), CUDA events; compares with the C-order
layout's values for one problem (bit-exact check against the oracle is in tests/test_bl_gpu.py)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2410_16727_b200 import bl, spec, synth  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
pb = synth.config3_problems(P, seed=0)
boxes = torch.as_tensor(pb.boxes).cuda()
grid = spec.GridSpec()
out = torch.empty((P,) + grid.n, device="cuda")
for _ in range(2):
    bl.esdf_build(boxes, grid, layout=bl.ESDF_BRICKED, out=out)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    bl.esdf_build(boxes, grid, layout=bl.ESDF_BRICKED, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"esdf_build P={P}: {ms:.3f} ms, {P * grid.n_nodes * 4 / ms / 1e6:.0f} GB/s written; checksum {out.double().sum().item():.6e}")
