"""B200-native seeding hot path of DiffusionSeeder (arXiv 2410.16727).

Batched conditional diffusion sampling of seed trajectories followed by fused
collision/smoothness refinement, feasibility flags and best-seed selection, as
hand-written sm_100a CUDA behind the C-ABI in include/ps_b200.h.  The host layer
keeps the sampler / refiner / planner API of the reference package `planseed`
(/root/reference/pkg/src/planseed) and adds batched-over-problems variants.

Modules
  spec, synth   BASELINE-profile pinned choices and seeded synthetic inputs
  bl            BASELINE-profile ESDF build / refine / select over the C-ABI
  _lib, build   the ctypes binding and the in-tree nvcc build
"""

__version__ = "0.1.0"
