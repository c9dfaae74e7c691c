"""Reference-profile drop-in: planseed's own sampler / refiner / planner API
(src/diffusion.py, src/trajopt.py, src/pipeline.py) on sm_100a CUDA kernels.

    from paper_2410_16727_b200.ref import trajopt, diffusion, pipeline
    pipeline.plan_diffusion(arm, net, schedule, req)   # same call as planseed's

Objects from planseed itself (ArmModel, SdfGrid, DenoiserNet, DepthScan, Pose2,
CostWeights) are accepted as well as this package's compatible types."""

from . import diffusion, pipeline, train, trajopt, types  # noqa: F401
