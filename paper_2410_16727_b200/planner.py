"""Batched BASELINE-profile planner: the seeding hot path end to end on one GPU.

plan_batch() is the batched counterpart of planseed's plan_diffusion
(pipeline.py:172-209) for P problems at once:

  ESDF build (per-problem boxes)  ~ build_planner_esdf     pipeline.py:115-132
  encode (depth images -> cond)   ~ encode_condition       diffusion.py:260-269
  sample (DDPM / strided DDIM)    ~ ddim_sample            diffusion.py:559-569
  refine (fixed-step) + flags     ~ optimize + planner_success  trajopt.py:140-177,
                                                                 pipeline.py:139-157
  select                          ~ select_best            pipeline.py:160-165

All device buffers are preallocated for the maximum batch (no allocation in the
hot path); inputs can be device tensors (device-resident mode) or host arrays
(end-to-end mode: host->device copies and the result read-back are part of the call).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import _lib, bl, spec
from .sampler import SeedSampler


@dataclass(frozen=True)
class GuidanceParams:
    """planseed pipeline.GuidanceParams (pipeline.py:58-61): cost-guided DDIM seeding."""

    k_guide_frac: float = 0.6
    n_grad: int = 20
    alpha_guide: float = 1.0


@dataclass
class PlanBatchResult:
    trajectories: object    # (P*S, T, 7) refined, physical radians
    seeds: object           # (P*S, T, 7) sampler output
    cost: object            # (P*S,)
    feasible: object        # (P*S,) bool/uint8
    clamped: object         # (P*S,)
    best_index: object      # (P,) int32


class BLPlanner:
    def __init__(self, params: dict, enc: spec.EncoderArch = spec.ENCODER_CFG3,
                 arch: spec.UNetArch = spec.UNetArch(), mode: int = 1, S: int = 32,
                 T: int = spec.T_DEFAULT, robot: spec.DHRobot | None = None,
                 grid: spec.GridSpec = spec.GridSpec(), cost: spec.BLCost = spec.BLCost(),
                 steps=None, max_problems: int = 1024, n_images: int = 2,
                 image_shape=(240, 320), n_boxes: int = spec.N_BOXES, hp_rsq: float | None = None, betas=None,
                 strict: bool = False, guidance: GuidanceParams | None = None):
        torch = _lib.require_cuda()
        self.sampler = SeedSampler(params, enc, arch, mode=mode, hp_rsq=hp_rsq, betas=betas)
        self.S, self.T = int(S), int(T)
        self.robot = robot or spec.make_bl_robot()
        self.grid, self.cost = grid, cost
        self.steps = steps
        # strict=True: planseed's contract -- seeds leaving the ESDF extent raise ValueError before
        # refinement (trajopt.optimize, trajopt.py:157-163).  Default False: at BASELINE config 3 every
        # seed of a random-init U-Net leaves the 1.28 m grid (the arm reaches ~1.6 m from its centre),
        # so the planner reports them per seed in `clamped` instead of raising (their lookups clamp to the
        # grid boundary, as planseed's sample_esdf_many does, geometry.py:223-240).
        self.strict = bool(strict)
        # guidance (plan_diffusion's guided branch, pipeline.py:189-197): strided DDIM over `steps`
        # with the BL-cost guide step against each problem's ESDF (SeedSampler.guided_sample)
        self.guidance = guidance
        if guidance is not None and guidance.alpha_guide != 0.0:
            if steps is None or list(steps) != list(spec.strided_steps(100, len(steps))):
                raise ValueError("guidance needs a strided DDIM schedule: steps = spec.strided_steps(K, n)")
        self.Pmax = int(max_problems)
        B = self.Pmax * self.S
        dev = "cuda"
        self.esdf = torch.empty((self.Pmax,) + tuple(grid.n), dtype=torch.float32, device=dev)
        # per-problem ESDFs in 4^3 bricks (PS_ESDF_CORDER=1: C order): each refinement lookup's 8
        # corners share one or two cache lines, so the 1024 ESDFs' working set fits L2 far better
        bricks_ok = all(v % 4 == 0 for v in grid.n) and n_boxes <= 32
        self.esdf_layout = bl.ESDF_BRICKED if bricks_ok and not os.environ.get("PS_ESDF_CORDER") else bl.ESDF_C_ORDER
        self.seeds = torch.empty((B, self.T, 7), dtype=torch.float32, device=dev)
        self.out = (torch.empty((B, self.T, 7), dtype=torch.float32, device=dev),
                    torch.empty(B, dtype=torch.float32, device=dev),
                    torch.empty(B, dtype=torch.uint8, device=dev),
                    torch.empty(B, dtype=torch.uint8, device=dev))
        self.best = torch.empty(self.Pmax, dtype=torch.int32, device=dev)
        self.film_a = torch.empty((self.Pmax, 3584), dtype=torch.float32, device=dev)
        self.cond = torch.empty((self.Pmax, spec.COND_DIM), dtype=torch.float32, device=dev)
        # device copies of host inputs for the end-to-end path
        self.d_images = torch.empty((self.Pmax, n_images) + tuple(image_shape), dtype=torch.float32,
                                    device=dev)
        self.d_q = torch.empty((self.Pmax, 7), dtype=torch.float32, device=dev)
        self.d_goal = torch.empty((self.Pmax, 7), dtype=torch.float32, device=dev)
        self.d_boxes = torch.empty((self.Pmax, n_boxes, 6), dtype=torch.float32, device=dev)
        self.timing = {}

    @classmethod
    def from_checkpoint(cls, path, **kw) -> "BLPlanner":
        """A planner over a unet1d PSCK checkpoint (checkpoint.py): weights, encoder depth and the
        noise schedule come from the file."""
        from .checkpoint import load_checkpoint
        params, enc, arch, betas, _ = load_checkpoint(path)
        return cls(params, enc, arch, betas=betas, **kw)

    # ------------------------------------------------------------------ device
    def plan_batch_device(self, images, q_start, goal, boxes, p0: int = 0, events=None, images_ready=None):
        """All inputs already on the device.  Returns PlanBatchResult of device tensors.
        `events` (optional dict of CUDA events) records "sample_start"/"sample_end" around the
        sampler and, when present, "refine_start"/"refine_end" around the refinement;
        `images_ready` (optional CUDA event, or a list of (event, p_begin, p_end) chunks) is waited on
        before the encoder -- chunk by chunk, so an image upload on another stream overlaps the ESDF
        build and the encoding of the chunks that already arrived."""
        torch = _lib.require_cuda()
        P = int(q_start.shape[0])
        if P > self.Pmax:
            raise ValueError("batch larger than max_problems")
        if P == 0:
            raise ValueError("need at least one problem")   # planseed: "need at least one seed"
        B = P * self.S
        esdf = self.esdf[:P]
        self._esdf_build(boxes, esdf)
        if isinstance(images_ready, (list, tuple)):
            cond = self.cond[:P]
            for ev, c0, c1 in images_ready:
                torch.cuda.current_stream().wait_event(ev)
                self.sampler.encode(images[c0:c1], q_start[c0:c1], goal[c0:c1], out=cond[c0:c1])
        else:
            if images_ready is not None:
                torch.cuda.current_stream().wait_event(images_ready)
            cond = self.sampler.encode(images, q_start, goal, out=self.cond[:P])
        fa = self.sampler.film(cond, out=self.film_a[:P])
        if events is not None:
            events["sample_start"].record()
        if self.guidance is not None and self.guidance.alpha_guide != 0.0:
            g = self.guidance
            seeds, _ = self.sampler.guided_sample(fa, q_start, self.S, esdf, self.robot, self.grid, self.cost, T=self.T,
                                                  p0=p0, n_steps=len(self.steps), k_guide_frac=g.k_guide_frac,
                                                  n_grad=g.n_grad, alpha_guide=g.alpha_guide,
                                                  esdf_layout=self.esdf_layout, strict=self.strict)
            self.seeds[:B].copy_(seeds)
            seeds = self.seeds[:B]
        else:
            seeds = self.sampler.sample(fa, q_start, self.S, self.T, p0=p0, steps=self.steps,
                                        out=self.seeds[:B])
        if events is not None:
            events["sample_end"].record()
        out = tuple(o[:B] for o in self.out)
        if events is not None and "refine_start" in events:
            events["refine_start"].record()
        if self.strict:
            bl.optimize(seeds, esdf, self.S, self.robot, self.grid, self.cost, out=out, esdf_layout=self.esdf_layout)
        else:
            bl.refine(seeds, esdf, self.S, self.robot, self.grid, self.cost, out=out,
                      esdf_layout=self.esdf_layout)
        if events is not None and "refine_end" in events:
            events["refine_end"].record()
        best = bl.select(out[1], out[2], self.S, out=self.best[:P])
        return PlanBatchResult(out[0], seeds, out[1], out[2], out[3], best)

    def _esdf_build(self, boxes, out):
        bl.esdf_build(boxes, self.grid, layout=self.esdf_layout, out=out)

    # ------------------------------------------------------------------ host
    def upload(self, images, q_start, goal, boxes, n_chunks: int = 4):
        """Host (ideally pinned) arrays -> this planner's device input buffers.  The small inputs go
        on the current stream; the images go on a side stream in `n_chunks` problem chunks, each with
        its completion event (self._img_chunks: [(event, p_begin, p_end)]), so the ESDF build and
        the encoding of arrived chunks overlap the rest of the upload.  Returns the device views."""
        torch = _lib.require_cuda()
        P = int(q_start.shape[0])
        if P > self.Pmax:
            raise ValueError("batch larger than max_problems")
        d_im, d_q, d_g, d_b = (self.d_images[:P], self.d_q[:P], self.d_goal[:P], self.d_boxes[:P])
        main = torch.cuda.current_stream()
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = torch.cuda.Stream()
            self._img_evs = []
        n_chunks = max(1, min(int(n_chunks), P))
        while len(self._img_evs) < n_chunks:
            self._img_evs.append(torch.cuda.Event())
        for dst, src in ((d_q, q_start), (d_g, goal), (d_b, boxes)):
            dst.copy_(torch.as_tensor(src), non_blocking=True)
        self._copy_stream.wait_stream(main)          # buffers free from the previous call
        h_im = torch.as_tensor(images)
        self._img_chunks = []
        with torch.cuda.stream(self._copy_stream):
            for i in range(n_chunks):
                c0, c1 = i * P // n_chunks, (i + 1) * P // n_chunks
                d_im[c0:c1].copy_(h_im[c0:c1], non_blocking=True)
                self._img_evs[i].record()
                self._img_chunks.append((self._img_evs[i], c0, c1))
        return d_im, d_q, d_g, d_b

    def plan_batch(self, images, q_start, goal, boxes, p0: int = 0, events=None):
        """End-to-end call from host (ideally pinned) arrays: H2D copies, the device
        pipeline, and a D2H read of trajectories, costs, flags and best indices."""
        torch = _lib.require_cuda()
        d = self.upload(images, q_start, goal, boxes)
        r = self.plan_batch_device(*d, p0=p0, images_ready=self._img_chunks, events=events)
        host = PlanBatchResult(r.trajectories.to("cpu", non_blocking=True), None,
                               r.cost.to("cpu", non_blocking=True),
                               r.feasible.to("cpu", non_blocking=True),
                               r.clamped.to("cpu", non_blocking=True),
                               r.best_index.to("cpu", non_blocking=True))
        torch.cuda.current_stream().synchronize()
        return host

    @staticmethod
    def result_bytes(P: int, S: int, T: int) -> int:
        B = P * S
        return B * T * 7 * 4 + B * 4 + B + B + P * 4
