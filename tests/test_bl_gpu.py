"""GPU parity tests of the BASELINE-profile refinement path, through the C-ABI.

The CUDA kernels follow the canonical fp32 operation order of oracle/c/bl_oracle.c,
so the bar here is BIT-EXACT equality (trajectories, costs, gradients, flags,
best-seed indices), not a tolerance.
"""

import numpy as np
import pytest

from paper_2410_16727_b200 import spec, synth

pytestmark = pytest.mark.gpu

RB = spec.make_bl_robot()
COST = spec.BLCost()


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test without a CUDA device")
    return torch


@pytest.fixture(scope="module")
def bl(torch_cuda):
    from paper_2410_16727_b200 import bl as _bl
    return _bl


def _esdf(bl, oracle_lib, grid, P, seed, n_boxes=20):
    rng = np.random.default_rng(seed)
    boxes = np.stack([synth.sample_boxes(rng, n_boxes, grid) for _ in range(P)]).astype(np.float32)
    dev = bl.esdf_build(boxes, grid)
    return boxes, dev


class TestEsdf:
    def test_bitwise_vs_oracle_full_grid(self, bl, oracle_lib):
        grid = spec.GridSpec()
        boxes, dev = _esdf(bl, oracle_lib, grid, 1, 0)
        ref = oracle_lib.esdf_build(boxes[0], grid)
        assert np.array_equal(dev[0].cpu().numpy(), ref)

    def test_bitwise_odd_grid_and_multi_problem(self, bl, oracle_lib):
        grid = spec.GridSpec(n=(17, 9, 13), h=0.05, origin=(0.1, -0.2, 0.05), cube=0.85)
        boxes, dev = _esdf(bl, oracle_lib, grid, 3, 1, n_boxes=5)
        for p in range(3):
            assert np.array_equal(dev[p].cpu().numpy(), oracle_lib.esdf_build(boxes[p], grid))

    def test_no_boxes_is_cap(self, bl):
        grid = spec.GridSpec(n=(8, 8, 8), h=0.1, cube=0.8)
        dev = bl.esdf_build(np.zeros((2, 0, 6), np.float32), grid)
        assert np.all(dev.cpu().numpy() == np.float32(grid.cap))


class TestCost:
    @pytest.mark.parametrize("T", [32, 64])
    def test_bitwise_vs_oracle(self, bl, oracle_lib, T):
        grid = spec.GridSpec()
        P, S = 2, 16
        _, dev = _esdf(bl, oracle_lib, grid, P, 2)
        q = synth.refine_init(P * S, t_len=T, seed=3)
        c, g, cl = bl.cost(q, dev, S, RB, grid, COST)
        ps = oracle_lib.BLProblemSet(RB, grid, COST, dev.cpu().numpy(), grid.n_nodes)
        rc, rg, rcl = oracle_lib.bl_cost(ps, q, S)
        assert np.array_equal(c.cpu().numpy(), rc)
        assert np.array_equal(g.cpu().numpy(), rg)
        assert np.array_equal(cl.cpu().numpy(), rcl)


class TestRefine:
    def _run(self, bl, oracle_lib, grid, P, S, T, n_iters, seed, n_boxes=20, q=None):
        _, dev = _esdf(bl, oracle_lib, grid, P, seed, n_boxes)
        if q is None:
            q = synth.refine_init(P * S, t_len=T, seed=seed + 1)
        out = bl.refine(q, dev, S, RB, grid, COST, n_iters=n_iters)
        ps = oracle_lib.BLProblemSet(RB, grid, COST, dev.cpu().numpy(), grid.n_nodes)
        ref = oracle_lib.bl_refine(ps, q, S, n_iters)
        return [o.cpu().numpy() for o in out], ref, q

    @pytest.mark.parametrize("T", [32, 64])
    def test_bitwise_vs_oracle(self, bl, oracle_lib, T):
        got, ref, q = self._run(bl, oracle_lib, spec.GridSpec(), 4, 32, T, 10, 10)
        assert np.array_equal(got[0], ref[0])
        assert np.array_equal(got[1], ref[1])
        assert np.array_equal(got[2].astype(bool), ref[2])
        assert np.array_equal(got[3].astype(bool), ref[3])
        assert np.array_equal(got[0][:, 0], q[:, 0])

    def test_flags_mixed_and_select_exact(self, bl, oracle_lib):
        # few small boxes -> a mix of feasible and colliding seeds
        got, ref, _ = self._run(bl, oracle_lib, spec.GridSpec(), 8, 32, 32, 10, 20, n_boxes=3)
        feas = ref[2]
        assert 0 < feas.sum() < feas.size
        best = bl.select(got[1], got[2], 32).cpu().numpy()
        assert np.array_equal(best, oracle_lib.select(ref[1], ref[2], 32))

    def test_config2_full_size_bitwise(self, bl, oracle_lib):
        # BASELINE config 2: 2048 trajectories, one shared 128^3 ESDF, 10 iterations
        grid = spec.GridSpec()
        _, dev = _esdf(bl, oracle_lib, grid, 1, 30)
        q = synth.refine_init(2048, seed=31)
        got = [o.cpu().numpy() for o in bl.refine(q, dev[0], 2048, RB, grid, COST)]
        ps = oracle_lib.BLProblemSet(RB, grid, COST, dev.cpu().numpy(), 0)
        ref = oracle_lib.bl_refine(ps, q, 2048, 10)
        assert np.array_equal(got[0], ref[0])
        assert np.array_equal(got[1], ref[1])
        assert np.array_equal(got[2].astype(bool), ref[2])

    def test_deterministic_and_split_invariant(self, bl, oracle_lib):
        grid = spec.GridSpec()
        _, dev = _esdf(bl, oracle_lib, grid, 4, 40)
        q = synth.refine_init(128, seed=41)
        a = [o.cpu().numpy() for o in bl.refine(q, dev, 32, RB, grid, COST)]
        b = [o.cpu().numpy() for o in bl.refine(q, dev, 32, RB, grid, COST)]
        lo = [o.cpu().numpy() for o in bl.refine(q[:64], dev[:2], 32, RB, grid, COST)]
        hi = [o.cpu().numpy() for o in bl.refine(q[64:], dev[2:], 32, RB, grid, COST)]
        for i in range(4):
            assert np.array_equal(a[i], b[i])
            assert np.array_equal(a[i], np.concatenate([lo[i], hi[i]]))

    def test_out_of_grid_flags(self, bl, oracle_lib):
        grid = spec.GridSpec(n=(32, 32, 32), h=0.01, origin=(0.48, 0.48, 0.48), cube=0.32)
        got, ref, _ = self._run(bl, oracle_lib, grid, 1, 32, 32, 3, 50, n_boxes=2)
        assert ref[3].all()                       # a 0.32 m box cannot hold the arm
        assert np.array_equal(got[3].astype(bool), ref[3])
        assert np.array_equal(got[0], ref[0])

    def test_empty_batch_and_bad_shapes(self, bl, torch_cuda):
        grid = spec.GridSpec(n=(8, 8, 8), h=0.1, cube=0.8)
        dev = bl.esdf_build(np.zeros((1, 1, 6), np.float32), grid)
        q = np.zeros((0, 32, 7), np.float32)
        out = bl.refine(q, dev, 4, RB, grid, COST)
        assert out[0].shape == (0, 32, 7)
        with pytest.raises(ValueError):
            bl.refine(np.zeros((4, 48, 7), np.float32), dev, 4, RB, grid, COST)


class TestReferenceSemantics:
    """evaluate_cost_batch / optimize raise planseed's ValueError naming the out-of-grid seeds
    (trajopt.py:116-118, :157-163); in-grid batches give refine()'s exact results."""

    def _setup(self, bl, n_grid=128, h=0.025):
        grid = spec.GridSpec(n=(n_grid,) * 3, h=h, cube=n_grid * h)
        import dataclasses
        robot = dataclasses.replace(RB, base=np.full(3, n_grid * h / 2))
        boxes = np.stack([synth.sample_boxes(np.random.default_rng(3), 6, grid)]).astype(np.float32)
        return grid, robot, bl.esdf_build(boxes, grid)

    def test_in_grid_optimize_equals_refine(self, bl):
        grid, robot, esdf = self._setup(bl)
        q = synth.refine_init(64, seed=4) * 0.3
        _, _, cl0 = bl.cost(q, esdf, 1, robot, grid, COST)
        q = q[~cl0.cpu().numpy()][:16]            # seeds that start inside the grid
        assert len(q) == 16
        a = [o.cpu().numpy() for o in bl.refine(q, esdf, 16, robot, grid, COST)]
        b = [o.cpu().numpy() for o in bl.optimize(q, esdf, 16, robot, grid, COST)]
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        c, g = bl.evaluate_cost_batch(q, esdf, 16, robot, grid, COST)
        c2, g2, _ = bl.cost(q, esdf, 16, robot, grid, COST)
        assert np.array_equal(c.cpu().numpy(), c2.cpu().numpy())

    def test_out_of_grid_raises_naming_seeds(self, bl):
        grid, robot, esdf = self._setup(bl)
        q = synth.refine_init(8, seed=4) * 0.3
        far = robot.__class__(**{**robot.__dict__, "base": np.full(3, 0.05)})   # arm leaves the grid
        _, _, cl = bl.cost(q, esdf, 8, far, grid, COST)
        want = np.nonzero(cl.cpu().numpy())[0].tolist()
        assert want
        with pytest.raises(ValueError, match=r"leave the ESDF extent \(seeds " + str(want).replace("[", r"\[").replace("]", r"\]")):
            bl.optimize(q, esdf, 8, far, grid, COST)
        with pytest.raises(ValueError, match="leave the ESDF extent"):
            bl.evaluate_cost_batch(q, esdf, 8, far, grid, COST)
        with pytest.raises(ValueError, match="n_iters"):
            bl.optimize(q, esdf, 8, robot, grid, COST, n_iters=0)
        with pytest.raises(ValueError, match="at least one seed"):
            bl.optimize(q[:0], esdf, 8, robot, grid, COST)

    def test_strict_planner_raises_at_config3(self, torch_cuda):
        from paper_2410_16727_b200.planner import BLPlanner
        params = spec.random_model(spec.ENCODER_CFG3)
        pb = synth.config3_problems(1, p0=0, seed=0)
        pl = BLPlanner(params, spec.ENCODER_CFG3, mode=1, S=8, max_problems=1, strict=True)
        with pytest.raises(ValueError, match="leave the ESDF extent"):
            pl.plan_batch(pb.images, pb.q_start, pb.goal, pb.boxes)
        pbw, grid, robot = synth.config3_wide(1, p0=0)
        pw = BLPlanner(params, spec.ENCODER_CFG3, mode=1, S=8, max_problems=1, strict=True, grid=grid, robot=robot)
        r = pw.plan_batch(pbw.images, pbw.q_start, pbw.goal, pbw.boxes)
        assert not np.asarray(r.clamped).any()


class TestMetrics:
    """bl.metrics (ps_bl_metrics, fp32) against the float64 oracle's trajopt.metrics restatement
    (oracle/bl_numpy.bl_metrics, pinned to planseed in test_bl_oracle.TestMetricsOracle).
    Bounds: clearance / translation error within 2e-5 m, angle within 1e-2 deg, motion time and
    max jerk within 1e-4 relative; flags equal wherever the value is not within that bound of
    its threshold."""

    def _case(self, P=6, S=8, seed=0):
        from oracle import bl_numpy as bn
        pb, grid, robot = synth.config3_wide(P, p0=seed)
        q = synth.refine_init(P * S, seed=seed + 1) * 0.35
        # half the problems get their goal at the end pose of a collision-free seed (success then
        # decided by the thresholds), the rest a random goal
        goal = pb.goal.astype(np.float64).copy()
        for p in range(0, P, 2):
            clr = [bn.traj_min_clearance(robot, pb.boxes[p], q[p * S + s].astype(np.float64), grid.cap)
                   for s in range(S)]
            s_free = int(np.argmax(clr))
            F = bn.dh_frames(robot, q[p * S + s_free, -1].astype(np.float64))[-1]
            R = F[:3, :3]
            w = np.sqrt(max(1e-12, 1 + np.trace(R))) / 2
            goal[p] = np.concatenate([F[:3, 3] - robot.base, [w, (R[2, 1] - R[1, 2]) / (4 * w),
                                      (R[0, 2] - R[2, 0]) / (4 * w), (R[1, 0] - R[0, 1]) / (4 * w)]])
        return pb.boxes, goal.astype(np.float32), q, robot, grid

    @pytest.mark.parametrize("T", [32, 64])
    def test_vs_oracle(self, bl, T):
        from oracle import bl_numpy as bn
        S = 8
        boxes, goal, q, robot, grid = self._case(S=S)
        if T == 64:
            q = np.repeat(q, 2, axis=1)
        m = bl.metrics(q, boxes, goal, S, robot, cap=grid.cap)
        got = {k: getattr(m, k).cpu().numpy() for k in ("clearance", "translation_error", "angle_error_deg",
                                                         "motion_time", "max_jerk", "success", "collision_free")}
        n_succ = 0
        for b in range(len(q)):
            r = bn.bl_metrics(robot, boxes[b // S], goal[b // S].astype(np.float64), q[b].astype(np.float64),
                              grid.cap)
            assert abs(got["clearance"][b] - r["clearance"]) < 2e-5
            assert abs(got["translation_error"][b] - r["translation_error"]) < 2e-5
            assert abs(got["angle_error_deg"][b] - r["angle_error_deg"]) < 1e-2
            assert got["motion_time"][b] == pytest.approx(r["motion_time"], rel=1e-4)
            assert got["max_jerk"][b] == pytest.approx(r["max_jerk"], rel=1e-4)
            if abs(r["clearance"]) > 2e-5:
                assert bool(got["collision_free"][b]) == r["collision_free"]
                if (abs(r["translation_error"] - spec.DELTA_T) > 2e-5 and abs(r["angle_error_deg"] - spec.DELTA_R_DEG) > 1e-2):
                    assert bool(got["success"][b]) == r["success"]
            n_succ += r["success"]
        assert 0 < n_succ < len(q)                     # both outcomes exercised
        assert 0 < got["collision_free"].mean() < 1


class TestSelect:
    def test_matches_oracle_with_ties(self, bl, oracle_lib):
        rng = np.random.default_rng(7)
        for S in (1, 8, 32, 100):
            P = 37
            c = rng.integers(0, 4, size=P * S).astype(np.float32)
            f = rng.random(P * S) < 0.15
            got = bl.select(c, f.astype(np.uint8), S).cpu().numpy()
            assert np.array_equal(got, oracle_lib.select(c, f, S))


class TestBrickedEsdf:
    """The planner's 4^3-brick ESDF layout: same values (unbrick == C order, bitwise) and the
    refinement over it is bit-identical to the refinement over the C-order grid."""

    def test_unbrick_equals_c_order(self, bl):
        grid = spec.GridSpec()
        rng = np.random.default_rng(5)
        boxes = np.stack([synth.sample_boxes(rng, 20, grid) for _ in range(3)]).astype(np.float32)
        c = bl.esdf_build(boxes, grid)
        b = bl.esdf_build(boxes, grid, layout=bl.ESDF_BRICKED)
        assert np.array_equal(bl.unbrick(b, grid).cpu().numpy(), c.cpu().numpy())

    def test_refine_identical_on_bricks(self, bl, torch_cuda):
        grid = spec.GridSpec()
        P, S = 6, 32
        rng = np.random.default_rng(6)
        boxes = np.stack([synth.sample_boxes(rng, 20, grid) for _ in range(P)]).astype(np.float32)
        c = bl.esdf_build(boxes, grid)
        b = bl.esdf_build(boxes, grid, layout=bl.ESDF_BRICKED)
        q = synth.refine_init(P * S, seed=11)
        r0 = [o.cpu().numpy() for o in bl.refine(q, c, S, RB, grid, COST)]
        r1 = [o.cpu().numpy() for o in bl.refine(q, b, S, RB, grid, COST, esdf_layout=bl.ESDF_BRICKED)]
        for u, v in zip(r0, r1):
            assert np.array_equal(u, v)
        assert np.unique(r0[1]).size > P * S // 2   # non-trivial costs


def test_depth_images_rendered_on_device_bitwise(torch_cuda):
    """ps_render_depth_rects rasterises synth.image_params to the host generator's bits."""
    pb = synth.config3_problems(5, p0=17)
    prm = synth.image_params(5, p0=17)
    got = synth.render_images_device(prm, (240, 320)).cpu().numpy()
    assert np.array_equal(got, pb.images)
    p0 = synth.config0_problems(2, p0=3)
    got0 = synth.render_images_device(synth.image_params(2, p0=3, image_shape=(128, 128), n_images=1, n_rect=5),
                                      (128, 128)).cpu().numpy()
    assert np.array_equal(got0, p0.images)


@pytest.mark.parametrize("shared", [True, False])
def test_quad_brick_layout_bitwise(bl, oracle_lib, shared):
    """Layout 2 (quad bricks, two 16-B loads per lookup) gives the C-order results bit for bit:
    refinement, cost/gradient and flags, for a shared ESDF (config 2) and per-problem ESDFs."""
    grid = spec.GridSpec()
    P, S = (1, 64) if shared else (3, 16)
    boxes = np.stack([synth.sample_boxes(np.random.default_rng(9 + i), 20, grid) for i in range(P)]).astype(np.float32)
    c_order = bl.esdf_build(boxes, grid)
    quad = bl.esdf_build(boxes, grid, layout=bl.ESDF_QUAD)
    assert quad.shape == (P, 128, 128, 128, 4)
    e0, e2 = (c_order[0], quad[0]) if shared else (c_order, quad)
    q = synth.refine_init(P * S if not shared else S, seed=12)
    a = [o.cpu().numpy() for o in bl.refine(q, e0, S, RB, grid, COST)]
    b = [o.cpu().numpy() for o in bl.refine(q, e2, S, RB, grid, COST, esdf_layout=bl.ESDF_QUAD)]
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    ca = [o.cpu().numpy() for o in bl.cost(q, e0, S, RB, grid, COST)]
    cb = [o.cpu().numpy() for o in bl.cost(q, e2, S, RB, grid, COST, esdf_layout=bl.ESDF_QUAD)]
    for x, y in zip(ca, cb):
        assert np.array_equal(x, y)
