"""CPU tests of the BASELINE-profile refinement oracle (no GPU).

Pins the canonical-fp32 C oracle against the independent float64 numpy oracle, the
numpy oracle against finite differences and known answers, and both against the
reference package itself in the planar degenerate configuration (bridge tests,
SURVEY.md §7.3 step 1).
"""

import math

import numpy as np
import pytest

from oracle import bl_numpy as bn
from paper_2410_16727_b200 import spec, synth

RB = spec.make_bl_robot()
COST = spec.BLCost()


def small_grid(n=48, h=0.0275):
    return spec.GridSpec(n=(n, n, n), h=h, cube=h * n)


class TestPhilox:
    # Random123 known-answer vectors for Philox4x32-10
    KAT = [
        ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
        ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
        ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
         [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
    ]

    @pytest.mark.parametrize("ctr,key,want", KAT)
    def test_known_answers(self, oracle_lib, ctr, key, want):
        assert list(oracle_lib.philox(ctr, key)) == want


class TestSpec:
    def test_unet_size_matches_survey(self):
        a = spec.UNetArch()
        assert a.n_params() == 5386119                     # ~5.39 M
        assert a.flops_per_traj_step(32) == 72814592        # 72.8 MFLOP
        assert a.flops_per_traj_step(64) == 2 * 72814592
        assert a.film_flops() == 2852864                    # 2.85 MFLOP per (problem, step)

    def test_sphere_table_sorted(self):
        assert np.all(np.diff(RB.sphere_link) >= 0)
        assert RB.n_spheres == 50
        assert np.all((RB.sphere_radius >= 0.03) & (RB.sphere_radius <= 0.08))
        assert np.all((RB.a >= 0.1) & (RB.a <= 0.35))

    def test_cosine_schedule(self):
        b = spec.cosine_betas()
        assert b.shape == (100,) and np.all(b > 0) and b[-1] == pytest.approx(0.999)
        ab = np.cumprod(1 - b)
        assert np.all(np.diff(ab) < 0)

    def test_strided_steps_round_half_even(self):
        # planseed/diffusion.py:520-526; (100,5) -> 50 not 51
        assert list(spec.strided_steps(100, 5)) == [100, 75, 50, 26, 1]
        s10 = spec.strided_steps(100, 10)
        assert s10[0] == 100 and s10[-1] == 1 and len(s10) == 10


class TestStencils:
    def test_jerk_operator_matches_numpy_gradient(self):
        # planseed tests/test_trajopt.py:267-271
        rng = np.random.default_rng(42)
        q = rng.standard_normal((32, 7))
        D = bn.diff_matrix(32)
        want = np.gradient(np.gradient(np.gradient(q, axis=0), axis=0), axis=0)
        np.testing.assert_allclose(D @ D @ D @ q, want, atol=1e-12)


class TestEsdf:
    def test_known_answers(self):
        g = spec.GridSpec(n=(5, 5, 5), h=0.25, cube=1.0)
        box = np.array([[0.25, 0.25, 0.25, 0.75, 0.75, 0.75]])
        v = bn.esdf_boxes(box, g)
        assert v[2, 2, 2] == pytest.approx(-0.25)          # centre: inside by 0.25
        assert v[0, 2, 2] == pytest.approx(0.25)           # face distance
        assert v[0, 0, 0] == pytest.approx(0.25 * math.sqrt(3))

    def test_empty_world_is_cap(self, oracle_lib):
        g = small_grid(8, 0.1)
        v = oracle_lib.esdf_build(np.zeros((0, 6)), g)
        assert np.all(v == np.float32(g.cap))

    def test_c_matches_numpy(self, oracle_lib):
        g = small_grid()
        boxes = synth.sample_boxes(np.random.default_rng(3), 20, g)
        c = oracle_lib.esdf_build(boxes, g)
        n = bn.esdf_boxes(boxes.astype(np.float32).astype(np.float64), g)
        assert np.abs(c - n).max() < 2e-6


def _problem_set(oracle_lib, grid, n_prob=2, seed=0, n_boxes=20):
    rng = np.random.default_rng(seed)
    esdf = np.stack([oracle_lib.esdf_build(synth.sample_boxes(rng, n_boxes, grid), grid)
                     for _ in range(n_prob)])
    return oracle_lib.BLProblemSet(RB, grid, COST, esdf, grid.n_nodes), esdf


class TestCostGradient:
    def test_c_fp32_matches_numpy_fp64(self, oracle_lib):
        grid = spec.GridSpec()
        ps, esdf = _problem_set(oracle_lib, grid, 2)
        q = synth.refine_init(8, seed=1)
        c32, g32, cl32 = oracle_lib.bl_cost(ps, q, 4)
        vals = lambda p: esdf[p].astype(np.float64)
        c64, g64, cl64 = bn.bl_cost(RB, vals, grid.origin, grid.h, COST, q, 4)
        np.testing.assert_allclose(c32, c64, rtol=2e-5)
        assert np.abs(g32 - g64).max() <= 1e-5 * max(1.0, np.abs(g64).max())
        assert np.array_equal(cl32, cl64)
        assert np.all(g32[:, 0] == 0)

    def test_numpy_gradient_matches_finite_differences(self):
        # affine ESDF => trilinear interpolant is globally C^1 and central differences
        # are exact up to rounding (planseed tests/test_trajopt.py:25-34, :113-152)
        g = spec.GridSpec(n=(130, 130, 130), h=0.02, origin=(-0.66, -0.66, -0.66), cube=2.6)
        ax = [g.origin[a] + g.h * np.arange(g.n[a]) for a in range(3)]
        X, Y, Z = np.meshgrid(*ax, indexing="ij")
        vals = 0.4 + 0.25 * X - 0.4 * Y + 0.3 * Z
        cost = spec.BLCost(w_coll=5.0, margin=2.0)         # every sphere active
        q = synth.refine_init(1, seed=5)[0].astype(np.float64) * 0.6
        f = lambda x: bn.bl_cost(RB, lambda p: vals, g.origin, g.h, cost, x[None], 1)[0][0]
        _, grad, cl = bn.bl_cost(RB, lambda p: vals, g.origin, g.h, cost, q[None], 1)
        assert not cl[0]
        fd = np.zeros_like(q)
        eps = 1e-6
        for t in range(1, q.shape[0]):
            for k in range(7):
                dp, dm = q.copy(), q.copy()
                dp[t, k] += eps
                dm[t, k] -= eps
                fd[t, k] = (f(dp) - f(dm)) / (2 * eps)
        assert np.linalg.norm(grad[0] - fd) / np.linalg.norm(fd) < 1e-6


class TestRefine:
    def test_c_matches_numpy_within_tolerance(self, oracle_lib):
        grid = spec.GridSpec()
        ps, esdf = _problem_set(oracle_lib, grid, 2, seed=4)
        q = synth.refine_init(16, seed=2)
        x32, c32, f32, _ = oracle_lib.bl_refine(ps, q, 8, 10)
        vals = lambda p: esdf[p].astype(np.float64)
        x64, c64, f64, mc = bn.bl_refine(RB, vals, grid.origin, grid.h, COST, q, 8, 10)
        # The trilinear interpolant is only C^0 across cell faces: when an fp32 and an
        # fp64 iterate land on opposite sides of a face the in-cell gradient jumps and
        # the two runs part.  That is why the device parity
        # anchor is the bit-exact canonical-fp32 C oracle; against fp64 we require the
        # north-star 1e-4 rad bound on the large majority of trajectories.
        err = np.abs(x32 - x64).max(axis=(1, 2))
        assert np.mean(err < 1e-4) >= 0.85
        assert err.max() < 5e-2
        ok = err < 1e-4
        np.testing.assert_allclose(c32[ok], c64[ok], rtol=1e-4)
        decided = ok & (np.abs(mc) > 1e-4)
        assert np.array_equal(f32[decided], f64[decided])
        assert np.array_equal(x32[:, 0], q[:, 0])         # row 0 pinned

    def test_zero_iterations_is_identity(self, oracle_lib):
        ps, _ = _problem_set(oracle_lib, small_grid(), 1)
        q = synth.refine_init(4, seed=3)
        x, _, _, _ = oracle_lib.bl_refine(ps, q, 4, 0)
        assert np.array_equal(x, q)

    def test_identical_seeds_identical_results(self, oracle_lib):
        ps, _ = _problem_set(oracle_lib, small_grid(), 1)
        q = np.repeat(synth.refine_init(1, seed=6), 6, axis=0)
        x, c, f, _ = oracle_lib.bl_refine(ps, q, 6, 10)
        assert all(np.array_equal(x[0], x[i]) for i in range(6))
        assert np.all(c == c[0])


class TestSelect:
    # planseed tests/test_pipeline.py:91-106 semantics
    def test_single(self, oracle_lib):
        assert oracle_lib.select(np.array([3.0]), np.array([False]), 1)[0] == 0

    def test_prefers_success(self, oracle_lib):
        assert oracle_lib.select(np.array([1.0, 5.0]), np.array([False, True]), 2)[0] == 1

    def test_tie_breaks_to_lower_index(self, oracle_lib):
        assert oracle_lib.select(np.array([2.0, 1.0, 1.0]), np.array([False] * 3), 3)[0] == 1

    def test_lowest_cost_among_successes(self, oracle_lib):
        c = np.array([0.5, 3.0, 2.0, 9.0])
        f = np.array([False, True, True, True])
        assert oracle_lib.select(c, f, 4)[0] == 2

    def test_c_matches_numpy_random(self, oracle_lib):
        rng = np.random.default_rng(9)
        c = rng.integers(0, 5, size=64 * 8).astype(np.float32)   # many ties
        f = rng.random(64 * 8) < 0.2
        assert np.array_equal(oracle_lib.select(c, f, 8), bn.select_best(c, f, 8))


@pytest.mark.reference
class TestBridgeToPlanseed:
    """Planar degenerate BL configuration == planseed's own cost kernel.

    DH with alpha = d = 0 and a_k = link length is the cumulative-angle planar chain;
    zero-radius spheres at the midpoint-rule fractions are planseed's collision points;
    an ESDF extruded along z makes trilinear == bilinear; margin = d_act, w_coll =
    w_world, (w_vel, w_acc, w_jerk) = (0, 0, w_smooth) give planseed's world + jerk
    terms (planseed/_kernels.py:165-312)."""

    def _setup(self, planseed):
        from planseed.arm import default_arm
        from planseed.geometry import Box, Circle, World, build_esdf
        arm = default_arm()
        world = World([Circle(center=(0.35, 0.1), radius=0.12), Box(lo=(-0.5, 0.3), hi=(-0.1, 0.6))])
        esdf2 = build_esdf(world, 0.01)
        m = arm.points_per_link
        fr = arm.point_fractions()
        link = np.repeat(np.arange(7), m)
        off = np.zeros((7 * m, 3))
        off[:, 0] = -(1.0 - np.tile(fr, 7)) * arm.lengths[link]
        robot = spec.DHRobot(a=arm.lengths.copy(), d=np.zeros(7), alpha=np.zeros(7),
                             base=np.array([0.0, 0.0, 0.005]), lo=arm.lo, hi=arm.hi,
                             sphere_link=link.astype(np.int32), sphere_offset=off,
                             sphere_radius=np.zeros(7 * m))
        vals3 = np.repeat(esdf2.values[:, :, None], 2, axis=2)
        grid = spec.GridSpec(n=(esdf2.nx, esdf2.ny, 2), h=esdf2.h,
                             origin=(esdf2.origin[0], esdf2.origin[1], 0.0), cube=2.0)
        return arm, world, esdf2, robot, vals3, grid

    def test_world_and_jerk_terms_match_planseed(self, planseed):
        from planseed.arm import Pose2
        from planseed.trajopt import CostWeights, evaluate_cost_batch
        arm, world, esdf2, robot, vals3, grid = self._setup(planseed)
        w_ref = CostWeights(w_goal_pos=0, w_goal_rot=0, w_self=0, w_smooth=1.0, w_world=50.0,
                            d_act=0.2)
        w_bl = spec.BLCost(w_coll=50.0, w_vel=0.0, w_acc=0.0, w_jerk=1.0, margin=0.2)
        rng = np.random.default_rng(2)
        q0 = rng.uniform(-1.2, 1.2, size=7)
        q1 = rng.uniform(-1.2, 1.2, size=7)
        trajs = q0 + np.linspace(0, 1, 32)[None, :, None] * (q1 - q0)
        trajs = trajs + 0.08 * rng.standard_normal((6, 32, 7))
        trajs[:, 0] = q0
        tot, grad, _ = evaluate_cost_batch(arm, esdf2, Pose2((0.3, 0.2), 0.5), trajs, w_ref)
        c64, g64, cl = bn.bl_cost(robot, lambda p: vals3, grid.origin, grid.h, w_bl, trajs, 6)
        assert not cl.any()
        np.testing.assert_allclose(c64, tot, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(g64, grad, rtol=1e-9, atol=1e-9)


class TestMetricsOracle:
    """oracle.bl_numpy ground-truth evaluation pinned to planseed's own retime / metrics /
    traj_min_clearance (trajopt.py:209-272, _kernels.py:144-162)."""

    def test_retime_matches_planseed(self, planseed):
        from planseed.arm import default_arm
        from planseed.trajopt import jerk_matrix, retime
        arm = default_arm()
        rng = np.random.default_rng(5)
        for T in (32, 64):
            traj = np.cumsum(rng.standard_normal((T, 7)) * 0.05, axis=0)
            mt_ref, _ = retime(arm, traj)
            dt = mt_ref / (T - 1)
            mj_ref = float(np.max(np.abs(jerk_matrix(T) @ traj)) / dt ** 3)
            mt, mj = bn.retime(traj, arm.vel_limit[0], arm.acc_limit[0], arm.jerk_limit[0])
            assert mt == pytest.approx(mt_ref, rel=1e-12) and mj == pytest.approx(mj_ref, rel=1e-9)
        assert bn.retime(np.zeros((32, 7)))[0] == 0.0
        assert (spec.VEL_LIMIT, spec.ACC_LIMIT, spec.JERK_LIMIT) == (arm.vel_limit[0], arm.acc_limit[0],
                                                                     arm.jerk_limit[0])

    def test_clearance_matches_planseed_in_the_planar_degenerate_case(self, planseed):
        # zero-radius spheres at planseed's collision points, boxes extruded along z: the 3-D
        # clearance equals planseed's traj_min_clearance over the same boxes
        from planseed import _kernels as K
        from planseed.arm import default_arm
        from planseed.geometry import Box, World
        arm = default_arm()
        world = World([Box(lo=(-0.5, 0.3), hi=(-0.1, 0.6)), Box(lo=(0.2, -0.7), hi=(0.6, -0.3))])
        m = arm.points_per_link
        fr = arm.point_fractions()
        link = np.repeat(np.arange(7), m)
        off = np.zeros((7 * m, 3))
        off[:, 0] = -(1.0 - np.tile(fr, 7)) * arm.lengths[link]
        robot = spec.DHRobot(a=arm.lengths.copy(), d=np.zeros(7), alpha=np.zeros(7),
                             base=np.array([arm.base[0], arm.base[1], 0.0]), lo=arm.lo, hi=arm.hi,
                             sphere_link=link.astype(np.int32), sphere_offset=off, sphere_radius=np.zeros(7 * m))
        boxes3 = np.array([[b[0], b[1], -50.0, b[2], b[3], 50.0] for b in world.box_arr])
        rng = np.random.default_rng(8)
        for _ in range(5):
            traj = np.cumsum(rng.standard_normal((32, 7)) * 0.1, axis=0)
            want = K.traj_min_clearance(traj, 4, arm.lengths, float(arm.base[0]), float(arm.base[1]),
                                        arm.point_fractions(), np.zeros((0, 3)), world.box_arr, world.sdf_cap)
            got = bn.traj_min_clearance(robot, boxes3, traj, world.sdf_cap, 4)
            assert got == pytest.approx(want, rel=1e-12, abs=1e-12)

    def test_end_pose_errors_zero_at_own_pose(self):
        rng = np.random.default_rng(3)
        q = rng.uniform(-2, 2, 7)
        F = bn.dh_frames(RB, q)[-1]
        R = F[:3, :3]
        w = np.sqrt(max(1e-12, 1 + np.trace(R))) / 2
        quat = np.array([w, (R[2, 1] - R[1, 2]) / (4 * w), (R[0, 2] - R[2, 0]) / (4 * w), (R[1, 0] - R[0, 1]) / (4 * w)])
        goal = np.concatenate([F[:3, 3] - RB.base, quat])
        terr, aerr = bn.end_pose_errors(RB, q, goal)
        assert terr < 1e-12 and aerr < 1e-6
        # a 10 degree turn about the goal z axis reads as 10 degrees
        c, s = np.cos(np.radians(5)), np.sin(np.radians(5))
        qz = np.array([c, 0, 0, s])
        def qmul(a, b):
            return np.array([a[0] * b[0] - a[1:] @ b[1:], *(a[0] * b[1:] + b[0] * a[1:] + np.cross(a[1:], b[1:]))])
        g2 = np.concatenate([goal[:3], qmul(quat, qz)])
        assert bn.end_pose_errors(RB, q, g2)[1] == pytest.approx(10.0, abs=1e-6)


class TestGuideOracle:
    def test_c_guide_is_planseeds_guide_loop(self, oracle_lib):
        """orc_bl_guide == planseed's guide() (diffusion.py:598-617) written over the BL cost in
        float32 numpy (cost_fn = the canonical C cost), bit for bit."""
        grid = small_grid()
        boxes = np.stack([synth.sample_boxes(np.random.default_rng(4), 8, grid)]).astype(np.float32)
        esdf = oracle_lib.esdf_build(boxes[0], grid)
        ps = oracle_lib.BLProblemSet(RB, grid, COST, esdf[None], grid.n_nodes)
        import dataclasses
        robot = dataclasses.replace(RB, base=np.full(3, grid.cube / 2))
        ps = oracle_lib.BLProblemSet(robot, grid, COST, esdf[None], grid.n_nodes)
        rng = np.random.default_rng(6)
        x0 = rng.uniform(0.3, 0.7, (6, 32, 7)).astype(np.float32)
        lo = np.full(7, -spec.JOINT_LIMIT, np.float32)
        span = np.full(7, 2 * spec.JOINT_LIMIT, np.float32)
        n_grad, alpha, max_halvings = 5, np.float32(1.0), 8

        def cost_fn(trajs):
            c, g, _ = oracle_lib.bl_cost(ps, trajs, len(trajs))
            return c, g

        x = x0.copy()
        for _ in range(n_grad):                      # planseed's loop, float32 throughout
            costs, grads = cost_fn(lo + x * span)
            g_norm = grads * span
            step = np.full(x.shape[0], alpha, np.float32)
            remaining = np.ones(x.shape[0], dtype=bool)
            for _ in range(max_halvings):
                if not remaining.any():
                    break
                cand = x - step[:, None, None] * g_norm
                new_costs, _ = cost_fn(lo + cand * span)
                improved = remaining & (new_costs < costs)
                x = np.where(improved[:, None, None], cand, x)
                remaining = remaining & ~improved
                step = np.where(remaining, step * np.float32(0.5), step)
        got, cl = oracle_lib.bl_guide(ps, x0, 6, lo, span, n_grad, float(alpha), max_halvings)
        assert np.array_equal(got, x)
        assert not np.array_equal(got, x0)           # guidance moved the seeds


def test_image_params_reproduce_the_generator():
    pb = synth.config3_problems(2, p0=9)
    prm = synth.image_params(2, p0=9)
    img = np.stack([[synth.render_depth_params(prm[i, m], 240, 320) for m in range(2)] for i in range(2)])
    assert np.array_equal(img.astype(np.float32), pb.images)
