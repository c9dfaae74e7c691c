"""Generate golden input/output fixtures from the reference package (planseed, imported
from /root/reference/pkg/src in the build container) for the ref-profile parity tests.

    PYTHONPATH=/root/reference/pkg/src python tools/make_golden.py

Writes tests/golden/ref_*.npz.  The GPU box has no /root/reference, so the tests there
compare the CUDA drop-in against these files; tests/test_golden_cpu.py re-runs this
generator in the container and checks the committed files are what planseed produces.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")
if str(REF) not in sys.path:
    sys.path.insert(0, str(REF))

from planseed import _kernels  # noqa: E402
from planseed.arm import Pose2, default_arm, fk_pose  # noqa: E402
from planseed.diffusion import (arch_for_arm, create_net, ddim_sample, encode_condition,  # noqa: E402
                                make_schedule, predict_noise)
from planseed.geometry import (Box, Circle, SdfGrid, SensorPose, World, build_esdf,  # noqa: E402
                               render_depth_scan)
from planseed.pipeline import PlanRequest, build_planner_esdf, plan_diffusion, planner_success  # noqa: E402
from planseed.trajopt import (CostWeights, _kernel_args, evaluate_cost_batch, linear_seed,  # noqa: E402
                              optimize)

ARM = default_arm()
T = 32


def linear_grid(a=1.0, bx=0.25, by=-0.4):
    h, n = 0.01, 201
    xs = -1.0 + h * np.arange(n)
    gx, gy = np.meshgrid(xs, xs, indexing="ij")
    return SdfGrid(origin=np.array([-1.0, -1.0]), h=h, nx=n, ny=n, values=a + bx * gx + by * gy)


def random_trajs(rng, n, scale=0.8):
    out = []
    for _ in range(n):
        q0 = rng.uniform(-1.2, 1.2, size=7)
        q1 = rng.uniform(-1.2, 1.2, size=7)
        tr = q0 + np.linspace(0, 1, T)[:, None] * (q1 - q0)
        tr += scale * 0.1 * rng.standard_normal((T, 7))
        tr[0] = q0
        out.append(tr)
    return np.stack(out)


def esdf_dict(e, prefix="esdf"):
    return {f"{prefix}_values": e.values, f"{prefix}_origin": np.asarray(e.origin), f"{prefix}_h": np.float64(e.h)}


def w_arr(w):
    return np.array([w.w_goal_pos, w.w_goal_rot, w.w_smooth, w.w_self, w.w_world, w.d_act, w.d_self])


def gen_cost():
    cases = {}
    world = World([Circle(center=(0.45, 0.15), radius=0.2), Box(lo=(-0.6, -0.7), hi=(-0.2, -0.35))])
    grids = {"real": build_esdf(world, 0.01), "linear": linear_grid()}
    ws = {"default": CostWeights(), "all": CostWeights(d_act=0.15, d_self=0.4),
          "world": CostWeights(w_goal_pos=0, w_goal_rot=0, w_smooth=0, w_self=0, d_act=1.5)}
    rng = np.random.default_rng(16)
    goal = Pose2(position=(0.3, 0.25), theta=0.7)
    i = 0
    for gname, g in grids.items():
        for wname, w in ws.items():
            trajs = random_trajs(rng, 6)
            terms, totals, grads, clamped = _kernels.cost_terms_batch(trajs, *_kernel_args(ARM, g, goal, w, T), True)
            cases[f"c{i}"] = dict(trajs=trajs, goal=np.array([*goal.pos, goal.theta]), w=w_arr(w),
                                  terms=terms, totals=totals, grads=grads, clamped=clamped,
                                  grid=gname, **esdf_dict(g))
            i += 1
    # out-of-extent points: clamped flags set, values from the clamped edge patch
    tiny = SdfGrid(origin=np.array([-0.1, -0.1]), h=0.05, nx=5, ny=5,
                   values=np.random.default_rng(3).uniform(0.0, 0.2, (5, 5)))
    trajs = random_trajs(rng, 4)
    w = CostWeights(d_act=0.3)
    terms, totals, grads, clamped = _kernels.cost_terms_batch(trajs, *_kernel_args(ARM, tiny, goal, w, T), True)
    cases["c6"] = dict(trajs=trajs, goal=np.array([*goal.pos, goal.theta]), w=w_arr(w), terms=terms,
                       totals=totals, grads=grads, clamped=clamped, grid="tiny", **esdf_dict(tiny))
    return cases


def gen_optimize():
    esdf = build_esdf(World([Circle(center=(0.4, 0.3), radius=0.15)]), 0.01)
    rng = np.random.default_rng(20)
    q0 = np.array([0.4, -0.3, 0.5, -0.2, 0.3, 0.1, -0.2])
    goal = Pose2(position=(0.1, 0.55), theta=1.2)
    seeds = np.stack([linear_seed(ARM, q0, goal, rng) for _ in range(6)])
    w = CostWeights()
    x, terms, totals, frozen, nacc = _kernels.optimize_batch(
        seeds.copy(), 40, 0.9, 1e-4, 0.5, 40, 1.0, 4.0, *_kernel_args(ARM, esdf, goal, w, T))
    # second case: an already optimal seed (constant at a pose whose FK is the goal, empty
    # world) freezes; mixed with linear seeds that do not
    esdf0 = build_esdf(World([]), 0.01)
    goal0 = fk_pose(ARM, q0)
    seeds0 = np.stack([np.tile(q0, (T, 1))] + [linear_seed(ARM, q0, goal0, rng) for _ in range(3)])
    x0, terms0, totals0, frozen0, nacc0 = _kernels.optimize_batch(
        seeds0.copy(), 25, 0.9, 1e-4, 0.5, 40, 1.0, 4.0, *_kernel_args(ARM, esdf0, goal0, w, T))
    return dict(seeds=seeds, goal=np.array([*goal.pos, goal.theta]), w=w_arr(w), n_iters=np.int64(40), x=x,
                terms=terms, totals=totals, frozen=frozen, n_acc=nacc, **esdf_dict(esdf),
                b_seeds=seeds0, b_goal=np.array([*goal0.pos, goal0.theta]), b_x=x0, b_totals=totals0,
                b_frozen=frozen0, b_n_acc=nacc0, **esdf_dict(esdf0, "b_esdf"))


def scene():
    world = World([Circle(center=(0.35, 0.2), radius=0.12), Box(lo=(0.55, -0.35), hi=(0.7, 0.1)),
                   Circle(center=(-0.3, 0.45), radius=0.1)])
    pose = SensorPose(position=(-0.6, 0.2), heading=-0.15)
    return world, render_depth_scan(world, pose)


def net_and_cond():
    cfg = arch_for_arm(ARM)
    net = create_net(cfg, seed=3)
    rng = np.random.default_rng(5)
    for name, p in net.params.items():           # exercise every path (FiLM, biases)
        p.data[:] = p.data + 0.02 * rng.standard_normal(p.data.shape)
    return net


def gen_sampler():
    net = net_and_cond()
    world, scan = scene()
    q0 = np.array([0.3, -0.5, 0.6, -0.4, 0.2, 0.3, -0.1])
    goal = Pose2(position=(0.45, 0.5), theta=0.9)
    cond = encode_condition(net, scan, q0, goal)
    rng = np.random.default_rng(9)
    x = rng.standard_normal((5, T, 7))
    eps = predict_noise(net, x, 37, cond)
    sched = make_schedule()
    x_K = rng.standard_normal((6, T, 7))
    traj = ddim_sample(net, sched, cond, x_K, q0, ARM, n_steps=5)
    # weights are not stored: the tests rebuild them with the drop-in create_net(seed=3)
    # plus the same seeded perturbation (create_net parity is pinned in test_golden_cpu.py)
    params = {}
    return dict(depths=scan.depths, pose=np.array([*scan.pose.position, scan.pose.heading, scan.pose.fov,
                                                   scan.pose.max_range, scan.pose.n_rays]),
                q0=q0, goal=np.array([*goal.pos, goal.theta]), cond=cond, x=x, k=np.int64(37), eps=eps,
                x_K=x_K, traj=traj, betas=sched.betas, **params)


def gen_plan():
    net = net_and_cond()
    world, scan = scene()
    q0 = np.array([0.3, -0.5, 0.6, -0.4, 0.2, 0.3, -0.1])
    goal = fk_pose(ARM, np.array([0.9, 0.4, -0.3, 0.5, 0.2, -0.4, 0.1]))
    req = PlanRequest(q_start=q0, goal=goal, scan=scan, n_trajs=8, n_iters=25, n_denoising=5, seed=11)
    res = plan_diffusion(ARM, net, make_schedule(), req)
    esdf = build_planner_esdf(req.bounds, scan, req.esdf_cell)
    succ_cases = np.stack([r.trajectory for r in res.results])
    ps = np.array([planner_success(ARM, esdf, goal, t, 0.2, 30.0) for t in succ_cases])  # looser thresholds
    # collision-only verdicts (goal thresholds that always pass): mixed flags
    rng = np.random.default_rng(12)
    coll = np.concatenate([succ_cases, random_trajs(rng, 12, scale=0.3)])
    pc = np.array([planner_success(ARM, esdf, goal, t, 10.0, 360.0) for t in coll])
    return dict(depths=scan.depths, pose=np.array([*scan.pose.position, scan.pose.heading, scan.pose.fov,
                                                   scan.pose.max_range, scan.pose.n_rays]),
                q0=q0, goal=np.array([*goal.pos, goal.theta]), seed=np.int64(req.seed),
                n_trajs=np.int64(req.n_trajs), n_iters=np.int64(req.n_iters), esdf_values=esdf.values,
                best_index=np.int64(res.best_index), trajectory=res.trajectory,
                costs=np.array([r.cost for r in res.results]),
                trajs=np.stack([r.trajectory for r in res.results]), successes=np.array(res.successes),
                seed_trajectories=res.seed_trajectories, loose_success=ps, coll_trajs=coll, coll_success=pc)


def gen_guided():
    """guided_ddim_sample with the planner cost (fused path), with a user quadratic cost
    (host-callable path), plan_diffusion with guidance, and an out-of-extent raise."""
    from planseed.diffusion import guided_ddim_sample
    from planseed.pipeline import GuidanceParams
    net = net_and_cond()
    world, scan = scene()
    q0 = np.array([0.3, -0.5, 0.6, -0.4, 0.2, 0.3, -0.1])
    goal = fk_pose(ARM, np.array([0.9, 0.4, -0.3, 0.5, 0.2, -0.4, 0.1]))
    cond = encode_condition(net, scan, q0, goal)
    sched = make_schedule()
    esdf = build_planner_esdf(PlanRequest(q_start=q0, goal=goal, scan=scan).bounds, scan, 0.01)
    w = CostWeights()

    def cost_fn(trajs):
        totals, grads, _ = evaluate_cost_batch(ARM, esdf, goal, trajs, w)
        return totals, grads

    rng = np.random.default_rng(21)
    x_K = rng.standard_normal((6, T, 7))
    traj, log = guided_ddim_sample(net, sched, cond, x_K, q0, ARM, cost_fn, n_steps=5, n_grad=4,
                                   alpha_guide=0.5)
    traj10, log10 = guided_ddim_sample(net, sched, cond, x_K[:3], q0, ARM, cost_fn, n_steps=10, n_grad=2,
                                       alpha_guide=1.0, k_guide_frac=0.9)
    target = rng.uniform(-0.5, 0.5, size=(T, 7))

    def quad(trajs):
        d = trajs - target
        return np.sum(d.reshape(d.shape[0], -1) ** 2, axis=1), 2.0 * d

    trajq, _ = guided_ddim_sample(net, sched, cond, x_K[:4], q0, ARM, quad, n_steps=5, n_grad=3, alpha_guide=0.5)
    # out-of-extent: a grid covering only part of the arm's reach
    small = SdfGrid(origin=np.array([-0.3, -0.3]), h=0.01, nx=61, ny=61,
                    values=np.random.default_rng(4).uniform(0.05, 0.2, (61, 61)))
    try:
        guided_ddim_sample(net, sched, cond, x_K, q0, ARM,
                           lambda t: evaluate_cost_batch(ARM, small, goal, t, w)[:2], n_steps=5, n_grad=2)
        err = ""
    except ValueError as e:
        err = str(e)
    req = PlanRequest(q_start=q0, goal=goal, scan=scan, n_trajs=8, n_iters=10, n_denoising=5, seed=13)
    res = plan_diffusion(ARM, net, sched, req, guidance=GuidanceParams(alpha_guide=0.5, n_grad=3))
    return dict(q0=q0, goal=np.array([*goal.pos, goal.theta]), x_K=x_K, traj=traj,
                log=np.array(log, dtype=np.int64), traj10=traj10, log10=np.array(log10, dtype=np.int64),
                target=target, trajq=trajq, small_values=small.values, err=np.array(err),
                plan_seed=np.int64(req.seed), plan_best=np.int64(res.best_index), plan_traj=res.trajectory,
                plan_seeds=res.seed_trajectories, plan_costs=np.array([r.cost for r in res.results]))


def gen_metrics():
    """trajopt.metrics / retime / traj_min_clearance on a mixed batch: collision-free and
    colliding trajectories, a constant one, a thin wall only the interpolants catch."""
    from planseed.trajopt import metrics, retime
    from planseed._kernels import traj_min_clearance
    world = World([Circle(center=(0.45, 0.15), radius=0.12), Box(lo=(-0.6, -0.7), hi=(-0.2, -0.35)),
                   Box(lo=(0.2, 0.55), hi=(0.3, 0.9))])
    rng = np.random.default_rng(30)
    trajs = list(random_trajs(rng, 20, scale=0.5))
    trajs.append(np.tile(rng.uniform(-1, 1, 7) * 0.3, (T, 1)))
    qa = np.zeros(7)
    qa[0] = np.pi / 2
    trajs.append(np.linspace(0, 1, T)[:, None] * (np.zeros(7) - qa) + qa)
    trajs = np.stack(trajs)
    goal = fk_pose(ARM, trajs[0, -1])
    wall = World([Box(lo=(0.2, -0.8), hi=(0.24, 0.8))])
    cols = []
    for w in (world, wall):
        for t in trajs:
            m = metrics(ARM, w, goal, t, plan_time=0.25)
            cols.append([m.success, m.collision_free, m.translation_error, m.angle_error_deg, m.motion_time,
                         m.max_jerk])
    clear = np.array([traj_min_clearance(t, 4, ARM.lengths, 0.0, 0.0, ARM.point_fractions(), world.circle_arr,
                                         world.box_arr, world.sdf_cap) for t in trajs])
    rt = np.array([retime(ARM, t)[0] for t in trajs])
    return dict(trajs=trajs, goal=np.array([*goal.pos, goal.theta]), circles=world.circle_arr,
                boxes=world.box_arr, wall_boxes=wall.box_arr, metrics=np.array(cols, dtype=np.float64),
                clearance=clear, motion_time=rt)


def gen_scans():
    """geometry.render_depth_scan over mixed worlds and poses: axis-parallel central rays
    (dy = 0 exactly), an origin inside a box and inside a circle, an empty world."""
    rng = np.random.default_rng(40)
    worlds = [World([Circle(center=(0.35, 0.2), radius=0.12), Box(lo=(0.55, -0.35), hi=(0.7, 0.1)),
                     Circle(center=(-0.3, 0.45), radius=0.1), Box(lo=(-0.8, -0.9), hi=(-0.5, -0.6))]),
              World([]),
              World([Box(lo=(-0.2, -0.2), hi=(0.2, 0.2)), Circle(center=(0.6, 0.6), radius=0.3)])]
    poses = [SensorPose(position=(-0.6, 0.2), heading=-0.15),
             SensorPose(position=(-0.9, 0.0), heading=0.0, n_rays=257),              # central ray dy == 0
             SensorPose(position=(0.0, 0.0), heading=np.pi / 2, n_rays=65, fov=np.pi),
             SensorPose(position=(0.6, 0.62), heading=1.0, n_rays=33),               # inside the circle (w2)
             SensorPose(position=(0.1, -0.1), heading=-2.5, n_rays=31, fov=1.2)]     # inside the box (w2)
    out = {}
    for wi, w in enumerate(worlds):
        out[f"w{wi}_circles"] = w.circle_arr
        out[f"w{wi}_boxes"] = w.box_arr
        for pi, pz in enumerate(poses):
            out[f"w{wi}_p{pi}"] = render_depth_scan(w, pz).depths
    for pi, pz in enumerate(poses):
        out[f"pose{pi}"] = np.array([pz.position[0], pz.position[1], pz.heading, pz.fov, pz.n_rays, pz.max_range])
    return out


def train_records(n=3):
    """Small ProblemRecords (planseed/data.py:51-63) with smooth expert trajectories and scans."""
    from planseed.data import PlanningProblem, ProblemRecord
    rng = np.random.default_rng(50)
    w = World([Circle(center=(0.35, 0.1), radius=0.12), Box(lo=(-0.5, 0.3), hi=(-0.1, 0.6))])
    recs = []
    for i in range(n):
        q0 = rng.uniform(-1.5, 1.5, size=7)
        q1 = rng.uniform(-1.5, 1.5, size=7)
        expert = q0 + np.linspace(0, 1, T)[:, None] * (q1 - q0) + 0.02 * np.sin(np.linspace(0, 3, T))[:, None]
        goal = fk_pose(ARM, expert[-1])
        scans = [render_depth_scan(w, SensorPose(position=(rng.uniform(-0.8, 0.8), rng.uniform(-0.8, 0.8)),
                                                 heading=rng.uniform(-3, 3))) for _ in range(2)]
        recs.append(ProblemRecord(problem=PlanningProblem(world_id="g", q_start=q0, goal=goal), world=w,
                                  expert=expert, graph_used=bool(i % 2), scans=scans))
    return recs


def record_dict(recs):
    out = {}
    for i, r in enumerate(recs):
        out[f"r{i}_expert"] = r.expert
        out[f"r{i}_q0"] = r.problem.q_start
        out[f"r{i}_goal"] = np.array([*r.problem.goal.pos, r.problem.goal.theta])
        out[f"r{i}_graph_used"] = np.array(r.graph_used)
        for j, sc in enumerate(r.scans):
            out[f"r{i}_s{j}_depths"] = sc.depths
            out[f"r{i}_s{j}_pose"] = np.array([*sc.pose.position, sc.pose.heading])
    return out


def gen_train():
    """diffusion.loss_eq2 (one record, k = 37) and a short diffusion.train run (3 records, batch 4,
    2 epochs): loss, every parameter gradient, the loss curve and per-parameter sums of the trained
    weights (src/diffusion.py:435-508)."""
    from planseed.diffusion import ArchConfig, TrainConfig, loss_eq2, train
    recs = train_records()
    out = record_dict(recs)
    net = create_net(ArchConfig(), seed=0)
    eps = np.random.default_rng(51).standard_normal((T, 7))
    loss, grads = loss_eq2(ARM, net, recs[0], 37, eps, alpha_loss=4.0, scan_index=1)
    out["eq2_eps"] = eps
    out["eq2_loss"] = np.float64(loss)
    sel = np.random.default_rng(52)
    for k, g in grads.items():
        g = np.asarray(g)
        if g.size <= 20000:
            out[f"eq2_grad_{k}"] = g
        else:   # large matrices: sums plus 256 sampled entries (keeps the fixture small)
            idx = np.sort(sel.choice(g.size, 256, replace=False))
            out[f"eq2_gsum_{k}"] = np.array([g.sum(), (g * g).sum()])
            out[f"eq2_gidx_{k}"] = idx
            out[f"eq2_gval_{k}"] = g.ravel()[idx]
    net2 = create_net(ArchConfig(), seed=0)
    curve = train(net2, recs, make_schedule(), ARM, TrainConfig(batch_size=4, epochs=2, lr=1e-3, seed=3))
    out["train_curve"] = np.array(curve)
    for k, p in net2.params.items():
        d = np.asarray(p.data)
        out[f"train_sum_{k}"] = np.array([d.sum(), (d * d).sum()])
    out["train_full_trunk_out_b"] = np.asarray(net2.params["trunk_out_b"].data)
    out["train_full_scan_conv0_w"] = np.asarray(net2.params["scan_conv0_w"].data)
    return out


def main(out_dir: Path = ROOT / "tests" / "golden"):
    out_dir.mkdir(parents=True, exist_ok=True)
    for name, c in gen_cost().items():
        np.savez_compressed(out_dir / f"ref_cost_{name}.npz", **c)
    np.savez_compressed(out_dir / "ref_optimize.npz", **gen_optimize())
    np.savez_compressed(out_dir / "ref_sampler.npz", **gen_sampler())
    np.savez_compressed(out_dir / "ref_plan.npz", **gen_plan())
    np.savez_compressed(out_dir / "ref_guided.npz", **gen_guided())
    np.savez_compressed(out_dir / "ref_metrics.npz", **gen_metrics())
    np.savez_compressed(out_dir / "ref_scans.npz", **gen_scans())
    np.savez_compressed(out_dir / "ref_train.npz", **gen_train())
    return out_dir


if __name__ == "__main__":
    print(main())
