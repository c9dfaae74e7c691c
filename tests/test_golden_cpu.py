"""CPU checks of the ref-profile golden fixtures (tests/golden/, made from planseed by
tools/make_golden.py) and of the drop-in host pieces that must match planseed exactly
(create_net draws, PSCK checkpoints, schedule, step indices)."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"


def test_fixtures_present():
    names = sorted(p.name for p in GOLD.glob("ref_*.npz"))
    assert {"ref_optimize.npz", "ref_sampler.npz", "ref_plan.npz", "ref_guided.npz"} <= set(names)
    assert sum(n.startswith("ref_cost_") for n in names) == 7
    z = np.load(GOLD / "ref_cost_c0.npz")
    assert z["trajs"].shape == (6, 32, 7) and z["grads"].shape == (6, 32, 7)


def test_schedule_and_steps_match_reference_rules():
    from paper_2410_16727_b200.ref import diffusion
    s = diffusion.make_schedule()
    assert s.alpha_bar(1) == pytest.approx(1 - 1e-3)
    assert list(diffusion.ddim_steps(100, 5)) == [100, 75, 50, 26, 1]   # round-half-even


@pytest.mark.reference
def test_create_net_matches_planseed(planseed):
    from planseed.arm import default_arm
    from planseed.diffusion import arch_for_arm, create_net
    from paper_2410_16727_b200.ref import diffusion
    cfg_ref = arch_for_arm(default_arm())
    mine = diffusion.create_net(diffusion.arch_for_arm(default_arm()), seed=3)
    ref = create_net(cfg_ref, seed=3)
    assert list(mine.params) == list(ref.params)
    for k in ref.params:
        assert np.array_equal(mine.params[k], ref.params[k].data), k


@pytest.mark.reference
def test_checkpoint_interoperates_with_planseed(planseed, tmp_path):
    from planseed.diffusion import load_checkpoint as ref_load
    from paper_2410_16727_b200.ref import diffusion, types
    net = diffusion.create_net(diffusion.arch_for_arm(types.default_arm()), seed=1)
    diffusion.save_checkpoint(tmp_path / "m.ckpt", net, diffusion.make_schedule(), {"x": 1})
    rnet, rsched, meta = ref_load(tmp_path / "m.ckpt")
    assert meta == {"x": 1}
    for k in net.params:
        assert np.array_equal(rnet.params[k].data, net.params[k])
    back, _, _ = diffusion.load_checkpoint(tmp_path / "m.ckpt")
    assert back.config == net.config


@pytest.mark.reference
def test_committed_fixtures_are_planseed_outputs(planseed, tmp_path):
    sys.path.insert(0, str(ROOT / "tools"))
    import make_golden
    out = make_golden.main(tmp_path)
    for f in sorted(GOLD.glob("ref_*.npz")):
        a, b = np.load(f), np.load(out / f.name)
        assert sorted(a.files) == sorted(b.files)
        for k in a.files:
            assert np.array_equal(a[k], b[k]), (f.name, k)


@pytest.mark.reference
def test_golden_net_rebuild_matches_generator(planseed):
    sys.path.insert(0, str(ROOT / "tools"))
    import make_golden
    from golden_net import golden_net
    ref = make_golden.net_and_cond()
    mine = golden_net()
    for k in ref.params:
        assert np.array_equal(mine.params[k], ref.params[k].data), k
