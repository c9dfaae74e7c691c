"""GPU training of the reference profile's denoiser (ref/train.py + csrc/ref_train.cu) against
planseed's own loss_eq2 and train (src/diffusion.py:435-508), through the golden fixture
tests/golden/ref_train.npz (tools/make_golden.py:gen_train).  float64: loss and gradients within
1e-9 relative, the 2-epoch loss curve and the trained weights within 1e-8."""

from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "ref_train.npz"


@pytest.fixture(scope="module")
def z():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test without a CUDA device")
    return np.load(GOLD)


def _records(z, n=3):
    from paper_2410_16727_b200.ref.types import Pose2
    recs = []
    for i in range(n):
        scans = []
        j = 0
        while f"r{i}_s{j}_depths" in z.files:
            px, py, hd = z[f"r{i}_s{j}_pose"]
            scans.append(SimpleNamespace(depths=z[f"r{i}_s{j}_depths"],
                                         pose=SimpleNamespace(position=(px, py), heading=hd)))
            j += 1
        gx, gy, gth = z[f"r{i}_goal"]
        recs.append(SimpleNamespace(problem=SimpleNamespace(q_start=z[f"r{i}_q0"], goal=Pose2((gx, gy), gth)),
                                    expert=z[f"r{i}_expert"], graph_used=bool(z[f"r{i}_graph_used"]), scans=scans))
    return recs


def _net():
    from paper_2410_16727_b200.ref.diffusion import ArchConfig, create_net
    return create_net(ArchConfig(), seed=0)


def test_loss_eq2_matches_planseed(z):
    from paper_2410_16727_b200.ref import train
    from paper_2410_16727_b200.ref.types import default_arm
    loss, grads = train.loss_eq2(default_arm(), _net(), _records(z)[0], 37, z["eq2_eps"], alpha_loss=4.0,
                                 scan_index=1)
    assert loss == pytest.approx(float(z["eq2_loss"]), rel=1e-10)
    n_checked = 0
    for k, g in grads.items():
        if f"eq2_grad_{k}" in z.files:
            want = z[f"eq2_grad_{k}"]
            np.testing.assert_allclose(g, want, rtol=1e-8, atol=1e-12 * max(1.0, np.abs(want).max()))
        else:
            s = z[f"eq2_gsum_{k}"]
            assert g.sum() == pytest.approx(s[0], rel=1e-8, abs=1e-12)
            assert (g * g).sum() == pytest.approx(s[1], rel=1e-8)
            np.testing.assert_allclose(g.ravel()[z[f"eq2_gidx_{k}"]], z[f"eq2_gval_{k}"], rtol=1e-8, atol=1e-14)
        n_checked += 1
    assert n_checked == len(grads) and n_checked >= 30


def test_train_matches_planseed(z):
    from paper_2410_16727_b200.ref import train
    from paper_2410_16727_b200.ref.diffusion import make_schedule
    from paper_2410_16727_b200.ref.types import default_arm
    net = _net()
    curve = train.train(net, _records(z), make_schedule(), default_arm(),
                        train.TrainConfig(batch_size=4, epochs=2, lr=1e-3, seed=3))
    np.testing.assert_allclose(curve, z["train_curve"], rtol=1e-10)
    for k, p in net.params.items():
        p = np.asarray(getattr(p, "data", p))
        s = z[f"train_sum_{k}"]
        assert p.sum() == pytest.approx(s[0], rel=1e-8, abs=1e-10), k
        assert (p * p).sum() == pytest.approx(s[1], rel=1e-8), k
    np.testing.assert_allclose(np.asarray(net.params["trunk_out_b"]), z["train_full_trunk_out_b"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(np.asarray(net.params["scan_conv0_w"]), z["train_full_scan_conv0_w"], rtol=1e-8,
                               atol=1e-12)
