"""planseed-shaped request API of the BASELINE profile (paper_2410_16727_b200.pipeline): request
validation happens before any device work, with planseed's ValueError contract
(src/pipeline.py:37-54; tests/test_pipeline.py's invalid-request cases)."""

from types import SimpleNamespace

import numpy as np
import pytest

from paper_2410_16727_b200 import spec, synth
from paper_2410_16727_b200.pipeline import BLPlanRequest, plan_diffusion_batch, requests_from_problems


def _fake_planner(S=32, Pmax=4, steps=None):
    return SimpleNamespace(S=S, Pmax=Pmax, cost=spec.BLCost(), steps=steps, T=32)


def _reqs(P=2, **kw):
    pb = synth.make_problems(P, seed=5, image_shape=(16, 16), n_images=2)
    return requests_from_problems(pb, **kw)


def test_request_fields_and_split():
    rs = _reqs(3)
    assert len(rs) == 3 and rs[1].images.shape == (2, 16, 16) and rs[2].boxes.shape[1] == 6
    assert rs[0].n_trajs == 32 and rs[0].n_iters == 10 and rs[0].n_denoising == 100


@pytest.mark.parametrize("bad", [dict(n_trajs=0), dict(n_iters=0)])
def test_request_rejects_empty(bad):
    pb = synth.make_problems(1, seed=5, image_shape=(16, 16), n_images=1)
    with pytest.raises(ValueError):
        BLPlanRequest(pb.images[0], pb.q_start[0], pb.goal[0], pb.boxes[0], **bad)


@pytest.mark.parametrize("kw,msg", [(dict(n_trajs=16), "n_trajs"), (dict(n_iters=20), "n_iters"),
                                    (dict(n_denoising=10), "n_denoising")])
def test_batch_rejects_requests_the_planner_cannot_serve(kw, msg):
    with pytest.raises(ValueError, match=msg):
        plan_diffusion_batch(_fake_planner(), _reqs(2, **kw))


def test_batch_rejects_empty_and_oversized():
    with pytest.raises(ValueError, match="at least one"):
        plan_diffusion_batch(_fake_planner(), [])
    with pytest.raises(ValueError, match="max_problems"):
        plan_diffusion_batch(_fake_planner(Pmax=1), _reqs(2))


def test_strided_schedule_request_matches_planner_steps():
    # a planner with a 10-step strided schedule serves n_denoising=10 requests, not 100
    pl = _fake_planner(steps=spec.strided_steps(100, 10))
    with pytest.raises(ValueError, match="n_denoising"):
        plan_diffusion_batch(pl, _reqs(1))
    ok = _reqs(1, n_denoising=10)
    # validation passes; the call then needs a GPU (or fails loudly without one)
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        with pytest.raises(Exception) as e:
            plan_diffusion_batch(pl, ok)
        assert "n_denoising" not in str(e.value)
    assert np.asarray(ok[0].goal).shape == (7,)
