"""Race evidence without compute-sanitizer (closed on this GPU pool): the tcgen05 kernels synchronise
TMA, MMA and epilogue roles through mbarriers, CTA pairs through remote arrivals and layers through
programmatic dependent launch, and the persistent sampler through inter-CTA completion counters.  A
missed wait shows up as run-to-run differences, so every dispatch variant is run repeatedly over
batch shapes that exercise it -- one- and two-M-block tiles, CTA pairs with a phantom tile (odd tile
counts), channel-split slices, partial last tiles, T = 64 -- and the results must be bitwise equal.
A missed wait that never changes a result is not caught; the exhaustive-looking shape list is the
cover, the planner / sampler parity tests the oracle."""

import os

import numpy as np
import pytest

from paper_2410_16727_b200 import spec

pytestmark = pytest.mark.gpu

REPEATS = 5


@pytest.fixture(scope="module")
def smp():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test without a CUDA device")
    from paper_2410_16727_b200.sampler import SeedSampler
    return SeedSampler(spec.random_model(), mode=1)


def _cond(P, seed):
    rng = np.random.default_rng(seed)
    return np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)


def _with(persist, f):
    old = os.environ.get("PS_PERSIST")
    os.environ["PS_PERSIST"] = persist
    try:
        return f()
    finally:
        if old is None:
            os.environ.pop("PS_PERSIST", None)
        else:
            os.environ["PS_PERSIST"] = old


# (problems, seeds, horizon): tiny (channel-split slices), small (one-M-block tiles, odd pair
# counts), past the two-M-block threshold (1184 trajectories), T = 64
LAYERED = [(1, 5, 32), (3, 7, 32), (9, 16, 32), (37, 32, 32), (41, 29, 32), (80, 32, 32), (4, 32, 64)]


@pytest.mark.parametrize("P,S,T", LAYERED)
def test_layered_forward_repeatable(smp, P, S, T):
    x = np.random.default_rng(P * 100 + S).standard_normal((P * S, T, 7)).astype(np.float32)
    fa = smp.film(_cond(P, P + S))
    outs = [_with("0", lambda: smp.predict_noise(x, 47, fa, S).cpu().numpy()) for _ in range(REPEATS)]
    assert np.isfinite(outs[0]).all()
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


@pytest.mark.parametrize("P,S,T", [(2, 16, 32), (37, 32, 32), (3, 32, 64)])
def test_layered_sampler_repeatable(smp, P, S, T):
    # several denoising steps: cross-layer and cross-step ordering (PDL, the FINAL epilogue's state
    # and bf16-view writes read by the next step's first layer)
    from paper_2410_16727_b200 import synth
    q0 = synth.make_problems(P, seed=P).q_start
    fa = smp.film(_cond(P, 3 * P))
    steps = np.array([60, 45, 30, 15, 1])
    outs = [_with("0", lambda: smp.sample(fa, q0, S, T, steps=steps).cpu().numpy()) for _ in range(REPEATS)]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


@pytest.mark.parametrize("P,S,T", [(1, 8, 32), (3, 21, 32), (8, 32, 32), (2, 32, 64)])
def test_persistent_sampler_repeatable(smp, P, S, T):
    # the single-launch sampler: inter-CTA completion counters between layers and steps
    from paper_2410_16727_b200 import synth
    q0 = synth.make_problems(P, seed=P + 1).q_start
    fa = smp.film(_cond(P, 5 * P))
    outs = [_with("1", lambda: smp.sample(fa, q0, S, T).cpu().numpy()) for _ in range(REPEATS)]
    assert np.isfinite(outs[0]).all()
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
