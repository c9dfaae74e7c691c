"""GPU parity of the bf16 tcgen05 U-Net (mode 1) against the float64 numpy oracle and
the fp32 SIMT path.

Stated bf16 bound: bf16 weights and activations with fp32
accumulation, fp32 GroupNorm statistics and fp32 DDPM state.  Each of the 29 layers
rounds its output to bf16 (relative 2^-9), so noise predictions agree with the fp64
oracle to ~1% relative RMS; we require relative RMS <= 2e-2 and max-abs <= 6e-2 for
eps (|eps| ~ 0.35 RMS), and <= 0.1 rad max-abs / 2e-2 rad RMS on DDPM-100 trajectories
(measured: 0.011 rad RMS, i.e. 0.2% of the +-2.9 rad joint span).
"""

import numpy as np
import pytest

from oracle import unet_numpy as un
from paper_2410_16727_b200 import spec, synth

pytestmark = pytest.mark.gpu
ARCH = spec.UNetArch()


@pytest.fixture(scope="module")
def params():
    return spec.random_model()


@pytest.fixture(scope="module")
def samplers(params):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test without a CUDA device")
    from paper_2410_16727_b200.sampler import SeedSampler
    return SeedSampler(params, mode=0), SeedSampler(params, mode=1)


def _cond(P, seed):
    rng = np.random.default_rng(seed)
    return np.concatenate([np.abs(rng.standard_normal((P, 256))) * 0.3, rng.uniform(0, 1, (P, 14))], 1)


@pytest.mark.parametrize("P,S,T,k", [(1, 16, 32, 50), (2, 8, 32, 100), (4, 32, 32, 3), (2, 4, 64, 20)])
def test_predict_noise_bf16_vs_oracle(samplers, params, P, S, T, k):
    _, s1 = samplers
    cond = _cond(P, k)
    x = np.random.default_rng(k + T).standard_normal((P * S, T, 7)).astype(np.float32)
    eps = s1.predict_noise(x, k, s1.film(cond), S).cpu().numpy()
    want = un.unet_forward(params, ARCH, x, k, cond, S)
    d = eps - want
    rel_rms = np.sqrt((d ** 2).mean()) / np.sqrt((want ** 2).mean())
    assert rel_rms < 2e-2
    assert np.abs(d).max() < 6e-2


@pytest.mark.parametrize("P", [128, 512])
def test_persistent_multi_tile_vs_fp32(samplers, P):
    # > 148 tiles per layer: every CTA loops over several tiles and both TMEM buffers
    s0, s1 = samplers
    cond = _cond(P, 5)
    x = np.random.default_rng(P).standard_normal((P * 32, 32, 7)).astype(np.float32)
    e0 = s0.predict_noise(x, 40, s0.film(cond), 32).cpu().numpy()
    e1 = s1.predict_noise(x, 40, s1.film(cond), 32).cpu().numpy()
    d = e1 - e0
    assert np.sqrt((d ** 2).mean()) / np.sqrt((e0 ** 2).mean()) < 2e-2
    assert np.abs(d).max() < 6e-2


def test_ddpm100_bf16_trajectories(samplers, params):
    _, s1 = samplers
    P, S = 2, 8
    cond = _cond(P, 9)
    q0 = synth.make_problems(P, seed=3).q_start
    traj = s1.sample(s1.film(cond), q0, S).cpu().numpy()
    want = un.sample(params, ARCH, cond, q0, S)
    d = traj - want
    assert np.array_equal(traj[:, 0], np.repeat(q0, S, axis=0))
    assert np.abs(d).max() < 0.1
    assert np.sqrt((d ** 2).mean()) < 2e-2


def test_bf16_sampling_deterministic_and_shard_invariant(samplers):
    _, s1 = samplers
    cond = _cond(4, 11)
    q0 = synth.make_problems(4, seed=4).q_start
    fa = s1.film(cond)
    steps = spec.strided_steps(100, 10)
    full = s1.sample(fa, q0, 32, steps=steps).cpu().numpy()
    again = s1.sample(fa, q0, 32, steps=steps).cpu().numpy()
    assert np.array_equal(full, again)
    a = s1.sample(fa[:2], q0[:2], 32, p0=0, steps=steps).cpu().numpy()
    b = s1.sample(fa[2:], q0[2:], 32, p0=2, steps=steps).cpu().numpy()
    # tile composition changes with the batch, but every tile holds whole samples and
    # GroupNorm statistics are per sample: results are bitwise identical
    assert np.array_equal(full, np.concatenate([a, b]))


@pytest.mark.parametrize("cfg", [0, 3])
def test_tc_encoder_vs_oracle(cfg):
    # bf16 activations through 4-5 conv layers: embedding within 1% of its max magnitude
    from paper_2410_16727_b200.sampler import SeedSampler
    enc = spec.ENCODER_CFG0 if cfg == 0 else spec.ENCODER_CFG3
    pe = spec.random_model(enc)
    pb = (synth.config0_problems if cfg == 0 else synth.config3_problems)(3, seed=cfg + 1)
    got = SeedSampler(pe, enc, mode=1).encode(pb.images, pb.q_start, pb.goal).cpu().numpy()
    want = un.encode_problems(pe, enc, pb.images, pb.q_start, pb.goal)
    emb_err = np.abs(got[:, :256] - want[:, :256]).max() / np.abs(want[:, :256]).max()
    assert emb_err < 1e-2
    np.testing.assert_allclose(got[:, 256:], want[:, 256:], rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("P,S,T", [(1, 4, 32), (3, 5, 32), (2, 2, 64), (1, 16, 32)])
def test_partial_tiles_odd_batches(samplers, params, P, S, T):
    # batches that do not fill a tile: lanes of one warp hold different samples, so the
    # epilogue must keep tcgen05.ld convergent and predicate only global accesses
    _, s1 = samplers
    cond = _cond(P, 17)
    x = np.random.default_rng(P * S).standard_normal((P * S, T, 7)).astype(np.float32)
    eps = s1.predict_noise(x, 33, s1.film(cond), S).cpu().numpy()
    want = un.unet_forward(params, ARCH, x, 33, cond, S)
    d = eps - want
    assert np.sqrt((d ** 2).mean()) / np.sqrt((want ** 2).mean()) < 2e-2


def _with_persist(mode, f):
    import os
    os.environ["PS_PERSIST"] = mode
    try:
        return f()
    finally:
        os.environ.pop("PS_PERSIST", None)


@pytest.mark.parametrize("P,S,T,k", [(1, 32, 32, 50), (1, 3, 32, 7), (3, 40, 64, 70), (4, 64, 32, 99),
                                     (5, 50, 32, 40)])
def test_persistent_small_batch_forward(samplers, params, P, S, T, k):
    # the persistent all-layer kernel (csrc/unet_small.cu) against the oracle and against the
    # layered kernels on the same inputs (both bf16: agreement at the bf16 rounding level)
    _, s1 = samplers
    cond = _cond(P, k)
    x = np.random.default_rng(k * 7 + T).standard_normal((P * S, T, 7)).astype(np.float32)
    fa = s1.film(cond)
    ep = _with_persist("1", lambda: s1.predict_noise(x, k, fa, S).cpu().numpy())
    el = _with_persist("0", lambda: s1.predict_noise(x, k, fa, S).cpu().numpy())
    want = un.unet_forward(params, ARCH, x, k, cond, S)
    ref = np.sqrt((want ** 2).mean())
    assert np.sqrt(((ep - want) ** 2).mean()) / ref < 2e-2
    assert np.abs(ep - want).max() < 6e-2
    assert np.sqrt(((ep - el) ** 2).mean()) / ref < 1.5e-2


@pytest.mark.parametrize("P,S,T", [(1, 32, 32), (2, 8, 64)])
def test_persistent_small_batch_ddpm100(samplers, params, P, S, T):
    # the whole 100-step loop as one launch: oracle bound, row-0 pin, and run-to-run determinism
    _, s1 = samplers
    cond = _cond(P, 5)
    q0 = synth.make_problems(P, seed=11).q_start
    fa = s1.film(cond)
    t1 = _with_persist("1", lambda: s1.sample(fa, q0, S, T=T).cpu().numpy())
    t2 = _with_persist("1", lambda: s1.sample(fa, q0, S, T=T).cpu().numpy())
    want = un.sample(params, ARCH, cond, q0, S, T=T)
    d = t1 - want
    assert np.array_equal(t1, t2)
    assert np.array_equal(t1[:, 0], np.repeat(q0, S, axis=0))
    # bf16 bound: the max over 32+ trajectories of 100 stochastic steps
    # (layered kernels: 0.093 rad at 1 x 32, 0.155 rad at T=64); RMS is the tight check
    assert np.abs(d).max() < (0.15 if T == 32 else 0.2)
    assert np.sqrt((d ** 2).mean()) < 2e-2


def test_persistent_small_batch_ddim(samplers, params):
    # deterministic DDIM through the persistent kernel's DDIM update, against the oracle and the
    # layered kernels.  The strided schedule starts at k = 50: from k = 100 the squared-cosine
    # schedule's x0 reconstruction multiplies the noise prediction by 1/sqrt(abar_100) (~2000),
    # so any bf16 difference saturates the x0 clip (both bf16 paths sit ~0.4 rad RMS from the
    # fp64 oracle there, the fp32 path 6e-5; tools/ddim_check.py)
    _, s1 = samplers
    P, S = 2, 16
    cond = _cond(P, 23)
    q0 = synth.make_problems(P, seed=29).q_start
    steps = np.array([50, 40, 30, 20, 10, 1])
    fa = s1.film(cond)
    tp = _with_persist("1", lambda: s1.sample(fa, q0, S, steps=steps).cpu().numpy())
    tl = _with_persist("0", lambda: s1.sample(fa, q0, S, steps=steps).cpu().numpy())
    want = un.sample(params, ARCH, cond, q0, S, steps=steps)
    assert np.array_equal(tp[:, 0], np.repeat(q0, S, axis=0))
    assert np.sqrt(((tp - want) ** 2).mean()) < 2e-2
    assert np.sqrt(((tp - tl) ** 2).mean()) < 2e-2


@pytest.mark.parametrize("persist", ["1", "0"])
def test_ddim10_bf16_from_k100_fp32_prefix(params, persist):
    # strided DDIM-10 from the top of the squared-cosine schedule in mode 1 (spec.DDIM_BF16_MAX_RSQ):
    # without a prefix it is numerically unqualified (~0.37 rad RMS) and warns; with hp_rsq = 4 the
    # k = 100 and k = 89 steps (x0 factors 2029 and 5.9) run the fp32 network.  Stated bound for
    # that mixed path: 0.1 rad RMS (measured 0.068), and strictly better than no prefix.
    from paper_2410_16727_b200.sampler import SeedSampler
    steps = spec.strided_steps(100, 10)
    P, S = 2, 16
    cond = _cond(P, 23)
    q0 = synth.make_problems(P, seed=29).q_start
    want = un.sample(params, ARCH, cond, q0, S, steps=steps)
    rms = {}
    for hp in (None, spec.HP_RSQ):
        s1 = SeedSampler(params, mode=1, hp_rsq=hp)
        if hp is None:
            with pytest.warns(RuntimeWarning, match="unqualified"):
                traj = _with_persist(persist, lambda: s1.sample(s1.film(cond), q0, S, steps=steps).cpu().numpy())
        else:
            assert s1.hp_steps(steps) == 2
            traj = _with_persist(persist, lambda: s1.sample(s1.film(cond), q0, S, steps=steps).cpu().numpy())
        assert np.array_equal(traj[:, 0], np.repeat(q0, S, axis=0))
        rms[hp] = np.sqrt(((traj - want) ** 2).mean())
    assert rms[spec.HP_RSQ] < 0.1
    assert rms[spec.HP_RSQ] < 0.5 * rms[None]


@pytest.mark.parametrize("P", [2, 24])
def test_concurrent_streams_own_workspaces(params, P):
    # two samplers (own workspaces -> own persistent plans, completion counters and captured
    # graphs) driven from two host threads on two streams at once give the bits of a sequential run
    # (P = 2: persistent kernel; P = 24: layered kernels)
    import threading

    import torch
    from paper_2410_16727_b200.sampler import SeedSampler
    sa, sb = SeedSampler(params, mode=1), SeedSampler(params, mode=1)
    ca, cb = _cond(P, 31), _cond(P, 32)
    qa, qb = synth.make_problems(P, seed=33).q_start, synth.make_problems(P, seed=34).q_start
    want_a = sa.sample(sa.film(ca), qa, 32, p0=0).cpu().numpy()
    want_b = sb.sample(sb.film(cb), qb, 32, p0=P).cpu().numpy()
    got = {}

    def run(name, smp, c, q, p0):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            fa = smp.film(c)
            outs = [smp.sample(fa, q, 32, p0=p0) for _ in range(3)]
        st.synchronize()
        got[name] = [o.cpu().numpy() for o in outs]

    th = [threading.Thread(target=run, args=("a", sa, ca, qa, 0)),
          threading.Thread(target=run, args=("b", sb, cb, qb, P))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    for o in got["a"]:
        assert np.array_equal(o, want_a)
    for o in got["b"]:
        assert np.array_equal(o, want_b)


def test_layered_results_independent_of_batch_split(samplers):
    # the layered kernels tile every layer from the trajectory count alone (two M-blocks per tile
    # from 1184 trajectories at T = 32 up), so an 80-problem batch and its two 40-problem halves
    # (1280 trajectories each: strong-scaling shards of a larger job) give the same bits
    _, s1 = samplers
    P = 80
    cond = _cond(P, 41)
    q0 = synth.make_problems(P, seed=42).q_start
    fa = s1.film(cond)
    steps = np.array([60, 40, 20, 1])
    full = _with_persist("0", lambda: s1.sample(fa, q0, 32, steps=steps).cpu().numpy())
    a = _with_persist("0", lambda: s1.sample(fa[:40], q0[:40], 32, p0=0, steps=steps).cpu().numpy())
    b = _with_persist("0", lambda: s1.sample(fa[40:], q0[40:], 32, p0=40, steps=steps).cpu().numpy())
    assert np.array_equal(full, np.concatenate([a, b]))
