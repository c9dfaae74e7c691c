"""CPU pins of the BASELINE-profile sampler oracle (oracle/unet_numpy.py) and of the shared
spec tables, so that neither is its own oracle (VERDICT r01 "What's weak" 5):

  * every numpy primitive against torch.nn.functional in float64 (conv1d k5, strided conv k3 s2,
    transposed conv k4 s2, GroupNorm(8), Mish, conv2d 3x3 s2), and the whole U-Net forward
    against an independent channels-first torch restatement;
  * spec.sampler_tables against an independent derivation: the DDPM posterior
    q(x_{k-1} | x_k, x0) as the product of the two Gaussians N(x_k; sqrt(a_k) x_{k-1}, b_k) and
    N(x_{k-1}; sqrt(abar_{k-1}) x0, 1 - abar_{k-1}), with abar from the squared-cosine closed
    form f(t)/f(0) rather than the cumulative product;
  * spec.timestep_sinusoid / strided_steps against planseed's timestep_features / ddim_steps;
  * bridge (iii) of SURVEY.md §7.3: the oracle's strided DDIM loop equals planseed's own
    ddim_sample / _ddim_core (diffusion.py:535-569) given the same noise prediction.
"""

import math

import numpy as np
import pytest

from oracle import unet_numpy as un
from paper_2410_16727_b200 import spec

torch = pytest.importorskip("torch")
F = torch.nn.functional
ARCH = spec.UNetArch()


def _t(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64))


def _cl(x):  # (B,C,T) torch -> (B,T,C) numpy
    return x.permute(0, 2, 1).numpy()


RNG = np.random.default_rng(123)


class TestPrimitivesVsTorch:
    def test_conv1d_k5(self):
        x = RNG.standard_normal((3, 16, 12))
        w, b = RNG.standard_normal((10, 12, 5)), RNG.standard_normal(10)
        want = _cl(F.conv1d(_t(x).permute(0, 2, 1), _t(w), _t(b), padding=2))
        np.testing.assert_allclose(un.conv1d(x, w, b), want, rtol=0, atol=1e-12)

    def test_conv1d_k3_s2(self):
        x = RNG.standard_normal((2, 32, 8))
        w, b = RNG.standard_normal((8, 8, 3)), RNG.standard_normal(8)
        want = _cl(F.conv1d(_t(x).permute(0, 2, 1), _t(w), _t(b), stride=2, padding=1))
        np.testing.assert_allclose(un.conv1d(x, w, b, stride=2, pad=1), want, rtol=0, atol=1e-12)

    def test_conv1d_1x1(self):
        x = RNG.standard_normal((2, 8, 6))
        w, b = RNG.standard_normal((9, 6, 1)), RNG.standard_normal(9)
        want = _cl(F.conv1d(_t(x).permute(0, 2, 1), _t(w), _t(b)))
        np.testing.assert_allclose(un.conv1d(x, w, b), want, rtol=0, atol=1e-12)

    def test_conv_transpose1d_k4_s2(self):
        x = RNG.standard_normal((2, 8, 6))
        w, b = RNG.standard_normal((6, 5, 4)), RNG.standard_normal(5)
        want = _cl(F.conv_transpose1d(_t(x).permute(0, 2, 1), _t(w), _t(b), stride=2, padding=1))
        got = un.conv_transpose1d(x, w, b)
        assert got.shape == (2, 16, 5)
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)

    def test_group_norm(self):
        x = RNG.standard_normal((3, 8, 64)) * 2 + 0.5
        g, b = RNG.uniform(0.9, 1.1, 64), RNG.uniform(-0.1, 0.1, 64)
        want = _cl(F.group_norm(_t(x).permute(0, 2, 1), spec.GN_GROUPS, _t(g), _t(b), eps=spec.GN_EPS))
        np.testing.assert_allclose(un.group_norm(x, g, b), want, rtol=0, atol=1e-12)

    def test_mish(self):
        x = np.concatenate([np.linspace(-30, 30, 2001), RNG.standard_normal(100) * 5])
        np.testing.assert_allclose(un.mish(x), F.mish(_t(x)).numpy(), rtol=1e-14, atol=1e-300)

    @pytest.mark.parametrize("H,W", [(128, 128), (15, 20), (9, 9)])
    def test_conv2d_s2(self, H, W):
        x = RNG.standard_normal((3, H, W))
        w, b = RNG.standard_normal((4, 3, 3, 3)), RNG.standard_normal(4)
        want = F.conv2d(_t(x)[None], _t(w), _t(b), stride=2, padding=1)[0].numpy()
        np.testing.assert_allclose(un.conv2d_s2(x, w, b), want, rtol=0, atol=1e-12)


def _torch_unet(params, x, k, cond, S):
    """Independent channels-first restatement of spec.UNetArch with torch.nn.functional."""
    p = {n: _t(v) for n, v in params.items()}
    h = _t(x).permute(0, 2, 1)                                     # (B, 7, T)
    temb = _t(spec.timestep_sinusoid(k))
    temb = F.mish(temb @ p["t_fc1_w"] + p["t_fc1_b"]) @ p["t_fc2_w"] + p["t_fc2_b"]
    c = _t(cond)
    e = F.mish(torch.cat([temb.expand(c.shape[0], -1), c], 1))

    def block(name, xin):
        co = p[f"{name}_c0_b"].shape[0]
        f = e @ p[f"{name}_film_w"] + p[f"{name}_film_b"]
        sc, sh = f[:, :co].repeat_interleave(S, 0)[:, :, None], f[:, co:].repeat_interleave(S, 0)[:, :, None]
        y = F.conv1d(xin, p[f"{name}_c0_w"], p[f"{name}_c0_b"], padding=2)
        y = F.mish(F.group_norm(y, 8, p[f"{name}_gn0_g"], p[f"{name}_gn0_b"], eps=1e-5))
        y = y * (1 + sc) + sh
        y = F.conv1d(y, p[f"{name}_c1_w"], p[f"{name}_c1_b"], padding=2)
        y = F.mish(F.group_norm(y, 8, p[f"{name}_gn1_g"], p[f"{name}_gn1_b"], eps=1e-5))
        r = F.conv1d(xin, p[f"{name}_res_w"], p[f"{name}_res_b"]) if f"{name}_res_w" in p else xin
        return y + r

    h = block("d0r1", block("d0r0", h))
    h = F.conv1d(h, p["down0_w"], p["down0_b"], stride=2, padding=1)
    h = s1 = block("d1r1", block("d1r0", h))
    h = F.conv1d(h, p["down1_w"], p["down1_b"], stride=2, padding=1)
    h = s2 = block("d2r1", block("d2r0", h))
    h = block("m1", block("m0", h))
    h = block("u0r1", block("u0r0", torch.cat([h, s2], 1)))
    h = F.conv_transpose1d(h, p["up0_w"], p["up0_b"], stride=2, padding=1)
    h = block("u1r1", block("u1r0", torch.cat([h, s1], 1)))
    h = F.conv_transpose1d(h, p["up1_w"], p["up1_b"], stride=2, padding=1)
    h = F.conv1d(h, p["fin_c_w"], p["fin_c_b"], padding=2)
    h = F.mish(F.group_norm(h, 8, p["fin_gn_g"], p["fin_gn_b"], eps=1e-5))
    return _cl(F.conv1d(h, p["out_w"], p["out_b"]))


@pytest.mark.parametrize("T,k", [(32, 100), (64, 7)])
def test_unet_forward_vs_torch(T, k):
    params = spec.random_model()
    P, S = 2, 3
    cond = np.concatenate([np.abs(RNG.standard_normal((P, 256))) * 0.3, RNG.uniform(0, 1, (P, 14))], 1)
    x = RNG.standard_normal((P * S, T, 7))
    got = un.unet_forward(params, ARCH, x, k, cond, S)
    want = _torch_unet(params, x, k, cond, S)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-10)


def test_encoder_vs_torch():
    enc = spec.ENCODER_CFG3
    pe = spec.random_model(enc)
    img = RNG.uniform(0.3, 2.0, (60, 80))
    h = _t(img / spec.DEPTH_SCALE)[None, None]
    for i in range(len(enc.channels)):
        h = F.relu(F.conv2d(h, _t(pe[f"enc{i}_w"]), _t(pe[f"enc{i}_b"]), stride=2, padding=1))
    want = h.mean(dim=(2, 3))[0].numpy()
    np.testing.assert_allclose(un.encode_image(pe, enc, img), want, rtol=0, atol=1e-12)


class TestScheduleTables:
    @staticmethod
    def closed_form_abar(K=spec.K_STEPS, s=spec.COSINE_S):
        f = lambda t: math.cos(((t / K) + s) / (1 + s) * math.pi / 2) ** 2
        return np.array([f(t) / f(0) for t in range(K + 1)])        # abar_0 = 1 .. abar_K

    def test_abar_closed_form(self):
        b = spec.cosine_betas()
        ab = np.cumprod(1 - b)
        cf = self.closed_form_abar()
        # identical up to the beta <= 0.999 clip, which binds only at k = K (f(K) = 0)
        np.testing.assert_allclose(ab[:-1], cf[1:-1], rtol=1e-12, atol=0)
        assert b[-1] == 0.999 and cf[-1] < 1e-30

    def test_posterior_is_gaussian_product(self):
        b = spec.cosine_betas()
        tab = spec.sampler_tables(b)
        ab = np.concatenate([[1.0], np.cumprod(1 - b)])              # ab[k] = abar_k, ab[0] = 1
        for k in range(2, spec.K_STEPS + 1):
            a_k, b_k = 1 - b[k - 1], b[k - 1]
            prec = a_k / b_k + 1 / (1 - ab[k - 1])
            var = 1 / prec
            c1 = var * math.sqrt(a_k) / b_k
            c0 = var * math.sqrt(ab[k - 1]) / (1 - ab[k - 1])
            assert tab.c0[k] == pytest.approx(c0, rel=2e-7, abs=1e-9)
            assert tab.c1[k] == pytest.approx(c1, rel=2e-7, abs=1e-9)
            assert tab.sig[k] == pytest.approx(math.sqrt(var), rel=2e-7)
        # k = 1: the posterior collapses onto x0 (abar_0 = 1): mean = x0, no noise
        assert tab.c0[1] == pytest.approx(1.0, rel=1e-7) and abs(tab.c1[1]) < 1e-7 and tab.sig[1] == 0.0

    def test_reconstruction_tables(self):
        b = spec.cosine_betas()
        tab = spec.sampler_tables(b)
        ab = np.cumprod(1 - b)
        for k in (1, 50, 89, 100):
            assert tab.sq[k] == np.float32(math.sqrt(ab[k - 1]))
            assert tab.sq1m[k] == np.float32(math.sqrt(1 - ab[k - 1]))
            assert tab.rsq[k] == np.float32(1 / math.sqrt(ab[k - 1]))


@pytest.mark.reference
class TestBridgeToPlanseedSampler:
    def test_sinusoid_and_steps(self, planseed):
        from planseed import diffusion as D
        cfg = D.ArchConfig(t_embed=spec.T_EMB)
        ks = np.array([1, 2, 37, 89, 100])
        np.testing.assert_array_equal(spec.timestep_sinusoid(ks), D.timestep_features(cfg, ks, 100))
        for n in (1, 2, 5, 10, 17, 100):
            np.testing.assert_array_equal(spec.strided_steps(100, n), D.ddim_steps(100, n))

    @pytest.mark.parametrize("n_steps", [5, 10])
    def test_ddim_loop_equals_ddim_sample(self, planseed, monkeypatch, n_steps):
        """Same noise prediction on both sides (a fixed nonlinear map of (x, k)); the oracle's DDIM
        update, x0 clip, denormalisation and row-0 pin must reproduce planseed's ddim_sample."""
        from planseed import arm as A
        from planseed import diffusion as D

        mix = np.random.default_rng(5).standard_normal((7, 7)) * 0.4

        def eps_fn(x, k):
            x = np.asarray(x, dtype=np.float64)
            return np.tanh(x @ mix + 0.013 * k) * 0.9 + 0.05 * np.roll(x, 1, axis=-2)

        monkeypatch.setattr(D, "predict_noise", lambda net, x, k, cond, K=100: eps_fn(x, k))
        monkeypatch.setattr(un, "unet_forward", lambda params, arch, x, k, cond, S, dtype=np.float64: eps_fn(x, k))
        sched = D.NoiseSchedule(betas=spec.cosine_betas())
        arm = A.default_arm(7)
        assert np.all(arm.lo == -spec.JOINT_LIMIT) and np.all(arm.hi == spec.JOINT_LIMIT)
        S = 6
        x_K = np.random.default_rng(9).standard_normal((S, 32, 7))
        q0 = np.random.default_rng(10).uniform(-2, 2, 7)
        want = D.ddim_sample(None, sched, np.zeros(3), x_K, q0, arm, n_steps=n_steps)
        kw = dict(steps=spec.strided_steps(100, n_steps), x_init=x_K)
        got = un.sample({}, ARCH, np.zeros((1, spec.COND_DIM)), q0[None], S, table_dtype=np.float64, **kw)
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)
        # with the device's float32 coefficient tables (relative rounding 6e-8, amplified by
        # 1/sqrt(abar_100) ~ 2e3 at the first step) the oracle stays within 1e-5 rad
        got32 = un.sample({}, ARCH, np.zeros((1, spec.COND_DIM)), q0[None], S, **kw)
        np.testing.assert_allclose(got32, want, rtol=0, atol=1e-5)
