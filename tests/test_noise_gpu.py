"""The fused-epilogue noise transform (normal4_tc / box_muller_tc, csrc/tc_ptx.cuh) -- the noise
the layered and persistent DDPM epilogues inject -- checked on the device function itself.

Bound (written here): every draw within 1e-5 absolute of the float64 Box-Muller transform of the
same raw Philox words, never non-finite.  The radius word (a >> 8) and the angle word (b >> 8)
each take 2^24 values; both are checked exhaustively, which covers the u1 -> 1 corner where an
approximate log can go positive (VERDICT r01 / ADVICE r01).
"""

import math

import numpy as np
import pytest

from oracle import unet_numpy as un
from paper_2410_16727_b200 import _lib, spec

pytestmark = pytest.mark.gpu
N24 = 1 << 24


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test without a CUDA device")
    return torch


def _bm(torch, a, b):
    n = a.numel()
    z = torch.empty(2 * n, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().ps_box_muller_probe(_lib.ptr(a), _lib.ptr(b), n, _lib.ptr(z), _lib.stream_handle()),
               "box_muller_probe")
    return z.view(n, 2).cpu().numpy().astype(np.float64)


def _u32(torch, v):
    # uint32 words through an int32 tensor (same bits)
    return torch.as_tensor(np.asarray(v, dtype=np.uint32).view(np.int32), device="cuda")


def test_radius_word_exhaustive(torch):
    m = np.arange(N24, dtype=np.uint64)
    low = np.random.default_rng(0).integers(0, 256, N24, dtype=np.uint64)
    a = ((m << np.uint64(8)) | low).astype(np.uint32)          # every value of a >> 8, incl. >= 2^24 - 64
    b = np.full(N24, 0x80000000, dtype=np.uint32)                # u2 = 1/2: angle pi, z0 = -rad
    z = _bm(torch, _u32(torch, a), _u32(torch, b))
    assert np.isfinite(z).all()
    u1 = (m.astype(np.float64) + 1.0) / N24
    rad = np.sqrt(-2.0 * np.log(u1))
    err = np.abs(z[:, 0] - rad * math.cos(math.pi))
    assert err.max() < 1e-5, f"max radius error {err.max():.3e} at a>>8={int(err.argmax())}"
    assert np.abs(z[:, 1]).max() < 1e-5
    # the top 64 words (u1 within 64 * 2^-24 of 1): the radius is tiny, never NaN, never inflated
    top = slice(N24 - 64, N24)
    assert np.abs(z[top, 0] + rad[top]).max() < 1e-6


def test_angle_word_exhaustive(torch):
    m = np.arange(N24, dtype=np.uint64)
    a = np.zeros(N24, dtype=np.uint32)                            # u1 = 2^-24: the largest radius, 5.77
    b = ((m << np.uint64(8)) | np.uint64(0x5A)).astype(np.uint32)
    z = _bm(torch, _u32(torch, a), _u32(torch, b))
    assert np.isfinite(z).all()
    rad = math.sqrt(-2.0 * math.log(1.0 / N24))
    ang = 2.0 * math.pi * (m.astype(np.float64) / N24)
    e0 = np.abs(z[:, 0] - rad * np.cos(ang)).max()
    e1 = np.abs(z[:, 1] - rad * np.sin(ang)).max()
    assert max(e0, e1) < 1e-5, (e0, e1)


@pytest.mark.parametrize("step,prob,seed", [(0, 0, 0), (100, 1023, 31), (57, 4095, 127), (2, 16383, 5)])
def test_normal4_matches_oracle_stream(torch, step, prob, seed):
    nb = 64                                                        # 256 elements: a T=32 x 7 trajectory +
    out = torch.empty(4 * nb, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().ps_normal4_probe(_lib.ptr(out), nb, step, prob, seed, spec.NOISE_SEED,
                                           _lib.stream_handle()), "normal4_probe")
    got = out.cpu().numpy()
    want = un.noise(step, np.array([prob]), np.array([seed]), 32, D=8).ravel()   # 256 = 32 x 8 elements
    assert np.abs(got - want).max() < 1e-5


def test_scan_1e8_draws_finite_and_normal(torch):
    # 1024 problems x 32 seeds x 1024 blocks x 4 = 1.34e8 draws of one step
    nonfinite = torch.zeros(1, dtype=torch.int64, device="cuda")
    mx = torch.zeros(1, dtype=torch.int32, device="cuda")
    mom = torch.zeros(2, dtype=torch.float64, device="cuda")
    n_prob, n_seed, n_blk = 1024, 32, 1024
    _lib.check(_lib.lib().ps_noise_scan(37, n_prob, n_seed, n_blk, spec.NOISE_SEED, _lib.ptr(nonfinite),
                                        _lib.ptr(mx), _lib.ptr(mom), _lib.stream_handle()), "noise_scan")
    n = n_prob * n_seed * n_blk * 4
    assert n >= 1e8
    assert int(nonfinite.item()) == 0
    zmax = float(np.array([mx.item()], dtype=np.int32).view(np.float32)[0])
    assert 4.5 < zmax <= math.sqrt(-2.0 * math.log(1.0 / N24)) + 1e-5
    m1, m2 = (mom.cpu().numpy() / n).tolist()
    assert abs(m1) < 1e-3 and abs(m2 - 1.0) < 1e-3
