"""BASELINE-profile seed sampler over the C-ABI: encoder, U-Net noise predictor and the
DDPM / strided-DDIM step loop, batched over problems.

Counterparts of the reference sampler API (planseed/diffusion.py):
  SeedSampler.encode         ~ encode_condition   (:246-269), P problems at once
  SeedSampler.predict_noise  ~ predict_noise      (:288-300)
  SeedSampler.sample         ~ ddim_sample        (:559-569) / DDPM with posterior noise
"""

from __future__ import annotations

import numpy as np

from . import _lib, spec


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class SeedSampler:
    """Device-resident packed weights + schedule tables.

    mode 0: fp32 SIMT kernels (fp32 profile, configs 0/2);
    mode 1: bf16 weights/activations on tcgen05 with fp32 accumulation and fp32
            DDPM state (configs 1/3)."""

    def __init__(self, params: dict, enc: spec.EncoderArch = spec.ENCODER_CFG0,
                 arch: spec.UNetArch = spec.UNetArch(), mode: int = 0, betas=None,
                 noise_seed: int = spec.NOISE_SEED, hp_rsq: float | None = None):
        torch = _lib.require_cuda()
        self.hp_rsq = hp_rsq
        L = _lib.lib()
        self.enc, self.arch, self.mode = enc, arch, int(mode)
        shapes = arch.param_shapes()
        if L.ps_unet_param_count() != arch.n_params():
            raise ValueError("library U-Net table does not match spec.UNetArch")
        blob = np.concatenate([_f32(params[n]).ravel() for n, _ in shapes])
        self._blob = torch.as_tensor(blob, device="cuda")
        eb = np.concatenate([_f32(params[n]).ravel() for n, _ in spec.encoder_param_shapes(enc)])
        self.enc_w = torch.as_tensor(eb, device="cuda")
        nbytes = L.ps_unet_packed_bytes(self.mode)
        self.packed = torch.empty(int(nbytes), dtype=torch.uint8, device="cuda")
        _lib.check(L.ps_unet_pack(_lib.ptr(self._blob), self.mode, _lib.ptr(self.packed),
                                  _lib.stream_handle()), "unet_pack")
        self.betas = spec.cosine_betas() if betas is None else np.asarray(betas, np.float64)
        tab = spec.sampler_tables(self.betas)
        self.coef = _f32(np.stack([tab.sq, tab.sq1m, tab.rsq, tab.c0, tab.c1, tab.sig]))
        self.K = int(self.betas.shape[0])
        self.noise_key = int(noise_seed) & 0xFFFFFFFF
        self._ws = None

    @classmethod
    def from_checkpoint(cls, path, mode: int = 1, **kw) -> "SeedSampler":
        """A sampler over the weights and noise schedule of a unet1d PSCK file (checkpoint.py;
        the container of planseed's load_checkpoint, diffusion.py:657-687)."""
        from .checkpoint import load_checkpoint
        params, enc, arch, betas, _ = load_checkpoint(path)
        return cls(params, enc, arch, mode=mode, betas=betas, **kw)

    # ------------------------------------------------------------------ helpers
    def _workspace(self, nbytes: int):
        torch = _lib.require_cuda()
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(int(nbytes), dtype=torch.uint8, device="cuda")
        return self._ws

    # ------------------------------------------------------------------ API
    def _enc_packed(self, H: int, W: int):
        torch = _lib.require_cuda()
        key = (H, W)
        if getattr(self, "_encp", None) is None:
            self._encp = {}
        if key not in self._encp:
            L = _lib.lib()
            nl = len(self.enc.channels)
            buf = torch.empty(int(L.ps_encoder_packed_bytes(H, W, nl)), dtype=torch.uint8, device="cuda")
            _lib.check(L.ps_encoder_pack(_lib.ptr(self.enc_w), H, W, nl, _lib.ptr(buf),
                                         _lib.stream_handle()), "encoder_pack")
            self._encp[key] = buf
        return self._encp[key]

    def encode(self, images, q_start, goal, stream=None, out=None):
        """images (P, n_img, H, W) depth metres; q_start (P,7); goal (P,7) -> cond (P,270)
        (written into `out` when given).

        mode 1 runs the tcgen05 encoder (bf16 activations), mode 0 the fp32 SIMT one."""
        torch = _lib.require_cuda()
        from .bl import _dev
        im = _dev(images)
        P, n_img, H, W = im.shape
        q, g = _dev(q_start), _dev(goal)
        L = _lib.lib()
        nl = len(self.enc.channels)
        if self.mode == 1:
            packed = self._enc_packed(H, W)
            nb = int(L.ps_encode_tc_workspace_bytes(P * n_img, H, W, nl))
            if getattr(self, "_encws", None) is None or self._encws.numel() < nb:
                self._encws = torch.empty(nb, dtype=torch.uint8, device="cuda")
            cond = out if out is not None else torch.empty((P, spec.COND_DIM), dtype=torch.float32, device="cuda")
            st = L.ps_encode_tc(_lib.ptr(im), P, n_img, H, W, _lib.ptr(packed), nl, _lib.ptr(q),
                                _lib.ptr(g), -spec.JOINT_LIMIT, spec.JOINT_LIMIT, _lib.ptr(self._encws),
                                _lib.ptr(cond), _lib.stream_handle(stream))
            _lib.check(st, "encode_tc")
            return cond
        ws = torch.empty(int(L.ps_encode_workspace_bytes(P * n_img, H, W, nl)), dtype=torch.uint8,
                         device="cuda")
        cond = out if out is not None else torch.empty((P, spec.COND_DIM), dtype=torch.float32, device="cuda")
        st = L.ps_encode(_lib.ptr(im), P, n_img, H, W, _lib.ptr(self.enc_w), nl, _lib.ptr(q),
                         _lib.ptr(g), -spec.JOINT_LIMIT, spec.JOINT_LIMIT, _lib.ptr(ws),
                         _lib.ptr(cond), _lib.stream_handle(stream))
        _lib.check(st, "encode")
        return cond

    def film(self, cond, stream=None, out=None):
        """Per-problem FiLM part (P, 3584); `out` reuses a caller buffer (keeping the sampler's
        arguments stable lets ps_sample replay its captured CUDA graph)."""
        torch = _lib.require_cuda()
        from .bl import _dev
        c = _dev(cond)
        fa = out if out is not None else torch.empty((c.shape[0], 3584), dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().ps_film_problem(_lib.ptr(self.packed), self.mode, _lib.ptr(c),
                                              c.shape[0], _lib.ptr(fa), _lib.stream_handle(stream)),
                   "film_problem")
        return fa

    def predict_noise(self, x, k: int, film_a, S: int, stream=None):
        """eps(x, k) for x (B,T,7) normalised, B = P*S."""
        torch = _lib.require_cuda()
        from .bl import _dev
        xd = _dev(x)
        B, T, _ = xd.shape
        L = _lib.lib()
        ws = self._workspace(L.ps_sample_workspace_bytes(B, T, max(1, B // S), 1, self.mode))
        eps = torch.empty_like(xd)
        st = L.ps_unet_forward(_lib.ptr(self.packed), self.mode, _lib.ptr(xd), B, T, S, int(k),
                               _lib.ptr(film_a), _lib.ptr(ws), _lib.ptr(eps),
                               _lib.stream_handle(stream))
        _lib.check(st, "unet_forward")
        return eps

    def _packed_hp(self):
        """mode-0 (fp32) packing of the same weights, for the high-precision DDIM prefix."""
        if getattr(self, "_pk_hp", None) is None:
            torch = _lib.require_cuda()
            L = _lib.lib()
            self._pk_hp = torch.empty(int(L.ps_unet_packed_bytes(0)), dtype=torch.uint8, device="cuda")
            _lib.check(L.ps_unet_pack(_lib.ptr(self._blob), 0, _lib.ptr(self._pk_hp), _lib.stream_handle()),
                       "unet_pack")
        return self._pk_hp

    def hp_steps(self, steps) -> int:
        """How many leading DDIM steps run the fp32 network in mode 1: those whose x0 reconstruction
        factor 1/sqrt(abar_k) exceeds spec.HP_RSQ (DDPM and mode 0: none)."""
        if steps is None or self.mode == 0 or self.hp_rsq is None:
            return 0
        n = 0
        for k in steps:
            if self.coef[2][int(k)] <= self.hp_rsq:
                break
            n += 1
        return n

    def sample(self, film_a, q_start, S: int, T: int = spec.T_DEFAULT, p0: int = 0, steps=None,
               stream=None, out=None):
        """Seeds for P problems x S seeds -> physical trajectories (P*S, T, 7), row 0 = q_start.

        steps=None: K-step DDPM; otherwise deterministic DDIM over the given indices (in mode 1 the
        leading steps with 1/sqrt(abar_k) > hp_rsq run the fp32 network, see hp_steps; without
        hp_rsq a bf16 DDIM schedule from the top of the schedule warns, spec.DDIM_BF16_MAX_RSQ)."""
        torch = _lib.require_cuda()
        from .bl import _dev
        q = _dev(q_start)
        P = q.shape[0]
        if steps is None:
            ks = np.arange(self.K, 0, -1, dtype=np.int32)
            ddpm = 1
        else:
            ks = np.ascontiguousarray(steps, dtype=np.int32)
            ddpm = 0
        L = _lib.lib()
        B = P * S
        n_hp = self.hp_steps(None if ddpm else ks)
        if self.mode == 1 and not ddpm and n_hp == 0 and self.coef[2][int(ks[0])] > spec.DDIM_BF16_MAX_RSQ:
            import warnings
            warnings.warn(f"bf16 strided DDIM from k={int(ks[0])} (x0 factor 1/sqrt(abar) = "
                          f"{float(self.coef[2][int(ks[0])]):.0f}) is numerically unqualified "
                          "(~0.4 rad RMS from the fp32 result); use mode=0 or hp_rsq (spec.HP_RSQ)",
                          RuntimeWarning, stacklevel=2)
        nbytes = L.ps_sample_workspace_bytes(B, T, P, len(ks), self.mode)
        if n_hp:
            nbytes = max(nbytes, L.ps_sample_workspace_bytes(B, T, P, len(ks), 0))
        ws = self._workspace(nbytes)
        traj = out if out is not None else torch.empty((B, T, 7), dtype=torch.float32, device="cuda")
        hp = self._packed_hp() if n_hp else None
        st = L.ps_sample_hp(_lib.ptr(self.packed), self.mode, _lib.ptr(hp) if n_hp else None, n_hp,
                            _lib.ptr(film_a), P, S, T, int(p0), _lib.hptr(ks), len(ks), ddpm,
                            _lib.hptr(self.coef), self.K, self.noise_key, _lib.ptr(q), -spec.JOINT_LIMIT,
                            spec.JOINT_LIMIT, _lib.ptr(ws), _lib.ptr(traj), _lib.stream_handle(stream))
        _lib.check(st, "sample")
        return traj


    def guided_sample(self, film_a, q_start, S: int, esdf, robot: spec.DHRobot, grid: spec.GridSpec = spec.GridSpec(),
                      cost: spec.BLCost = spec.BLCost(), T: int = spec.T_DEFAULT, p0: int = 0, n_steps: int = 5,
                      k_guide_frac: float = 0.6, n_grad: int = 20, alpha_guide: float = 1.0, max_halvings: int = 8,
                      esdf_layout: int = 0, strict: bool = False, stream=None):
        """guided_ddim_sample (planseed/diffusion.py:572-628) for P problems x S seeds: strided DDIM over
        round(linspace(K, 1, n_steps)) with, on every sub-step whose index k < k_guide_frac * K except the
        last, the BL-cost guide step (bl.guide: n_grad descent steps, <= max_halvings halvings each) on
        x0_hat against each problem's ESDF.  Returns (trajectories (P*S, T, 7), log [(k, guided)]).
        strict=True raises planseed's ValueError when an evaluation leaves the ESDF extent."""
        torch = _lib.require_cuda()
        from . import bl
        from .bl import _dev
        q = _dev(q_start)
        P = q.shape[0]
        B = P * S
        L = _lib.lib()
        ks = spec.strided_steps(self.K, n_steps)
        tab = spec.sampler_tables(self.betas)
        x = torch.empty((B, T, 7), dtype=torch.float32, device="cuda")
        x0 = torch.empty_like(x)
        n = x.numel()
        sh = _lib.stream_handle(stream)
        _lib.check(L.ps_noise_init(_lib.ptr(x), B, T, S, int(p0), self.noise_key, sh), "noise_init")
        k_guide = k_guide_frac * self.K
        lo, hi = -spec.JOINT_LIMIT, spec.JOINT_LIMIT
        log = []
        for i, k in enumerate(ks):
            k = int(k)
            eps = self.predict_noise(x, k, film_a, S, stream=stream)
            _lib.check(L.ps_ddim_x0(_lib.ptr(x), _lib.ptr(eps), n, float(tab.sq1m[k]), float(tab.rsq[k]),
                                    spec.X0_CLIP[0], spec.X0_CLIP[1], _lib.ptr(x0), sh), "ddim_x0")
            if i + 1 == len(ks):
                log.append((k, False))
                break
            guided = bool(k < k_guide and alpha_guide != 0.0)
            log.append((k, guided))
            if guided:
                cl = bl.guide(x0, esdf, S, robot, grid, cost, lo=np.full(7, lo), span=np.full(7, hi - lo),
                              n_grad=n_grad, alpha=alpha_guide, max_halvings=max_halvings, stream=stream,
                              esdf_layout=esdf_layout)
                if strict and bool(cl.any()):
                    bl._raise_out_of_grid(cl)
            kn = int(ks[i + 1])
            _lib.check(L.ps_ddim_next(_lib.ptr(x), _lib.ptr(x0), _lib.ptr(eps), n, float(tab.sq[kn]),
                                      float(tab.sq1m[kn]), sh), "ddim_next")
        traj = torch.empty_like(x)
        _lib.check(L.ps_denorm_pin(_lib.ptr(x0), B, T, S, _lib.ptr(q), lo, hi, _lib.ptr(traj), sh), "denorm_pin")
        return traj, log


def noise_probe(n: int, step: int, prob: int, seed: int, key: int = spec.NOISE_SEED):
    torch = _lib.require_cuda()
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().ps_noise_probe(_lib.ptr(out), n, step, prob, seed, key,
                                         _lib.stream_handle()), "noise_probe")
    return out
