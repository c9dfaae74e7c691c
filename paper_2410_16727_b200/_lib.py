"""ctypes binding of libps_b200.so (the C-ABI declared in include/ps_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA device
is visible, every entry point raises.  Tensors cross the boundary as raw device
pointers plus sizes; torch is only the allocator and stream provider.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import build as _build

PS_OK, PS_ERR_OUT_OF_GRID, PS_ERR_SHAPE, PS_ERR_CUDA = 0, 1, 2, 3

_c_int, _c_ll, _c_f, _vp = ctypes.c_int, ctypes.c_longlong, ctypes.c_float, ctypes.c_void_p
_c_d = ctypes.c_double
# lengths, basex, basey, fracs, M, pair_a, pair_b, n_pairs, grid, nx, ny, gox, goy, gh,
# goal_x, goal_y, goal_th, weights, d_act, d_self, jerk_mat, jerk_quad
_REF_ARM = [_vp, _c_d, _c_d, _vp, _c_int, _vp, _vp, _c_int, _vp, _c_int, _c_int, _c_d, _c_d, _c_d,
            _c_d, _c_d, _c_d, _vp, _c_d, _c_d, _vp, _vp]

# name -> argtypes ; every function returns int (status) unless listed in _RESTYPE
_SIGS = {
    "ps_version": [],
    "ps_launch_count": [],
    "ps_esdf_build_boxes": [_vp, _c_int, _c_int, _vp, _vp, _c_f, _c_f, _vp, _vp],
    "ps_esdf_build_boxes_layout": [_vp, _c_int, _c_int, _vp, _vp, _c_f, _c_f, _vp, _c_int, _vp],
    "ps_bl_refine_layout": [_vp, _c_int, _c_int, _c_int, _vp, _c_ll, _c_int, _vp, _vp, _c_f, _vp, _vp, _vp, _vp,
                            _c_int, _vp, _c_int, _vp, _vp, _vp, _vp, _vp],
    "ps_esdf_quad_expand": [_vp, _c_int, _vp, _vp, _vp],
    "ps_bl_cost": [_vp, _c_int, _c_int, _c_int, _vp, _c_ll, _vp, _vp, _c_f, _vp, _vp, _vp, _vp,
                   _c_int, _vp, _vp, _vp, _vp, _vp],
    "ps_bl_refine": [_vp, _c_int, _c_int, _c_int, _vp, _c_ll, _vp, _vp, _c_f, _vp, _vp, _vp, _vp,
                     _c_int, _vp, _c_int, _vp, _vp, _vp, _vp, _vp],
    "ps_bl_cost_layout": [_vp, _c_int, _c_int, _c_int, _vp, _c_ll, _c_int, _vp, _vp, _c_f, _vp, _vp, _vp, _vp,
                          _c_int, _vp, _vp, _vp, _vp, _vp],
    "ps_bl_optimize": [_vp, _c_int, _c_int, _c_int, _vp, _c_ll, _c_int, _vp, _vp, _c_f, _vp, _vp, _vp, _vp,
                       _c_int, _vp, _c_int, _vp, _vp, _vp, _vp, _vp, _vp],
    "ps_bl_metrics": [_vp, _c_int, _c_int, _c_int, _vp, _c_int, _vp, _vp, _vp, _vp, _vp, _c_int, _vp, _c_f, _c_f,
                      _c_f, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "ps_bl_guide": [_vp, _c_int, _c_int, _c_int, _vp, _c_ll, _c_int, _vp, _vp, _c_f, _vp, _vp, _vp, _vp, _c_int,
                    _vp, _vp, _vp, _c_int, _c_f, _c_int, _vp, _vp],
    "ps_render_depth_rects": [_vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp],
    "ps_noise_init": [_vp, _c_int, _c_int, _c_int, _c_int, ctypes.c_uint, _vp],
    "ps_ddim_x0": [_vp, _vp, _c_ll, _c_f, _c_f, _c_f, _c_f, _vp, _vp],
    "ps_ddim_next": [_vp, _vp, _vp, _c_ll, _c_f, _c_f, _vp],
    "ps_denorm_pin": [_vp, _c_int, _c_int, _c_int, _vp, _c_f, _c_f, _vp, _vp],
    "ps_select": [_vp, _vp, _c_int, _c_int, _vp, _vp],
    "ps_unet_param_count": [],
    "ps_unet_param_offset": [ctypes.c_char_p],
    "ps_unet_packed_bytes": [_c_int],
    "ps_unet_pack": [_vp, _c_int, _vp, _vp],
    "ps_encode_workspace_bytes": [_c_int, _c_int, _c_int, _c_int],
    "ps_encode": [_vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _vp, _vp, _c_f, _c_f, _vp, _vp,
                  _vp],
    "ps_film_problem": [_vp, _c_int, _vp, _c_int, _vp, _vp],
    "ps_film_steps": [_vp, _c_int, _vp, _c_int, _vp, _vp, _vp],
    "ps_unet_forward": [_vp, _c_int, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp],
    "ps_sample_workspace_bytes": [_c_int, _c_int, _c_int, _c_int, _c_int],
    "ps_sample": [_vp, _c_int, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _c_int, _vp, _c_int,
                  ctypes.c_uint, _vp, _c_f, _c_f, _vp, _vp, _vp],
    "ps_sample_hp": [_vp, _c_int, _vp, _c_int, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _c_int, _vp,
                     _c_int, ctypes.c_uint, _vp, _c_f, _c_f, _vp, _vp, _vp],
    "ps_noise_probe": [_vp, _c_int, _c_int, _c_int, _c_int, ctypes.c_uint, _vp],
    "ps_box_muller_probe": [_vp, _vp, _c_int, _vp, _vp],
    "ps_normal4_probe": [_vp, _c_int, _c_int, _c_int, _c_int, ctypes.c_uint, _vp],
    "ps_noise_scan": [_c_int, _c_int, _c_int, _c_int, ctypes.c_uint, _vp, _vp, _vp, _vp],
    "ps_ref_cost_terms": [_c_int, _vp, _c_int, _c_int, _c_int] + _REF_ARM + [_c_int, _vp, _vp, _vp, _vp,
                                                                          _vp],
    "ps_ref_optimize": [_c_int, _vp, _c_int, _c_int, _c_int, _c_int, _c_d, _c_d, _c_d, _c_int, _c_d, _c_d]
                       + _REF_ARM + [_vp, _vp, _vp, _vp, _vp, _vp],
    "ps_ref_planner_esdf": [_vp, _c_int, _c_d, _c_d, _c_d, _c_d, _c_d, _c_d, _c_d, _c_d, _c_d, _c_d, _c_int,
                            _c_int, _vp, _vp],
    "ps_ref_render_scan": [_vp, _c_int, _vp, _c_int, _c_d, _c_d, _c_d, _c_d, _c_int, _c_d, _vp, _vp],
    "ps_ref_planner_success": [_vp, _c_int, _c_int, _c_int] + _REF_ARM + [_c_d, _c_d, _c_int, _vp, _vp],
    "ps_ref_select": [_vp, _vp, _c_int, _c_int, _vp, _vp],
    "ps_ref_linear": [_vp, _c_int, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _vp],
    "ps_ref_film": [_vp, _vp, _vp, _c_int, _c_int, _vp],
    "ps_ref_conv1d_silu": [_vp, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _c_int, _vp, _vp],
    "ps_ref_sinusoid": [_c_d, _c_int, _vp, _vp],
    "ps_ref_div": [_vp, _c_int, _c_d, _vp, _vp],
    "ps_ref_ddim_update": [_vp, _vp, _c_int, _c_d, _c_d, _c_int, _c_d, _c_d, _vp, _vp],
    "ps_ref_ddim_next": [_vp, _vp, _vp, _c_int, _c_d, _vp],
    "ps_ref_guide": [_c_int, _vp, _c_int, _c_int, _c_int] + _REF_ARM + [_vp, _vp, _vp, _c_int, _c_d, _c_int, _vp,
                                                                     _vp, _vp],
    "ps_ref_metrics": [_vp, _c_int, _c_int, _c_int, _vp, _c_d, _c_d, _vp, _c_int, _vp, _c_int, _vp, _c_int, _c_d,
                       _c_d, _c_d, _c_d, _vp, _vp, _vp, _vp, _c_int, _vp, _vp],
    "ps_ref_denorm_pin": [_vp, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp],
    "ps_ref_linear_dt": [_c_int, _vp, _c_int, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _vp],
    "ps_ref_film_dt": [_c_int, _vp, _vp, _vp, _c_int, _c_int, _vp],
    "ps_ref_conv1d_silu_dt": [_c_int, _vp, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _c_int, _vp, _vp],
    "ps_ref_sinusoid_dt": [_c_int, _c_d, _c_int, _vp, _vp],
    "ps_ref_div_dt": [_c_int, _vp, _c_int, _c_d, _vp, _vp],
    "ps_ref_ddim_update_dt": [_c_int, _vp, _vp, _c_int, _c_d, _c_d, _c_int, _c_d, _c_d, _vp, _vp],
    "ps_ref_denorm_pin_dt": [_c_int, _vp, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp],
    "ps_train_gemm": [_vp, _c_int, _c_int, _vp, _c_int, _c_int, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp],
    "ps_train_bias_act": [_vp, _c_int, _vp, _c_int, _c_int, _c_int, _vp, _vp],
    "ps_train_silu_bwd": [_vp, _c_int, _vp, _c_int, _c_int, _vp],
    "ps_train_colsum": [_vp, _c_int, _c_int, _c_int, _vp, _c_int, _vp],
    "ps_train_film": [_vp, _vp, _vp, _c_int, _vp, _vp],
    "ps_train_film_bwd": [_vp, _vp, _vp, _c_int, _vp, _vp, _vp],
    "ps_train_conv1d": [_vp, _c_int, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _c_int, _vp, _vp, _vp],
    "ps_train_conv1d_bwd": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp],
    "ps_train_fk_loss": [_vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _c_d, _c_d, _c_d, _vp, _vp,
                         _vp, _vp],
    "ps_train_adam": [_vp, _vp, _vp, _vp, _c_ll, _c_d, _c_d, _c_d, _c_d, _c_d, _c_d, _vp],
    "ps_encoder_packed_bytes": [_c_int, _c_int, _c_int],
    "ps_encoder_pack": [_vp, _c_int, _c_int, _c_int, _vp, _vp],
    "ps_encode_tc_workspace_bytes": [_c_int, _c_int, _c_int, _c_int],
    "ps_encode_tc": [_vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _vp, _vp, _c_f, _c_f, _vp, _vp,
                     _vp],
}
_RESTYPE = {"ps_version": ctypes.c_char_p, "ps_launch_count": _c_ll, "ps_unet_param_count": _c_ll,
            "ps_unet_param_offset": _c_ll, "ps_unet_packed_bytes": _c_ll,
            "ps_encode_workspace_bytes": _c_ll, "ps_sample_workspace_bytes": _c_ll,
            "ps_encoder_packed_bytes": _c_ll, "ps_encode_tc_workspace_bytes": _c_ll}

_lib = None


class PSError(RuntimeError):
    pass


def lib():
    """Load (never build) the in-tree library; fail loudly if it is absent."""
    global _lib
    if _lib is None:
        path = _build.LIB
        if not path.exists():
            raise PSError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback)")
        import os
        alt = os.environ.get("PS_LIB_OVERRIDE")   # A/B timing of an alternative build (tools only)
        L = ctypes.CDLL(alt if alt else str(path))
        for name, args in _SIGS.items():
            if alt and not hasattr(L, name):   # an older build under A/B: bind what it has
                continue
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, ctypes.c_int)
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(status: int, what: str):
    if status == PS_OK:
        return
    if status == PS_ERR_OUT_OF_GRID:
        raise ValueError(f"{what}: trajectory collision points leave the ESDF extent")
    if status == PS_ERR_SHAPE:
        raise ValueError(f"{what}: bad shape or argument")
    raise PSError(f"{what}: CUDA error (status {status})")


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise PSError("no CUDA device visible: the B200 path has no CPU fallback")
    return torch


def ptr(t) -> int:
    return t.data_ptr()


def hptr(a: np.ndarray) -> int:
    return a.ctypes.data


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
