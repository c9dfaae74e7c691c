"""The binding a planseed maintainer would drop in as planseed/_kernels_b200.py
(INTEGRATION.md §2): numba-compatible signatures of cost_terms_batch / optimize_batch
(src/_kernels.py:165-176, :315-324) over libps_b200.so via ctypes."""

import ctypes
from pathlib import Path

import numpy as np
import torch

_LIB = Path(__file__).resolve().parents[1] / "paper_2410_16727_b200" / "_build" / "libps_b200.so"
_L = ctypes.CDLL(str(_LIB))
d, i, p = ctypes.c_double, ctypes.c_int, ctypes.c_void_p
ARM = [p, d, d, p, i, p, p, i, p, i, i, d, d, d, d, d, d, p, d, d, p, p]   # PS_REF_ARM_ARGS
_L.ps_ref_cost_terms.argtypes = [i, p, i, i, i] + ARM + [i, p, p, p, p, p]
_L.ps_ref_optimize.argtypes = [i, p, i, i, i, i, d, d, d, i, d, d] + ARM + [p, p, p, p, p, p]


def _dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def _arm(lengths, basex, basey, fracs, pair_a, pair_b, grid_values, grid_ox, grid_oy, grid_h, goal_x,
         goal_y, goal_th, weights, d_act, d_self, jerk_mat, jerk_quad):
    keep = [np.ascontiguousarray(x) for x in (np.asarray(lengths, np.float64), np.asarray(fracs, np.float64),
                                               np.asarray(pair_a, np.int64), np.asarray(pair_b, np.int64),
                                               np.asarray(weights, np.float64))]
    g, jm, jq = _dev(grid_values), _dev(jerk_mat), _dev(jerk_quad)
    args = [keep[0].ctypes.data, basex, basey, keep[1].ctypes.data, len(keep[1]), keep[2].ctypes.data,
            keep[3].ctypes.data, len(keep[2]), g.data_ptr(), g.shape[0], g.shape[1], grid_ox, grid_oy,
            grid_h, goal_x, goal_y, goal_th, keep[4].ctypes.data, d_act, d_self, jm.data_ptr(),
            jq.data_ptr()]
    return args, (keep, g, jm, jq)


def cost_terms_batch(qs, *arm_and_want_grad):
    *arm, want_grad = arm_and_want_grad
    q = _dev(qs)
    S, T, D = q.shape
    args, keep = _arm(*arm)
    f64 = dict(dtype=torch.float64, device="cuda")
    terms, totals = torch.empty((S, 5), **f64), torch.empty(S, **f64)
    grads, clamped = torch.empty_like(q), torch.empty(S, dtype=torch.uint8, device="cuda")
    st = _L.ps_ref_cost_terms(0, q.data_ptr(), S, T, D, *args, int(want_grad), terms.data_ptr(),
                              totals.data_ptr(), grads.data_ptr(), clamped.data_ptr(),
                              torch.cuda.current_stream().cuda_stream)
    if st:
        raise RuntimeError(f"ps_ref_cost_terms status {st}")
    return (terms.cpu().numpy(), totals.cpu().numpy(), grads.cpu().numpy(),
            clamped.cpu().numpy().astype(bool))


def optimize_batch(seeds, n_iters, momentum, armijo_c, shrink, max_backtracks, alpha0, alpha_max, *arm):
    q = _dev(seeds)
    S, T, D = q.shape
    args, keep = _arm(*arm)
    f64 = dict(dtype=torch.float64, device="cuda")
    x, terms, totals = torch.empty_like(q), torch.empty((S, 5), **f64), torch.empty(S, **f64)
    frozen = torch.empty(S, dtype=torch.uint8, device="cuda")
    nacc = torch.empty(S, dtype=torch.int64, device="cuda")
    st = _L.ps_ref_optimize(0, q.data_ptr(), S, T, D, int(n_iters), momentum, armijo_c, shrink,
                            int(max_backtracks), alpha0, alpha_max, *args, x.data_ptr(), terms.data_ptr(),
                            totals.data_ptr(), frozen.data_ptr(), nacc.data_ptr(),
                            torch.cuda.current_stream().cuda_stream)
    if st:
        raise RuntimeError(f"ps_ref_optimize status {st}")
    return (x.cpu().numpy(), terms.cpu().numpy(), totals.cpu().numpy(), frozen.cpu().numpy().astype(bool),
            nacc.cpu().numpy())
