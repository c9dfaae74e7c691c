"""ORACLE -- test infrastructure, never product code.

CPU restatements of the reference hot path, used only by tests/, by
__graft_entry__.smoke() and by bench.py's CPU legs (cpu_baseline and
--impl reference) as the checker / CPU baseline.  The product package
(paper_2410_16727_b200) never imports this package.

  oracle/c/bl_oracle.c   canonical-fp32 C restatement of the BASELINE-profile
                         refinement (bit-exact target for the CUDA kernels)
  oracle/bl_numpy.py     independent float64 numpy restatement of the same
  oracle/unet_numpy.py   encoder / U-Net / DDPM restatement (BASELINE profile)
  oracle/pipeline_cpu.py the BASELINE planning pipeline on host cores (CPU baseline)

The ref profile (planseed's own planar / FC / DDIM / Armijo path) needs no
restatement: its oracle is planseed itself (imported from /root/reference when
present) and the golden fixtures in tests/golden/ generated from planseed by
tools/make_golden.py.  The BASELINE restatements are pinned to torch.nn.functional
and to planseed by tests/test_unet_oracle_cpu.py and tests/test_bl_oracle.py.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
BUILD = HERE / "_build"
LIB = BUILD / "liboracle.so"
SOURCES = [HERE / "c" / "bl_oracle.c"]


def build(force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    newest = max(s.stat().st_mtime for s in SOURCES)
    if LIB.exists() and not force and LIB.stat().st_mtime >= newest:
        return LIB
    cmd = ["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
           "-std=c11", "-o", str(LIB)] + [str(s) for s in SOURCES] + ["-lm"]
    subprocess.run(cmd, check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = ctypes.CDLL(str(LIB))
    return _lib


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class BLProblemSet:
    """Host-side bundle of what the BL refine oracle needs."""

    def __init__(self, robot, grid, cost, esdf: np.ndarray, esdf_stride: int):
        self.robot, self.grid, self.cost = robot, grid, cost
        self.esdf = _f(esdf)
        self.esdf_stride = int(esdf_stride)
        self.dh = _f(robot.dh_table_f32())
        self.base = _f(robot.base)
        self.sph = _f(robot.sphere_table_f32())
        self.link = np.ascontiguousarray(robot.sphere_link, dtype=np.int32)
        self.n = np.array(grid.n, dtype=np.int32)
        self.origin = _f(grid.origin)
        self.w = _f(cost.as_f32())


def esdf_build(boxes: np.ndarray, grid) -> np.ndarray:
    boxes = _f(boxes)
    out = np.empty(grid.n, dtype=np.float32)
    n = np.array(grid.n, dtype=np.int32)
    lib().orc_esdf_build(_p(boxes), ctypes.c_int(boxes.shape[0]), _p(n), _p(_f(grid.origin)),
                         ctypes.c_float(grid.h), ctypes.c_float(grid.cap), _p(out))
    return out


def bl_cost(ps: BLProblemSet, q: np.ndarray, S: int):
    q = _f(q)
    B, T, _ = q.shape
    cost = np.empty(B, np.float32)
    grad = np.empty_like(q)
    cl = np.empty(B, np.int32)
    lib().orc_bl_cost(_p(q), B, T, S, _p(ps.esdf), ctypes.c_longlong(ps.esdf_stride), _p(ps.n),
                      _p(ps.origin), ctypes.c_float(ps.grid.h), _p(ps.dh), _p(ps.base), _p(ps.sph),
                      _p(ps.link), ctypes.c_int(len(ps.link)), _p(ps.w), _p(cost), _p(grad), _p(cl))
    return cost, grad, cl.astype(bool)


def bl_refine(ps: BLProblemSet, q: np.ndarray, S: int, n_iters: int):
    q = _f(q)
    B, T, _ = q.shape
    out = np.empty_like(q)
    cost = np.empty(B, np.float32)
    feas = np.empty(B, np.int32)
    cl = np.empty(B, np.int32)
    lib().orc_bl_refine(_p(q), B, T, S, _p(ps.esdf), ctypes.c_longlong(ps.esdf_stride), _p(ps.n),
                        _p(ps.origin), ctypes.c_float(ps.grid.h), _p(ps.dh), _p(ps.base),
                        _p(ps.sph), _p(ps.link), ctypes.c_int(len(ps.link)), _p(ps.w),
                        ctypes.c_int(n_iters), _p(out), _p(cost), _p(feas), _p(cl))
    return out, cost, feas.astype(bool), cl.astype(bool)


def bl_guide(ps: BLProblemSet, x0: np.ndarray, S: int, lo, span, n_grad: int, alpha: float,
             max_halvings: int):
    """guided_ddim_sample's guide() on normalised x0 (B,T,7) -> (guided x0, clamped flags)."""
    x = _f(x0).copy()
    B, T, _ = x.shape
    cl = np.empty(B, np.int32)
    lib().orc_bl_guide(_p(x), B, T, S, _p(ps.esdf), ctypes.c_longlong(ps.esdf_stride), _p(ps.n), _p(ps.origin),
                       ctypes.c_float(ps.grid.h), _p(ps.dh), _p(ps.base), _p(ps.sph), _p(ps.link),
                       ctypes.c_int(len(ps.link)), _p(ps.w), _p(_f(lo)), _p(_f(span)), ctypes.c_int(n_grad),
                       ctypes.c_float(alpha), ctypes.c_int(max_halvings), _p(cl))
    return x, cl.astype(bool)


def select(cost: np.ndarray, feasible: np.ndarray, S: int) -> np.ndarray:
    cost = _f(cost)
    feas = np.ascontiguousarray(feasible, dtype=np.int32)
    P = cost.shape[0] // S
    best = np.empty(P, np.int32)
    lib().orc_select(_p(cost), _p(feas), P, S, _p(best))
    return best


def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.empty(4, np.uint32)
    lib().orc_philox(_p(c), _p(k), _p(out))
    return out
