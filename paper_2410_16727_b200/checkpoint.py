"""PSCK checkpoints for the BASELINE-profile model (depth encoder + 1-D temporal U-Net).

Same container as planseed's save_checkpoint / load_checkpoint (diffusion.py:635-687): the 4-byte
magic b"PSCK", a little-endian u64 header length, a sorted-key JSON header (format, arch,
init_seed, schedule betas, meta, params [{name, shape}]) and the little-endian float64 parameter
blob in table order.  The header's arch carries kind = "unet1d" plus the pinned architecture
(spec.UNetArch / spec.EncoderArch), so a trained U-Net reaches the GPU through the reference's
weight format; the parameter table order is spec.model_param_shapes (encoder, then U-Net).

Errors follow the reference loader: FileNotFoundError for a missing file, ValueError for a wrong
magic or a blob-size mismatch; additionally ValueError for a header whose arch is not a unet1d this
build can run (e.g. a planseed FC-denoiser checkpoint -- load that with ref.load_checkpoint) or
whose parameter table disagrees with the architecture.
"""

from __future__ import annotations

import json
import struct
from pathlib import Path
from typing import Optional, Tuple

import numpy as np

from . import spec

CKPT_MAGIC = b"PSCK"
ARCH_KIND = "unet1d"


def arch_header(enc: spec.EncoderArch, arch: spec.UNetArch) -> dict:
    return {"kind": ARCH_KIND, "dof": arch.dof, "dims": list(arch.dims), "cond_dim": arch.cond_dim,
            "ksize": spec.KSIZE, "gn_groups": spec.GN_GROUPS, "gn_eps": spec.GN_EPS, "t_emb": spec.T_EMB,
            "t_hidden": spec.T_HIDDEN, "encoder_channels": list(enc.channels),
            "encoder_in_channels": enc.in_channels, "x0_clip": list(spec.X0_CLIP),
            "joint_lo": [-spec.JOINT_LIMIT] * arch.dof, "joint_hi": [spec.JOINT_LIMIT] * arch.dof}


def save_checkpoint(path, params: dict, enc: spec.EncoderArch = spec.ENCODER_CFG3,
                    arch: spec.UNetArch = spec.UNetArch(), betas: Optional[np.ndarray] = None,
                    meta: Optional[dict] = None, init_seed: int = spec.WEIGHT_SEED) -> None:
    """Write `params` (name -> array, spec.model_param_shapes(enc, arch) names) as a PSCK file."""
    shapes = spec.model_param_shapes(enc, arch)
    for n, sh in shapes:
        if n not in params:
            raise ValueError(f"missing parameter {n}")
        if tuple(np.shape(params[n])) != tuple(sh):
            raise ValueError(f"parameter {n} has shape {np.shape(params[n])}, expected {sh}")
    betas = spec.cosine_betas() if betas is None else np.asarray(betas, dtype=np.float64)
    header = {"format": 1, "arch": arch_header(enc, arch), "init_seed": int(init_seed),
              "schedule": {"betas": [float(x) for x in betas.ravel()]}, "meta": meta or {},
              "params": [{"name": n, "shape": list(sh)} for n, sh in shapes]}
    blob = b"".join(np.ascontiguousarray(params[n], dtype="<f8").tobytes() for n, _ in shapes)
    head = json.dumps(header, sort_keys=True).encode()
    with open(path, "wb") as f:
        f.write(CKPT_MAGIC)
        f.write(struct.pack("<Q", len(head)))
        f.write(head)
        f.write(blob)


def read_header(path) -> Tuple[dict, bytes]:
    path = Path(path)
    if not path.exists():
        raise FileNotFoundError(f"checkpoint not found: {path}")
    with open(path, "rb") as f:
        if f.read(4) != CKPT_MAGIC:
            raise ValueError(f"{path} is not a checkpoint file")
        (hlen,) = struct.unpack("<Q", f.read(8))
        header = json.loads(f.read(hlen).decode())
        blob = f.read()
    return header, blob


def load_checkpoint(path):
    """-> (params dict of float64 arrays, EncoderArch, UNetArch, betas, meta)."""
    header, blob = read_header(path)
    a = header.get("arch", {})
    if a.get("kind") != ARCH_KIND:
        raise ValueError(f"{path}: arch kind {a.get('kind', 'fc (planseed)')!r} is not {ARCH_KIND!r}; "
                         "planseed FC-denoiser checkpoints load with ref.load_checkpoint")
    enc = spec.EncoderArch(channels=tuple(a["encoder_channels"]), in_channels=int(a["encoder_in_channels"]))
    arch = spec.UNetArch(dof=int(a["dof"]), dims=tuple(a["dims"]), cond_dim=int(a["cond_dim"]))
    want = arch_header(enc, arch)
    for k in ("ksize", "gn_groups", "gn_eps", "t_emb", "t_hidden", "x0_clip"):
        if a.get(k) != want[k]:
            raise ValueError(f"{path}: arch field {k}={a.get(k)!r} is not supported (this build: {want[k]!r})")
    shapes = spec.model_param_shapes(enc, arch)
    listed = [(p["name"], tuple(p["shape"])) for p in header["params"]]
    if listed != [(n, tuple(sh)) for n, sh in shapes]:
        raise ValueError(f"{path}: parameter table does not match the unet1d architecture")
    params, off = {}, 0
    for name, shape in listed:
        n = int(np.prod(shape))
        if off + 8 * n > len(blob):
            raise ValueError(f"checkpoint blob size mismatch in {path}")
        params[name] = np.frombuffer(blob, dtype="<f8", count=n, offset=off).reshape(shape).copy()
        off += n * 8
    if off != len(blob):
        raise ValueError(f"checkpoint blob size mismatch in {path}")
    return params, enc, arch, np.array(header["schedule"]["betas"], dtype=np.float64), header.get("meta", {})
