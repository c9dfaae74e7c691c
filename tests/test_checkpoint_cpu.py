"""PSCK checkpoints of the BASELINE U-Net (paper_2410_16727_b200/checkpoint.py): the container of
planseed's save/load_checkpoint (diffusion.py:635-687) with arch kind "unet1d"."""

import json
import struct

import numpy as np
import pytest

from paper_2410_16727_b200 import checkpoint as ck
from paper_2410_16727_b200 import spec


def test_round_trip_bitwise(tmp_path):
    params = spec.random_model(spec.ENCODER_CFG3)
    betas = spec.cosine_betas()
    p = tmp_path / "unet.psck"
    ck.save_checkpoint(p, params, spec.ENCODER_CFG3, spec.UNetArch(), betas, meta={"step": 7})
    got, enc, arch, b2, meta = ck.load_checkpoint(p)
    assert enc == spec.ENCODER_CFG3 and arch == spec.UNetArch() and meta == {"step": 7}
    assert np.array_equal(b2, betas)
    assert set(got) == set(params)
    for n in params:
        assert np.array_equal(got[n], params[n]) and got[n].dtype == np.float64


def test_container_matches_reference_layout(tmp_path):
    # magic, <Q header length, sorted-key JSON, <f8 blob in table order
    params = spec.random_model()
    p = tmp_path / "u.psck"
    ck.save_checkpoint(p, params, spec.ENCODER_CFG0)
    raw = p.read_bytes()
    assert raw[:4] == b"PSCK"
    (hlen,) = struct.unpack("<Q", raw[4:12])
    header = json.loads(raw[12:12 + hlen])
    assert raw[12:12 + hlen].decode() == json.dumps(header, sort_keys=True)
    names = [n for n, _ in spec.model_param_shapes(spec.ENCODER_CFG0)]
    assert [q["name"] for q in header["params"]] == names
    blob = np.frombuffer(raw[12 + hlen:], dtype="<f8")
    assert blob.size == sum(params[n].size for n in names)
    assert np.array_equal(blob[:params[names[0]].size], params[names[0]].ravel())


def test_errors(tmp_path):
    with pytest.raises(FileNotFoundError):
        ck.load_checkpoint(tmp_path / "missing.psck")
    bad = tmp_path / "bad.psck"
    bad.write_bytes(b"NOPE" + b"\0" * 16)
    with pytest.raises(ValueError, match="not a checkpoint"):
        ck.load_checkpoint(bad)
    p = tmp_path / "t.psck"
    ck.save_checkpoint(p, spec.random_model(), spec.ENCODER_CFG0)
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(ValueError, match="size mismatch"):
        ck.load_checkpoint(p)
    with pytest.raises(ValueError, match="shape"):
        prm = spec.random_model()
        prm["out_b"] = np.zeros(3)
        ck.save_checkpoint(tmp_path / "s.psck", prm, spec.ENCODER_CFG0)


def test_planseed_checkpoint_is_rejected_with_pointer(tmp_path):
    from paper_2410_16727_b200.ref import diffusion as rd
    net = rd.create_net(rd.ArchConfig(), seed=0)
    p = tmp_path / "fc.psck"
    rd.save_checkpoint(p, net, rd.make_schedule())
    with pytest.raises(ValueError, match="unet1d"):
        ck.load_checkpoint(p)
