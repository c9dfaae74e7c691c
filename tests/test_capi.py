"""CPU checks of the C-ABI library: it builds, loads and exports every symbol that
include/ps_b200.h declares (no compute calls without a GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "ps_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ps_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2410_16727_b200 import build
    return build.build(verbose=False)


def test_header_declares_entry_points():
    syms = header_symbols()
    assert "ps_bl_refine" in syms and "ps_select" in syms and len(syms) >= 5


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(str(libpath))
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_header(libpath):
    from paper_2410_16727_b200 import _lib
    assert set(header_symbols()) <= set(_lib.exported_symbols())


def test_version_string(libpath):
    from paper_2410_16727_b200 import _lib
    assert b"sm_100a" in _lib.lib().ps_version()


def test_sass_is_sm100a(libpath):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(libpath)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_unet_param_table_matches_spec(libpath):
    import numpy as np
    from paper_2410_16727_b200 import _lib, spec
    L = _lib.lib()
    arch = spec.UNetArch()
    assert L.ps_unet_param_count() == arch.n_params()
    off = 0
    for name, shape in arch.param_shapes():
        assert L.ps_unet_param_offset(name.encode()) == off, name
        off += int(np.prod(shape))
    assert L.ps_unet_param_offset(b"nope") == -1


def test_packed_sizes(libpath):
    from paper_2410_16727_b200 import _lib
    L = _lib.lib()
    assert L.ps_unet_packed_bytes(0) > 4 * 5_000_000
    assert L.ps_unet_packed_bytes(1) > 2 * 5_000_000
    assert L.ps_unet_packed_bytes(7) == -1
