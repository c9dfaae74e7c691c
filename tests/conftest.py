import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REF_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libps_b200.so")
    config.addinivalue_line("markers", "reference: needs the planseed reference importable")


def have_reference() -> bool:
    return (REF_SRC / "planseed").exists()


@pytest.fixture(scope="session")
def planseed():
    if not have_reference():
        pytest.skip("planseed reference not present (GPU box)")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import planseed as ps
    return ps


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    oracle.build()
    return oracle
