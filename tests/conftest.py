import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 (B200) GPU and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def orc():
    from oracle import CpuOracle
    return CpuOracle("orc")


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.available("ref"):
        pytest.skip("reference library oracle/_ref/libmpm_ref.so not built (needs /root/reference)")
    return oracle.CpuOracle("ref")
