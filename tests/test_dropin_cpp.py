"""C++ drop-in layer on the GPU:
* the reference's own tests/test_stepper.cpp, compiled UNMODIFIED against include/mpm_gpu/mpm/stepper.hpp
  (its Stepper / run / RunResult run on the B200), must pass;
* tests/cpp/test_dropin.cpp compares mpm::gpu:: with the reference's CPU functions in one binary."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BUILD = Path(__file__).resolve().parent / "_build"


@pytest.mark.parametrize("exe", ["test_stepper_gpu", "test_dropin"])
def test_cpp_dropin(exe):
    p = BUILD / exe
    if not p.exists():
        pytest.skip(f"{p} not built (needs /root/reference at build time)")
    out = subprocess.run([str(p)], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-2000:]
    assert "failed: 0" in out.stdout
