"""The reference's own unit tests (proj/tests/*.cpp), compiled unmodified against the Eigen and
doctest shims (oracle/Makefile), must pass: this validates the shims the oracle stands on."""
import subprocess
from pathlib import Path

import pytest

REF = Path(__file__).resolve().parents[1] / "oracle" / "_ref"
TESTS = ["test_bspline", "test_scene", "test_transfer", "test_constitutive", "test_contact", "test_stepper"]


@pytest.mark.parametrize("name", TESTS)
def test_reference_unit_tests_pass(name):
    exe = REF / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (needs /root/reference)")
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:]
    assert "failed: 0" in out.stdout
