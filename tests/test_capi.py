"""The C-ABI library loads on CPU and exports every entry point include/mpm_capi.h declares; the
Python mirror binds exactly those; and without a GPU it refuses to run (no CPU fallback)."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_2507_04192_b200 import capi

HEADER = Path(__file__).resolve().parents[1] / "include" / "mpm_capi.h"


def declared():
    txt = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(mpm_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_expected_api():
    names = declared()
    for must in ("mpm_ctx_create", "mpm_advance", "mpm_step_vjp", "mpm_backprop", "mpm_state_upload",
                 "mpm_state_download", "mpm_p2g", "mpm_g2p", "mpm_grid_corrections"):
        assert must in names
    assert sorted(capi.exported_symbols()) == names


def test_library_exports_every_declared_symbol():
    if not capi.LIB_PATH.exists():
        pytest.fail("libmpm_b200.so is not built: run __graft_entry__.build()")
    lib = C.CDLL(str(capi.LIB_PATH))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.mpm_version() == 1


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2507_04192_b200.errors import DeviceError
    from paper_2507_04192_b200.presets import small_fluid_scene
    from paper_2507_04192_b200.solver import Context
    with pytest.raises(DeviceError):
        Context(small_fluid_scene(), 100)


def test_library_loads_before_torch():
    """NCCL is resolved at run time (dyn::api in context.cu): loading the library first must not pin
    an older system libnccl.so.2 that torch's own libtorch_cuda.so then fails to link against"""
    import subprocess
    import sys
    if not capi.LIB_PATH.exists():
        pytest.fail("libmpm_b200.so is not built: run __graft_entry__.build()")
    needed = subprocess.run(["readelf", "-d", str(capi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "libnccl" not in needed
    code = f"import ctypes; ctypes.CDLL({str(capi.LIB_PATH)!r}); import torch; print(torch.__version__)"
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
