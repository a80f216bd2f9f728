"""bench.py's roofline helpers (CPU): the FP64 denominator is the measured ceiling when
profiles/fp64_peak.json is committed, and the per-kernel fractions divide by it."""
import json
import sys
from pathlib import Path
from types import SimpleNamespace

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def test_fp64_roofline_uses_measured_ceiling():
    a = SimpleNamespace(config="C4", dtype="f64")
    prof = {"k_p2g": {"ms_per_launch": 0.5}, "k_g2p": {"ms_per_launch": 0.35}}
    out = bench.fp64_for(prof, a)
    assert out is not None
    meas = json.loads((ROOT / "profiles" / "fp64_peak.json").read_text())
    assert out["peak_tflops"] == meas["fp64_tflops"]
    assert "measured" in out["peak_source"]
    ref = json.loads((ROOT / "profiles" / "fp64.json").read_text())
    tf = ref["k_p2g"]["fp64_flops"] / 0.5e-3 / 1e12
    assert abs(out["k_p2g"]["achieved"] - tf) < 1e-9
    assert abs(out["k_p2g"]["frac"] - tf / meas["fp64_tflops"]) < 1e-12


def test_fp64_roofline_only_for_c4_f64():
    prof = {"k_p2g": {"ms_per_launch": 0.5}}
    assert bench.fp64_for(prof, SimpleNamespace(config="C3", dtype="f64")) is None
    assert bench.fp64_for(prof, SimpleNamespace(config="C4", dtype="f32")) is None
