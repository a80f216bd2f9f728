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


def test_kernel_roofline_uses_survey_compulsory_bytes():
    """k_p2g is scored on SURVEY 8(d)'s compulsory bytes (x v m V sigma read once, the
    active nodes' m p f written once): 14 x 8 B x 4,194,304 + 588,060 x 7 x 8 B = 502.7 MB at C4,
    not the 580 MB the implementation moves (perm / keys, (B+2)^3 tiles)."""
    from paper_2507_04192_b200.presets import c4_column3d
    s = c4_column3d()
    alg, need, moved = bench.kernel_bytes(s, 4_194_304, 588_060, 1_000)
    assert abs(alg["k_p2g"] - (14 * 8 * 4_194_304 + 588_060 * 7 * 8)) < 1
    assert abs(alg["k_p2g"] / 1e6 - 502.7) < 0.1
    assert moved["k_p2g"] > alg["k_p2g"]
    # g2p: reads x v V rho sigma eps, writes the same + grad v; needed drops grad v (FLIP)
    assert alg["k_g2p"] - need["k_g2p"] == 9 * 8 * 4_194_304


def test_fwd_adj_bytes_count_passes_executed():
    """with one segment nothing is replayed: B = 1 x B_fwd + B_vjp, not 2 x B_fwd + B_vjp."""
    from paper_2507_04192_b200.presets import c4_column3d
    s = c4_column3d()
    n = 4_194_304
    B_fwd, IN, _ = bench.bytes_model(s, n, 588_060)
    two = bench.vjp_bytes(s, n, 588_060, B_fwd, IN)
    one = bench.vjp_bytes(s, n, 588_060, B_fwd, IN, 1.0)
    assert abs(two - one - B_fwd) < 1e-9
