"""Parity on BASELINE.json's own configs: the benched scenes themselves, not
small stand-ins, through the C ABI against the CPU oracle (bit-identical to the reference compiled
unmodified, tests/test_oracle_vs_ref.py) and against a golden fixture made by the reference.

Tolerances (SURVEY §8(c) parity policy, f64):
  * C4 / C2 / reduced C5 forward, 2-20 steps: every particle field <= 1e-10 relative to its scale;
  * C1, all 1000 steps: x and v <= 1e-9; sigma <= 1e-8 (relative Frobenius) over the particles
    whose Drucker-Prager zone (constitutive.hpp:62-70, classified from the final stress) matches,
    and at least 99.5 % of particles zone-matched;
  * reduced C5 step_vjp (32 Coulomb segments): x / v cotangents and the 32 friction gradients
    <= 1e-9;
  * C3 1000-step inverse gradient (n_seg = 10) against tests/golden/c3_gradient.npz: loss and
    dL/dalpha <= 1e-7 relative, vbar(0) <= 1e-6 of its norm (1000 steps of roundoff growth through a
    chaotic free-surface flow; the fixture is the reference's own backprop_trajectory).
"""
import math
from pathlib import Path

import numpy as np
import pytest

from helpers import FLOORS, assert_state_close, rel_err
from paper_2507_04192_b200 import ParamGrads, StateCotangent, init_scene
from paper_2507_04192_b200.presets import c1_column, c2_dam_break, c3_inverse, c4_column3d, c5_landslide_eighth
from paper_2507_04192_b200.solver import Context

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"


def gpu_advance(s, st, n, guard=True):
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.advance(n, nan_guard=guard)
    out = ctx.download(st.copy())
    ctx.close()
    return out


def dp_zone(scene, sig, szz=None):
    """Which Drucker-Prager surfaces a returned stress sits on (constitutive.hpp:72-83
    invariants): bit 0 = on the shear surface (f_s within roundoff of 0), bit 1 = on the tension
    cap (f_t within roundoff of 0). A returned stress is feasible (f_s <= 0, f_t <= 0), so the
    label separates elastic particles from ones the last return map put on a surface."""
    m = scene.material
    d = sig.shape[-1]
    if d == 2:
        s3 = np.zeros(sig.shape[:-2] + (3, 3))
        s3[..., :2, :2] = sig
        s3[..., 2, 2] = szz
    else:
        s3 = sig
    sm = np.trace(s3, axis1=-2, axis2=-1) / 3.0
    dev = s3 - sm[..., None, None] * np.eye(3)
    tau = np.sqrt(0.5 * np.einsum("...ij,...ij->...", dev, dev))
    fs = tau - m.k_phi + m.q_phi * sm
    ft = sm - m.sigma_t
    tol = 1e-9 * (np.abs(s3).max(axis=(-2, -1)) + abs(m.k_phi) + 1.0)
    return (fs > -tol).astype(np.int8) + 2 * (ft > -tol).astype(np.int8)


def test_c4_full_scene_two_steps(orc):
    """C4 (4,194,304 particles, 256^3 cells, D-P, f64): the headline bench scene, 2 steps."""
    s = c4_column3d("f64")
    st = init_scene(s)
    assert st.particles.size() == 4_194_304
    got = gpu_advance(s, st, 2)
    want = orc.advance(s, st.copy(), 2)
    assert got.step == want.step == 2
    assert_state_close(got, want, 1e-10, what="C4x2")


def test_c2_twenty_steps(orc):
    """C2 (250,000-particle dam break, 512^2, fluid c 35, f64), 20 steps."""
    s = c2_dam_break("f64")
    st = init_scene(s)
    assert st.particles.size() == 250_000
    got = gpu_advance(s, st, 20)
    want = orc.advance(s, st.copy(), 20)
    assert_state_close(got, want, 1e-10, what="C2x20")


@pytest.mark.slow
def test_c1_all_1000_steps(orc):
    """C1 (20,000-particle Bui column, D-P, f64) through its whole 1000-step horizon."""
    s = c1_column("f64")
    st = init_scene(s)
    got = gpu_advance(s, st, 1000)
    want = orc.advance(s, st.copy(), 1000)
    p, q = got.particles, want.particles
    assert rel_err(p.x, q.x, FLOORS["x"]) <= 1e-9
    assert rel_err(p.v, q.v, FLOORS["v"]) <= 1e-9
    zg = dp_zone(s, p.sigma, p.sigma_zz)
    zw = dp_zone(s, q.sigma, q.sigma_zz)
    match = zg == zw
    assert match.mean() >= 0.995, f"zone match {match.mean():.4f}"
    scale = max(float(np.linalg.norm(q.sigma, axis=(1, 2)).max()), FLOORS["sigma"])
    err = np.linalg.norm(p.sigma - q.sigma, axis=(1, 2))[match].max() / scale
    assert err <= 1e-8, err
    assert np.array_equal(p.mass, q.mass)


def test_c5_reduced_forward_and_step_vjp(orc):
    """Reduced C5 (4,063,232 particles, 32 Coulomb friction segments): 2 forward steps, then one
    step_vjp with a random x / v cotangent; the friction gradients (adjoint.hpp:145) included."""
    s = c5_landslide_eighth()
    st = init_scene(s)
    assert st.particles.size() == 256 * 64 * 31 * 8
    got = gpu_advance(s, st, 2)
    want = orc.advance(s, st.copy(), 2)
    assert_state_close(got, want, 1e-10, what="C5/8x2")
    rng = np.random.default_rng(32)
    cot = StateCotangent.zeros_like(want.particles)
    cot.x[...] = rng.standard_normal(cot.x.shape)
    cot.v[...] = rng.standard_normal(cot.v.shape)
    ctx = Context(s, want.particles.size())
    gi = ctx.step_vjp(want, cot, pg_g := ParamGrads(s.boundary))
    ctx.close()
    ri, pg_r = orc.step_vjp(s, want, cot)
    for f in ("x", "v", "rho", "volume"):
        a, b = getattr(gi, f), getattr(ri, f)
        assert rel_err(a, b) <= 1e-9, (f, rel_err(a, b))
    fg, fr = pg_g.wall_friction[2], pg_r.wall_friction[2]
    assert len(fg) == 32 and np.abs(fr).max() > 0
    assert np.abs(fg - fr).max() <= 1e-9 * np.abs(fr).max(), (fg, fr)


def test_c3_inverse_gradient_matches_reference_golden():
    """C3 (102,400 particles, 1000 steps, n_seg = 10): the paper's inverse problem, loss on the
    final deposit of an alpha* = 2 twin, against the reference's own backprop_trajectory
    (tests/golden/make_c3_gradient.py)."""
    g = np.load(GOLDEN / "c3_gradient.npz")
    n_steps, nseg, stride = int(g["n_steps"]), int(g["n_segments"]), int(g["stride"])
    twin = c3_inverse(alpha=2.0)
    stt = init_scene(twin)
    ct = Context(twin, stt.particles.size())
    ct.upload(stt)
    ct.advance(n_steps)
    target = ct.download(stt.copy()).particles.x[None].copy()
    ct.close()
    assert rel_err(target[0, ::stride], g["target_sub"], 1.0) <= 1e-9
    s = c3_inverse(alpha=0.1)
    st0 = init_scene(s)
    assert st0.particles.size() == int(g["n_particles"])
    ctx = Context(s, st0.particles.size())
    c0, pg, res = ctx.backprop(st0, n_steps, nseg, {"field": "x", "obs_steps": [n_steps], "sel": None,
                                                    "target": target})
    ctx.close()
    alpha = s.geometry[0].velocity.alpha
    dl = float(np.sum(c0.v[:, 0] * st0.particles.v[:, 0]) / alpha)
    assert abs(res.loss - float(g["loss"])) <= 1e-7 * abs(float(g["loss"]))
    assert abs(dl - float(g["dL_dalpha"])) <= 1e-7 * abs(float(g["dL_dalpha"])), (dl, float(g["dL_dalpha"]))
    assert np.abs(c0.v[::stride] - g["vbar0_sub"]).max() <= 1e-6 * float(g["vbar0_norm"])
    assert np.abs(c0.x[::stride] - g["xbar0_sub"]).max() <= 1e-6 * float(g["xbar0_norm"])
