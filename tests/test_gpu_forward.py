"""GPU forward parity: the CUDA path (through the C ABI) against the CPU oracle on the same inputs.

Tolerances: f64 per phase / per step <= 1e-12 relative to the field's scale
(FLOORS in helpers.py give the physical scale of fields that are pure roundoff); f64 after
N <= 200 steps <= 1e-9; f32 <= 1e-4. Summation order differs from the reference's
particle-index order (cell-sorted, deterministic) and nvcc contracts FMAs, so agreement is at
rounding level, not bitwise.
"""
import math

import numpy as np
import pytest

from helpers import (assert_grid_close, assert_state_close, dp_block_scene, fluid_box_scene, random_block, rel_err,
                     single_particle_state)
from paper_2507_04192_b200 import GeometryRegion, Obstacle, SimState, VelocityExpr, Wall, init_scene
from paper_2507_04192_b200.errors import NumericalError, OutOfDomainError, ValidationError
from paper_2507_04192_b200.presets import bui_sand, c1_column, small_fluid_scene
from paper_2507_04192_b200.solver import Context, Stepper, run

pytestmark = pytest.mark.gpu

PHASE_RTOL = {"f64": 1e-12, "f32": 2e-5}
STEP_RTOL = {"f64": 1e-9, "f32": 1e-3}

SCENES = {
    "fluid2-pic": lambda d: fluid_box_scene(2, d, kind="pic"),
    "fluid2-flip": lambda d: fluid_box_scene(2, d, kind="flip"),
    "fluid2-blend": lambda d: fluid_box_scene(2, d, kind="blend", alpha=0.3),
    "fluid2-apic": lambda d: fluid_box_scene(2, d, kind="apic"),
    "fluid2-tpic-visc": lambda d: fluid_box_scene(2, d, kind="tpic", visc=0.5, rate_form=True),
    "dp2-noslip": lambda d: dp_block_scene(2, d),
    "dp2-coulomb-obstacle": lambda d: dp_block_scene(2, d, coulomb=True, obstacle=True),
    "dp3": lambda d: dp_block_scene(3, d, cells=[12, 12, 12]),
    "dp3-coulomb-obstacle": lambda d: dp_block_scene(3, d, coulomb=True, obstacle=True, cells=[16, 12, 12]),
    "fluid3-apic": lambda d: fluid_box_scene(3, d, kind="apic"),
    "fluid3-flip": lambda d: fluid_box_scene(3, d, kind="flip"),
}


def gpu_run(s, st, n, guard=True):
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.advance(n, nan_guard=guard)
    out = ctx.download(st.copy())
    ctx.close()
    return out


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("name", sorted(SCENES))
def test_n_step_parity(orc, name, dtype):
    s = SCENES[name](dtype)
    st = init_scene(s)
    want = orc.advance(s, st.copy(), 20)
    got = gpu_run(s, st, 20)
    assert got.step == 20 and got.time == pytest.approx(want.time)
    assert_state_close(got, want, STEP_RTOL[dtype], what=name)


@pytest.mark.parametrize("name", ["fluid2-flip", "dp2-coulomb-obstacle", "dp3", "fluid3-apic"])
def test_single_step_tight(orc, name):
    s = SCENES[name]("f64")
    st = init_scene(s)
    orc.advance(s, st, 5)
    want = orc.advance(s, st.copy(), 1)
    got = gpu_run(s, st, 1)
    assert_state_close(got, want, PHASE_RTOL["f64"], what=name)


@pytest.mark.parametrize("name", ["fluid2-apic", "fluid2-tpic-visc", "dp2-coulomb-obstacle", "dp3", "fluid3-flip"])
def test_phase_parity(orc, name):
    """p2g / grid_momentum_update / apply_grid_corrections / g2p / constitutive_update separately."""
    s = SCENES[name]("f64")
    st = init_scene(s)
    orc.advance(s, st, 3)
    rtol = PHASE_RTOL["f64"]
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.p2g()
    g_ref = orc.p2g(s, st)
    assert_grid_close(ctx.grid_download(), g_ref, rtol, "p2g")
    ctx.grid_momentum_update()
    g_ref = orc.grid_momentum_update(s, g_ref)
    assert_grid_close(ctx.grid_download(), g_ref, rtol, "momentum")
    ctx.grid_corrections()
    g_ref = orc.grid_corrections(s, g_ref)
    assert_grid_close(ctx.grid_download(), g_ref, rtol, "corrections")
    # g2p on the oracle's grid, then constitutive
    ctx.grid_upload(g_ref)
    ctx.g2p()
    want = orc.g2p(s, g_ref, st.copy())
    got = ctx.download(st.copy())
    assert_state_close(got, want, rtol, what="g2p")
    ctx.constitutive()
    want = orc.constitutive(s, want)
    got = ctx.download(st.copy())
    assert_state_close(got, want, rtol, what="constitutive")
    ctx.close()


def test_corrections_on_uploaded_grid(orc):
    """test_contact.cpp pipeline: walls, obstacles and Coulomb on every node of a random grid."""
    s = dp_block_scene(2, coulomb=True, obstacle=True)
    rng = np.random.default_rng(47)
    ctx = Context(s, 16)
    g = ctx.new_grid()
    g.v[...] = rng.uniform(-2, 2, g.v.shape)
    ctx.grid_upload(g)
    ctx.grid_corrections()
    got = ctx.grid_download()
    want = orc.grid_corrections(s, g)
    assert np.array_equal(got.v, want.v) or np.abs(got.v - want.v).max() < 1e-15
    assert (np.linalg.norm(got.v, axis=1) <= np.linalg.norm(g.v, axis=1) * (1 + 1e-14)).all()
    ctx.close()


@pytest.mark.slow
def test_c1_200_steps_f64(orc):
    """C1 (2-D D-P column, 20,000 particles) through 200 steps."""
    s = c1_column()
    st = init_scene(s)
    want = orc.advance(s, st.copy(), 200)
    got = gpu_run(s, st, 200)
    assert_state_close(got, want, 1e-9, what="C1x200")


def test_deterministic_and_grid_is_derived(orc):
    """test_stepper.cpp:168-196: bit-identical runs; poisoning the grid between steps changes nothing."""
    s = dp_block_scene(3, cells=[12, 12, 12])
    st = init_scene(s)
    a = Context(s, st.particles.size())
    a.upload(st)
    a.advance(30)
    b = Context(s, st.particles.size())
    b.upload(st)
    for _ in range(30):
        g = b.new_grid()
        g.mass[:] = 1e30
        g.v[:] = 1e30
        b.grid_upload(g)
        b.advance(1)
    assert a.digest() == b.digest()
    sa, sb = a.download(st.copy()), b.download(st.copy())
    for f in ("x", "v", "sigma", "grad_v"):
        assert np.array_equal(getattr(sa.particles, f), getattr(sb.particles, f))


@pytest.mark.parametrize("kind", ["flip", "blend", "tpic"])
def test_grad_v_stored_by_the_last_step_of_a_call(orc, kind):
    """Inside one advance() call only the last step stores grad v when no scheme reads it
    (DESIGN.md §5): any chunking of the same steps gives bit-identical states, grad v included,
    and the result matches the oracle."""
    s = fluid_box_scene(2, kind=kind, alpha=0.3) if kind == "blend" else fluid_box_scene(2, kind=kind)
    st = init_scene(s)
    ctxs = []
    for chunks in ([12], [7, 5], [1] * 12):
        c = Context(s, st.particles.size())
        c.upload(st)
        for k in chunks:
            c.advance(k)
        ctxs.append(c.download(st.copy()))
    for other in ctxs[1:]:
        for f in ("x", "v", "sigma", "rho", "volume", "grad_v"):
            assert np.array_equal(getattr(ctxs[0].particles, f), getattr(other.particles, f)), f
    ref = st.copy()
    orc.advance(s, ref, 12)
    assert_state_close(ctxs[0], ref, STEP_RTOL["f64"])


def test_stepper_api_mirror(orc):
    """Stepper(scene).advance(state) as in the reference (stepper.hpp:49-70)."""
    s = small_fluid_scene("flip")
    s.config.gravity = [0.0, -9.8]
    st = init_scene(s)
    ref = st.copy()
    stepper = Stepper(s)
    for _ in range(50):
        stepper.advance(st)
    orc.advance(s, ref, 50)
    expect = np.array([0.0, -9.8]) * 50 * s.config.dt
    assert (np.linalg.norm(st.particles.v - expect, axis=1) <= 1e-10 * np.linalg.norm(expect)).all()
    assert st.step == 50


def test_single_particle_unchanged():
    """test_stepper.cpp:10-23"""
    s = small_fluid_scene("pic")
    s.mass_epsilon = 1e-15
    st = single_particle_state(s, [0.513, 0.497], [0.0, 0.0])
    got = gpu_run(s, st, 1)
    assert got.step == 1 and np.array_equal(got.particles.x, st.particles.x)
    assert np.abs(got.particles.v).max() == 0 and np.abs(got.particles.sigma).max() == 0


def test_two_particle_mirror_symmetry():
    """test_stepper.cpp:40-66 on the GPU"""
    s = small_fluid_scene("pic")
    s.mass_epsilon = 1e-15
    st = SimState.zeros(2, 2, np.float64)
    dh = s.config.dh
    st.particles.mass[:] = 1000.0 * dh * dh / 4
    st.particles.rho[:] = 1000.0
    st.particles.volume[:] = st.particles.mass / 1000.0
    st.particles.x[:] = [[0.44, 0.5], [0.56, 0.5]]
    st.particles.v[:] = [[0.8, 0.0], [-0.8, 0.0]]
    ctx = Context(s, 2)
    ctx.upload(st)
    for _ in range(200):
        ctx.advance(1)
        c = ctx.download(st.copy())
        x, v = c.particles.x, c.particles.v
        assert abs((x[0, 0] - 0.5) + (x[1, 0] - 0.5)) < 1e-10
        assert abs(v[0, 0] + v[1, 0]) < 1e-10
        assert abs(x[0, 1] - x[1, 1]) < 1e-10


def test_run_snapshots_cfl_and_nan():
    """test_stepper.cpp:68-126"""
    s = small_fluid_scene("pic")
    st = init_scene(s)
    assert len(run(s, st, 0, 10).snapshots) == 1
    r = run(s, st, 8, 8)
    assert [x.step for x in r.snapshots] == [0, 8]
    assert [x.step for x in run(s, st, 9, 3).snapshots] == [0, 3, 6, 9]
    bad = st.copy()
    bad.particles.v[3, 0] = np.nan
    with pytest.raises(NumericalError):
        run(s, bad, 5, 0)
    s.config.dt = 1.0
    with pytest.raises(ValidationError):
        run(s, st, 1, 0)
    assert len(run(s, st, 0, 0, force=True).snapshots) == 1


def test_out_of_domain_names_lowest_particle(orc):
    """bspline.hpp:86-91 through the step: the smallest offending id is reported."""
    s = small_fluid_scene("pic")
    st = init_scene(s)
    st.particles.x[200] = [0.01, 0.5]
    st.particles.x[42] = [0.5, 0.99]
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    with pytest.raises(OutOfDomainError) as e:
        ctx.advance(1)
    assert e.value.particle == 42
    # a block thrown across the wall band in one step: the same id and step as the oracle
    s2 = small_fluid_scene("pic")
    s2.geometry[0] = GeometryRegion(lo=[0.6, 0.3], hi=[0.85, 0.6])
    s2.config.dt = 1e-4
    st2 = init_scene(s2)
    st2.particles.v[:, 0] = 3000.0  # after seeding (init_scene would refuse the CFL)
    ref = st2.copy()
    with pytest.raises(OutOfDomainError) as er:
        orc.advance(s2, ref, 5)
    ctx2 = Context(s2, st2.particles.size())
    ctx2.upload(st2)
    with pytest.raises(OutOfDomainError) as eg:
        ctx2.advance(5)
    assert eg.value.particle == er.value.particle
    assert ctx2.download(st2.copy()).step == ref.step


def test_closed_box_slip_momentum_1000_steps():
    """test_stepper.cpp:128-166 on the GPU: slip-wall momentum to 1e-8, mass exactly."""
    s = small_fluid_scene("pic")
    s.geometry[0] = GeometryRegion(lo=[0.2, 0.1], hi=[0.5, 0.3], velocity=VelocityExpr("constant", value=[1.0, 0.0]))
    st = init_scene(s)
    px0 = (st.particles.mass * st.particles.v[:, 0]).sum()
    got = gpu_run(s, st, 1000)
    px1 = (got.particles.mass * got.particles.v[:, 0]).sum()
    assert abs(px1 - px0) <= 1e-8 * abs(px0)
    assert np.array_equal(got.particles.mass, st.particles.mass)


def test_p2g_conservation_all_schemes():
    """test_transfer.cpp:69-102 on the GPU grid"""
    for kind in ("pic", "flip", "blend", "apic", "tpic"):
        s = small_fluid_scene(kind, 0.7)
        st = random_block(s, 101)
        rng = np.random.default_rng(7)
        if kind == "apic":
            st.particles.affine[...] = rng.uniform(-0.5, 0.5, st.particles.affine.shape)
        if kind == "tpic":
            st.particles.grad_v[...] = rng.uniform(-0.5, 0.5, st.particles.grad_v.shape)
        ctx = Context(s, st.particles.size())
        ctx.upload(st)
        ctx.p2g()
        g = ctx.grid_download()
        assert g.mass.sum() == pytest.approx(st.particles.mass.sum(), rel=1e-12)
        pm = (st.particles.mass[:, None] * st.particles.v).sum(axis=0)
        assert np.linalg.norm(g.momentum.sum(axis=0) - pm) <= 1e-12 * np.linalg.norm(pm)
        ctx.close()


def test_catastrophic_compression_raises():
    s = small_fluid_scene("pic")
    s.config.dt = 1.0
    st = single_particle_state(s, [0.5, 0.5], [0.0, 0.0])
    st.particles.grad_v[0] = [[-0.6, 0.0], [0.0, -0.6]]
    ctx = Context(s, 1)
    ctx.upload(st)
    with pytest.raises(NumericalError):
        ctx.constitutive()


def test_unsymmetric_stress_rejected():
    """the packed-symmetric contract is checked on the device copy: the lowest offending particle
    is reported and the context keeps its previous state"""
    s = small_fluid_scene("pic")
    st = init_scene(s)
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    d0 = ctx.digest()
    bad = st.copy()
    bad.particles.sigma[7] = [[1.0, 2.0], [3.0, 4.0]]
    bad.particles.sigma[3] = [[1.0, 2.0], [2.5, 4.0]]
    with pytest.raises(ValidationError, match="particle 3 "):
        ctx.upload(bad)
    assert ctx.digest() == d0
    ctx.advance(2)  # still usable
    ctx.close()


@pytest.mark.parametrize("dim", [2, 3])
def test_empty_state_steps_like_the_reference(orc, ref, dim):
    """an empty particle set is a valid state: the reference steps it (step and time advance, no
    particles); so do the device path, run() and step_vjp"""
    from paper_2507_04192_b200.solver import run, step_vjp
    from paper_2507_04192_b200.state import ParamGrads, SimState, StateCotangent

    from test_distributed import moving_fluid_scene

    s = moving_fluid_scene(dim) if dim == 3 else small_fluid_scene("flip")
    init_scene(s)  # sets mass_epsilon
    st = SimState.zeros(0, dim, s.np_dtype)
    want = st.copy()
    ref.advance(s, want, 3)
    ctx = Context(s, 0)
    ctx.upload(st)
    ctx.advance(3, nan_guard=True)
    got = ctx.download(st.copy())
    ctx.close()
    assert got.step == want.step == 3 and got.time == want.time and got.particles.size() == 0
    res = run(s, st, 4, 2)
    assert [x.step for x in res.snapshots] == [0, 2, 4]
    cin = step_vjp(s, st, StateCotangent.zeros_like(st.particles), None, ParamGrads(s.boundary))
    assert cin.x.shape == (0, dim)


@pytest.mark.parametrize("name", ["dp2-noslip", "fluid2-apic", "dp3", "fluid3-flip"])
def test_track_def_grad_parity(orc, name):
    """F <- (I + grad v dt) F when track_def_grad is set (stepper.hpp:39-42), in the G2P
    epilogue (all schemes) and in the separate constitutive phase; against the oracle."""
    s = SCENES[name]("f64")
    s.config.track_def_grad = True
    st = init_scene(s)
    assert st.particles.def_grad is not None
    want = orc.advance(s, st.copy(), 20)
    got = gpu_run(s, st, 20)
    assert_state_close(got, want, STEP_RTOL["f64"], what=name + "+F")
    assert rel_err(got.particles.def_grad, want.particles.def_grad, 1.0) <= 1e-10
    eye = np.eye(s.dim)
    assert np.abs(want.particles.def_grad - eye).max() > 1e-8  # F actually evolved
    # the phase path: constitutive_update alone on an uploaded state
    ctx = Context(s, st.particles.size())
    ctx.upload(want)
    ctx.constitutive()
    g1 = ctx.download(want.copy())
    ctx.close()
    w1 = orc.constitutive(s, want.copy())
    assert rel_err(g1.particles.def_grad, w1.particles.def_grad, 1.0) <= 1e-13


def test_particle_count_change_recaptures_the_step_graph(orc):
    """the captured step graph bakes in n. Upload n1, advance, upload a smaller
    (then a larger) state to the same context, advance again: identical to a fresh context."""
    s = dp_block_scene(3, cells=[12, 12, 12])
    st = init_scene(s)
    n1 = st.particles.size()
    small = SimState(st.particles.take(np.arange(0, n1, 2)))
    ctx = Context(s, n1)
    for state in (st, small, st):
        ctx.upload(state)
        ctx.advance(4)
        got = ctx.download(state.copy())
        fresh = Context(s, n1)
        fresh.upload(state)
        fresh.advance(4)
        want = fresh.download(state.copy())
        fresh.close()
        for f in ("x", "v", "sigma", "grad_v"):
            assert np.array_equal(getattr(got.particles, f), getattr(want.particles, f)), f
    ctx.close()
