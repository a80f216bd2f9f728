"""Pin the CPU oracle (oracle/mpm_oracle.cpp) against the reference's own known-answer tests.

Every case restates a check from /root/reference/proj/tests/*.cpp (cited per test) and runs
it through the oracle's stateless ABI -- the same entry points the GPU parity tests use.
"""
import math

import numpy as np
import pytest

from helpers import dp_block_scene, random_block, single_particle_state
from paper_2507_04192_b200 import (DruckerPragerParams, FluidParams, GeometryRegion, Obstacle, Scene, SimConfig,
                                   SimState, VelocityExpr, Wall, cfl_report, init_scene)
from paper_2507_04192_b200.errors import NumericalError, OutOfDomainError, ValidationError
from paper_2507_04192_b200.presets import bui_sand, small_fluid_scene


def _grid(orc, s):
    return orc.new_grid(s)


def test_single_particle_on_node_pic_pattern(orc):
    """test_transfer.cpp:48-67: particle exactly on node (10,10): m_node = m_p 0.75^2."""
    s = small_fluid_scene("pic")
    dh = s.config.dh
    st = single_particle_state(s, [10 * dh, 10 * dh], [0.3, -0.2])
    g = orc.p2g(s, st)
    mp = st.particles.mass[0]
    nk = g.node_index([10, 10])
    assert g.mass[nk] == pytest.approx(mp * 0.75 * 0.75, rel=1e-14)
    assert np.linalg.norm(g.momentum[nk] / g.mass[nk] - [0.3, -0.2]) < 1e-14
    assert g.mass.sum() == pytest.approx(mp, rel=1e-14)


@pytest.mark.parametrize("kind", ["pic", "flip", "blend", "apic", "tpic"])
def test_p2g_conserves_mass_and_momentum(orc, kind):
    """test_transfer.cpp:69-102 (seeds are ours; the reference uses mt19937_64)."""
    s = small_fluid_scene(kind, 0.7)
    st = random_block(s, 101)
    rng = np.random.default_rng(7)
    if kind == "apic":
        st.particles.affine[...] = rng.uniform(-0.5, 0.5, st.particles.affine.shape)
    if kind == "tpic":
        st.particles.grad_v[...] = rng.uniform(-0.5, 0.5, st.particles.grad_v.shape)
    g = orc.p2g(s, st)
    assert g.mass.sum() == pytest.approx(st.particles.mass.sum(), rel=1e-12)
    pm = (st.particles.mass[:, None] * st.particles.v).sum(axis=0)
    assert np.linalg.norm(g.momentum.sum(axis=0) - pm) <= 1e-12 * np.linalg.norm(pm)


def test_gravity_adds_g_dt(orc):
    """test_transfer.cpp:104-124"""
    s = small_fluid_scene("pic")
    st = random_block(s, 33)
    s.config.gravity = [0.0, -9.8]
    g = orc.p2g(s, st)
    g = orc.grid_momentum_update(s, g)
    act = g.mass > 1e-12
    dv = g.v[act] - g.v_old[act] - s.config.dt * np.array([0.0, -9.8])
    assert np.abs(dv).max() < 1e-14


def test_far_stencil_node_stays_zero(orc):
    """test_transfer.cpp:126-143"""
    s = small_fluid_scene("pic")
    dh = s.config.dh
    s.config.gravity = [0.0, -9.8]
    st = single_particle_state(s, [10.5 * dh, 10.5 * dh], [1.0, 0.0])
    g = orc.p2g(s, st)
    far = g.node_index([12, 12])
    assert g.mass[far] == 0.0
    s.mass_epsilon = 1e-12
    g = orc.grid_momentum_update(s, g)
    assert np.linalg.norm(g.v[far]) == 0.0 and np.isfinite(g.v).all()


@pytest.mark.parametrize("kind", ["pic", "flip", "blend", "apic", "tpic"])
def test_uniform_velocity_reproduces_itself(orc, kind):
    """test_transfer.cpp:145-163"""
    s = small_fluid_scene(kind, 0.4)
    st = init_scene(s)
    st.particles.v[...] = [0.4, -0.3]
    g = orc.p2g(s, st)
    g = orc.grid_momentum_update(s, g)
    st = orc.g2p(s, g, st)
    assert np.abs(st.particles.v - [0.4, -0.3]).max() < 1e-12
    assert np.abs(st.particles.grad_v).max() < 1e-12 / s.config.dh


@pytest.mark.parametrize("kind", ["pic", "flip"])
def test_free_fall_one_cycle(orc, kind):
    """test_transfer.cpp:186-201"""
    s = small_fluid_scene(kind)
    s.config.gravity = [0.0, -9.8]
    s.mass_epsilon = 1e-15
    st = single_particle_state(s, [0.512, 0.483], [0.2, 0.1])
    g = orc.p2g(s, st)
    g = orc.grid_momentum_update(s, g)
    st = orc.g2p(s, g, st)
    assert np.linalg.norm(st.particles.v[0] - (np.array([0.2, 0.1]) + 1e-4 * np.array([0, -9.8]))) < 1e-13


def test_repeated_p2g_bit_identical(orc):
    """test_transfer.cpp:247-256"""
    s = small_fluid_scene("apic")
    s.config.gravity = [0.0, -9.8]
    st = random_block(s, 5150)
    a, b = orc.p2g(s, st), orc.p2g(s, st)
    for f in ("mass", "momentum", "force"):
        assert np.array_equal(getattr(a, f), getattr(b, f))


def test_eos_hand_value(orc):
    """test_constitutive.cpp:72-82: 1% compression -> rho = 1010.1010101010102, p = 12373.7..."""
    s = small_fluid_scene("pic")
    s.material = FluidParams(1000.0, 0.0, 35.0)
    s.config.dt = 1.0
    st = single_particle_state(s, [0.5, 0.5], [0, 0])
    st.particles.grad_v[0] = [[-0.005, 0.0], [0.0, -0.005]]
    st = orc.constitutive(s, st)
    assert st.particles.rho[0] == pytest.approx(1010.1010101010102, rel=1e-12)
    assert -st.particles.sigma[0, 0, 0] == pytest.approx(12373.737373737447, rel=1e-12)


def test_catastrophic_compression_raises(orc):
    """test_constitutive.cpp:84-90"""
    s = small_fluid_scene("pic")
    s.material = FluidParams(1000.0, 0.0, 35.0)
    s.config.dt = 1.0
    st = single_particle_state(s, [0.5, 0.5], [0, 0])
    st.particles.grad_v[0] = [[-0.6, 0.0], [0.0, -0.6]]
    with pytest.raises(NumericalError):
        orc.constitutive(s, st)


def test_dp_derived_constants(orc):
    """test_constitutive.cpp:103-131"""
    p = orc.dp_make(2650.0, 0.7e6, 0.3, 19.8 * math.pi / 180.0, 0.0, 0.0, 0.0)
    assert p.q_psi == 0.0 and p.k_phi == 0.0 and p.tau_P == 0.0
    assert p.q_phi == pytest.approx(0.3514569291332422, rel=1e-12)
    assert p.alpha_P == pytest.approx(0.7085062650559565, rel=1e-12)
    p = orc.dp_make(2650.0, 0.7e6, 0.3, 0.3, 0.1, 2000.0, 500.0)
    assert p.tau_P == pytest.approx(p.k_phi - p.q_phi * 500.0, rel=1e-14)
    # the product's host-side make() restates the same derivation
    q = DruckerPragerParams.make(2650.0, 0.7e6, 0.3, 0.3, 0.1, 2000.0, 500.0)
    assert q.q_phi == p.q_phi and q.k_phi == p.k_phi and q.alpha_P == p.alpha_P and q.G == p.G


def _dp_particles(s, sig, szz, gv):
    n = len(sig)
    st = SimState.zeros(n, 2, np.float64)
    st.particles.x[:] = 0.5
    st.particles.mass[:] = 1.0
    st.particles.volume[:] = 1.0
    st.particles.rho[:] = 2650.0
    st.particles.sigma[...] = sig
    st.particles.sigma_zz[...] = szz
    st.particles.grad_v[...] = gv
    return st


def test_dp_tension_cap_hand_value(orc):
    """test_constitutive.cpp:142-154: hydrostatic 2 sigma_t -> sigma_t, deps = sqrt2/3 sigma_t/K"""
    c, sigma_t = 2000.0, 400.0
    s = small_fluid_scene()
    s.material = bui_sand(c, sigma_t)
    s.config.dt = 1e-5
    st = _dp_particles(s, [2 * sigma_t * np.eye(2)], [2 * sigma_t], [np.zeros((2, 2))])
    st = orc.constitutive(s, st)
    assert np.linalg.norm(st.particles.sigma[0] - sigma_t * np.eye(2)) < 1e-10
    assert st.particles.sigma_zz[0] == pytest.approx(sigma_t, rel=1e-12)
    assert st.particles.eps_eq[0] == pytest.approx(math.sqrt(2.0) / 3.0 * sigma_t / s.material.K, rel=1e-12)


@pytest.mark.parametrize("cohesive", [False, True])
def test_dp_random_trials_feasible(orc, cohesive):
    """test_constitutive.cpp:156-190 (feasibility half; zone labels are internal to the update)"""
    s = small_fluid_scene()
    s.material = bui_sand(2000.0, 800.0) if cohesive else bui_sand()
    s.config.dt = 1e-4
    rng = np.random.default_rng(21 if cohesive else 20)
    n = 10000
    a, b, c = rng.uniform(-5e3, 5e3, (3, n))
    sig = np.stack([np.stack([a, c], -1), np.stack([c, b], -1)], 1)
    szz = rng.uniform(-5e3, 5e3, n)
    gv = rng.uniform(-20, 20, (n, 2, 2))
    st = orc.constitutive(s, _dp_particles(s, sig, szz, gv))
    m = s.material
    S = np.zeros((n, 3, 3))
    S[:, :2, :2] = st.particles.sigma
    S[:, 2, 2] = st.particles.sigma_zz
    sm = np.trace(S, axis1=1, axis2=2) / 3
    dev = S - sm[:, None, None] * np.eye(3)
    tau = np.sqrt(0.5 * (dev ** 2).sum(axis=(1, 2)))
    scale = np.maximum(1.0, np.abs(sm) + tau)
    assert (tau - m.k_phi + m.q_phi * sm <= 1e-8 * scale).all()
    assert (sm <= m.sigma_t + 1e-10 * max(1.0, m.sigma_t)).all()
    assert (st.particles.eps_eq >= 0).all()


def test_coulomb_and_walls_hand_values(orc):
    """test_contact.cpp:19-65, 94-122: slip/no-slip bands, Coulomb (3,-1) mu 0.2 -> (2.8, 0), stick -> 0"""
    s = Scene(2)
    s.config.dh, s.config.cells = 0.1, [10, 10]
    s.config.dt = 1e-4
    s.boundary.walls[2] = Wall("coulomb", [0.2])
    g = orc.new_grid(s)
    g.v[g.node_index([5, 0])] = [3.0, -1.0]
    g.v[g.node_index([6, 1])] = [0.1, -1.0]
    g.v[g.node_index([7, 1])] = [0.5, 1.0]
    g.v[g.node_index([0, 5])] = [-1.0, 2.0]   # left slip band
    g.v[g.node_index([5, 5])] = [1.0, -1.0]   # interior
    g = orc.grid_corrections(s, g)
    assert g.v[g.node_index([5, 0])] == pytest.approx([2.8, 0.0], abs=1e-14)
    assert np.linalg.norm(g.v[g.node_index([6, 1])]) == 0.0
    assert list(g.v[g.node_index([7, 1])]) == [0.5, 1.0]
    assert list(g.v[g.node_index([0, 5])]) == [0.0, 2.0]
    assert list(g.v[g.node_index([5, 5])]) == [1.0, -1.0]
    s.boundary.walls[2] = Wall("no_slip")
    g = orc.new_grid(s)
    for iy in (0, 1, 2):
        g.v[g.node_index([5, iy])] = [1.0, -1.0]
    g = orc.grid_corrections(s, g)
    assert np.linalg.norm(g.v[g.node_index([5, 0])]) == 0 and np.linalg.norm(g.v[g.node_index([5, 1])]) == 0
    assert list(g.v[g.node_index([5, 2])]) == [1.0, -1.0]


def test_obstacle_contact(orc):
    """test_contact.cpp:190-205"""
    s = Scene(2)
    s.config.dh, s.config.cells, s.config.dt = 0.1, [10, 10], 1e-4
    s.obstacles.append(Obstacle([0.38, 0.38], [0.62, 0.62]))
    g = orc.new_grid(s)
    g.v[g.node_index([4, 5])] = [1.0, 0.2]
    g.v[g.node_index([2, 5])] = [5.0, 5.0]
    g = orc.grid_corrections(s, g)
    assert g.v[g.node_index([4, 5])] == pytest.approx([0.0, 0.2], abs=1e-15)
    assert list(g.v[g.node_index([2, 5])]) == [5.0, 5.0]


def test_cfl_report_values():
    """test_stepper.cpp:100-116"""
    cfg = SimConfig(dim=2, dh=0.004, dt=1e-5, cells=[10, 10])
    assert cfl_report(cfg, FluidParams(1000.0, 0.0, 35.0), 0.0) == pytest.approx(0.0875, rel=1e-12)
    cfg.dt = 2e-5
    dp = DruckerPragerParams.make(2650.0, 0.7e6, 0.3, 19.8 * math.pi / 180, 0.0, 0.0, 0.0)
    assert cfl_report(cfg, dp, 0.0) == pytest.approx(2e-5 * 20.65684801952119 / 0.004, rel=1e-10)


def test_free_fall_block_50_steps(orc):
    """test_stepper.cpp:25-38"""
    s = small_fluid_scene("flip")
    s.config.gravity = [0.0, -9.8]
    st = init_scene(s)
    orc.advance(s, st, 50)
    expect = np.array([0.0, -9.8]) * 50 * s.config.dt
    assert (np.linalg.norm(st.particles.v - expect, axis=1) <= 1e-10 * np.linalg.norm(expect)).all()


def test_two_particle_mirror_symmetry(orc):
    """test_stepper.cpp:40-66"""
    s = small_fluid_scene("pic")
    s.mass_epsilon = 1e-15
    st = SimState.zeros(2, 2, np.float64)
    dh = s.config.dh
    st.particles.mass[:] = 1000.0 * dh * dh / 4
    st.particles.rho[:] = 1000.0
    st.particles.volume[:] = st.particles.mass / 1000.0
    st.particles.x[:] = [[0.44, 0.5], [0.56, 0.5]]
    st.particles.v[:] = [[0.8, 0.0], [-0.8, 0.0]]
    for _ in range(200):
        orc.advance(s, st, 1)
        x, v = st.particles.x, st.particles.v
        assert abs((x[0, 0] - 0.5) + (x[1, 0] - 0.5)) < 1e-10
        assert abs(v[0, 0] + v[1, 0]) < 1e-10
        assert abs(x[0, 1] - x[1, 1]) < 1e-10


def test_nan_guard_and_out_of_domain(orc):
    """test_stepper.cpp:92-98 and test_bspline.cpp:108-123 through the step"""
    s = small_fluid_scene("pic")
    st = init_scene(s)
    st.particles.v[3, 0] = np.nan
    with pytest.raises(NumericalError):
        orc.advance(s, st.copy(), 5, nan_guard=True)
    st = init_scene(s)
    st.particles.x[42] = [0.01, 0.5]
    with pytest.raises(OutOfDomainError) as e:
        orc.advance(s, st, 1)
    assert e.value.particle == 42 and "42" in str(e.value)


def test_closed_box_conservation(orc):
    """test_stepper.cpp:128-166: slip-wall momentum to 1e-8 over 1000 steps"""
    s = small_fluid_scene("pic")
    s.geometry[0] = GeometryRegion(lo=[0.2, 0.1], hi=[0.5, 0.3], velocity=VelocityExpr("constant", value=[1.0, 0.0]))
    st = init_scene(s)
    px0 = (st.particles.mass * st.particles.v[:, 0]).sum()
    orc.advance(s, st, 1000, nan_guard=True)
    px1 = (st.particles.mass * st.particles.v[:, 0]).sum()
    assert abs(px1 - px0) <= 1e-8 * abs(px0)


def test_init_scene_counts_and_mass(orc):
    """test_scene.cpp:34-68 (column scene: 10,000 particles, 250 kg, linear-in-y profile)"""
    s = Scene(2)
    dh = 0.01
    s.config.dh, s.config.cells, s.config.dt = dh, [150, 60], 3e-5
    s.config.gravity = [0.0, -9.8]
    s.material = FluidParams(1000.0, 0.0, 50.0)
    s.geometry.append(GeometryRegion(lo=[2 * dh, 2 * dh], hi=[0.5 + 2 * dh, 0.5 + 2 * dh],
                                     velocity=VelocityExpr("linear_in_y", alpha=2.0, h0=0.5)))
    st = orc.init_scene(s.copy())
    assert st.particles.size() == 10000
    assert st.particles.mass.sum() == pytest.approx(250.0, rel=1e-10)
    y0 = 2 * dh
    assert np.allclose(st.particles.v[:, 0], 2.0 * (0.5 - (st.particles.x[:, 1] - y0)), rtol=1e-14)
    # the product-side seeding restates the same lattice, bit for bit
    mine = init_scene(s.copy())
    for f in ("x", "v", "mass", "volume", "rho"):
        assert np.array_equal(getattr(mine.particles, f), getattr(st.particles, f)), f
    s2 = s.copy()
    s2.geometry[0].lo[0] = 0.005
    with pytest.raises(ValidationError):
        init_scene(s2)


def test_oracle_dp_column_runs(orc):
    s = dp_block_scene(2)
    st = init_scene(s)
    orc.advance(s, st, 20, nan_guard=True)
    assert st.particles.all_finite() and (st.particles.eps_eq >= 0).all()
