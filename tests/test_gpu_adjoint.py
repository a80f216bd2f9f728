"""GPU adjoint parity: step_vjp and backprop_trajectory through the C ABI vs the CPU oracle
(itself bit-identical to the reference's step_vjp / backprop_trajectory), plus the SPEC.md
contracts: zero-in/zero-out, linearity, segment invariance (bit-identical), finite differences."""
import numpy as np
import pytest

from helpers import dp_block_scene, fluid_box_scene, rel_err
from paper_2507_04192_b200 import GeometryRegion, ParamGrads, StateCotangent, VelocityExpr, init_scene
from paper_2507_04192_b200.presets import small_fluid_scene
from paper_2507_04192_b200.solver import Context

pytestmark = pytest.mark.gpu

SCENES = {
    "fluid2-flip": lambda: fluid_box_scene(2, kind="flip"),
    "fluid2-pic-visc": lambda: fluid_box_scene(2, kind="pic", visc=0.5),
    "fluid2-apic": lambda: fluid_box_scene(2, kind="apic"),
    "fluid2-tpic-rate": lambda: fluid_box_scene(2, kind="tpic", visc=0.3, rate_form=True),
    "dp2-noslip": lambda: dp_block_scene(2),
    "dp2-coulomb-obstacle": lambda: dp_block_scene(2, coulomb=True, obstacle=True),
    "dp3": lambda: dp_block_scene(3, cells=[12, 12, 12]),
    "dp3-coulomb": lambda: dp_block_scene(3, coulomb=True, cells=[16, 12, 12]),
    "fluid3-apic": lambda: fluid_box_scene(3, kind="apic"),
}


def random_cot(st, seed):
    rng = np.random.default_rng(seed)
    c = StateCotangent.zeros_like(st.particles)
    for f in StateCotangent.FIELDS:
        a = getattr(c, f)
        if a is not None and a.size and f != "eps_eq":
            a[...] = rng.standard_normal(a.shape)
    return c


def cot_errs(got, want):
    out = {}
    for f in StateCotangent.FIELDS:
        a, b = getattr(got, f), getattr(want, f)
        if b is None or b.size == 0:
            continue
        out[f] = rel_err(a, b, 1e-300)
    return out


def well_conditioned_dp_stress(s, st, seed, margin=0.05):
    """Random symmetric stresses whose return-map branch (elastic / shear / apex / cap / tensile)
    is decided with a margin: the D-P update is only piecewise smooth, and at a branch boundary
    rounding-level differences in grad v legitimately select different branches."""
    m = s.material
    rng = np.random.default_rng(seed)
    n, d = st.particles.size(), s.dim
    out = np.zeros((n, 3, 3))
    k = 0
    while k < n:
        A = rng.uniform(-6e3, 3e3, (3, 3))
        S = 0.5 * (A + A.T)
        if d == 2:
            S[2, :2] = S[:2, 2] = 0.0
        sm = np.trace(S) / 3
        tau = np.sqrt(0.5 * ((S - sm * np.eye(3)) ** 2).sum())
        fs = tau - m.k_phi + m.q_phi * sm
        ft = sm - m.sigma_t
        h = tau - m.tau_P - m.alpha_P * (sm - m.sigma_t)
        denom = m.G + m.K * m.q_phi * m.q_psi
        sm_new = sm - m.K * m.q_psi * fs / denom
        tau_new = m.k_phi - m.q_phi * sm_new
        scale = abs(sm) + tau + 1.0
        if min(abs(fs), abs(ft), abs(h), abs(tau_new), abs(sm_new - m.sigma_t)) < margin * scale:
            continue
        out[k] = S
        k += 1
    st.particles.sigma[...] = out[:, :d, :d]
    if d == 2:
        st.particles.sigma_zz[...] = out[:, 2, 2]
    return st


@pytest.mark.parametrize("name", sorted(SCENES))
def test_step_vjp_parity(orc, name):
    s = SCENES[name]()
    st = init_scene(s)
    orc.advance(s, st, 8)
    if name.startswith("dp"):
        from paper_2507_04192_b200.presets import bui_sand
        s.material = bui_sand(2000.0, 800.0)  # cohesive: all three zones reachable
        well_conditioned_dp_stress(s, st, 9)
    cot = random_cot(st, 11)
    want, pg_w = orc.step_vjp(s, st, cot)
    ctx = Context(s, st.particles.size())
    pg = ParamGrads(s.boundary)
    got = ctx.step_vjp(st, cot, pg)
    errs = cot_errs(got, want)
    bad = {k: v for k, v in errs.items() if v > 1e-10}
    assert not bad, f"{name}: " + ", ".join(f"{k}={v:.2e}" for k, v in errs.items())
    for a, b in ((pg.sound_speed, pg_w.sound_speed), (pg.viscosity, pg_w.viscosity)):
        assert abs(a - b) <= 1e-10 * max(abs(b), 1e-30) + 1e-300
    for w in range(6):
        fw = pg_w.wall_friction[w]
        if len(fw):
            assert rel_err(pg.wall_friction[w], fw, 1e-300) < 1e-10
    ctx.close()


def test_step_vjp_zero_and_linearity():
    s = dp_block_scene(2, coulomb=True)
    st = init_scene(s)
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.advance(5)
    st = ctx.download(st.copy())
    z = ctx.step_vjp(st, StateCotangent.zeros_like(st.particles), ParamGrads(s.boundary))
    for f in StateCotangent.FIELDS:
        a = getattr(z, f)
        assert a is None or not np.any(a)
    a, b = random_cot(st, 1), random_cot(st, 2)
    ab = a.copy()
    ab.axpy(0.0, a)
    for f in StateCotangent.FIELDS:
        x = getattr(ab, f)
        if x is not None:
            x[...] = 2.0 * getattr(a, f) - 3.0 * getattr(b, f)
    ga = ctx.step_vjp(st, a, ParamGrads(s.boundary))
    gb = ctx.step_vjp(st, b, ParamGrads(s.boundary))
    gab = ctx.step_vjp(st, ab, ParamGrads(s.boundary))
    for f in StateCotangent.FIELDS:
        x = getattr(gab, f)
        if x is None or x.size == 0:
            continue
        lin = 2.0 * getattr(ga, f) - 3.0 * getattr(gb, f)
        assert rel_err(x, lin, 1e-300) < 1e-12, f


def _seeder_final_x(st_final, steps, offset=0.01):
    return {"field": "x", "obs_steps": [steps], "sel": None, "target": st_final.particles.x[None] + offset}


@pytest.mark.parametrize("nseg", [1, 3])
def test_backprop_parity(orc, nseg):
    s = fluid_box_scene(2, kind="flip")
    from paper_2507_04192_b200 import Obstacle, Wall
    s.boundary.walls[2] = Wall("coulomb", [0.1, 0.4, 0.2])
    s.obstacles.append(Obstacle([0.7, 0.0], [0.9, 0.3]))
    s.geometry[0].lo = [0.3, 0.1]
    st = init_scene(s)
    fin = orc.advance(s, st.copy(), 12)
    seeder = {"field": "x", "obs_steps": [6, 12], "sel": [3, 40, 77, 100],
              "target": np.stack([fin.particles.x[[3, 40, 77, 100]] + 0.01, fin.particles.x[[3, 40, 77, 100]] - 0.02])}
    c_w, pg_w, r_w = orc.backprop(s, st, 12, nseg, seeder)
    ctx = Context(s, st.particles.size())
    c_g, pg_g, r_g = ctx.backprop(st, 12, nseg, seeder)
    assert r_g.loss == pytest.approx(r_w.loss, rel=1e-10)
    assert r_g.peak_replay_states == r_w.peak_replay_states and r_g.checkpoints_stored == nseg
    errs = cot_errs(c_g, c_w)
    assert all(v < 1e-8 for v in errs.values()), errs
    assert rel_err(pg_g.wall_friction[2], pg_w.wall_friction[2], 1e-300) < 1e-8


def test_backprop_segment_invariance_bitwise():
    """SPEC.md:393 / acceptance 6: dL/d(state_0) bit-identical for n_segments in {1, 2, 5, 10}."""
    s = fluid_box_scene(2, kind="flip")
    st = init_scene(s)
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.advance(20)
    fin = ctx.download(st.copy())
    seeder = _seeder_final_x(fin, 20)
    outs = []
    for nseg in (1, 2, 5, 10):
        c, pg, r = ctx.backprop(st, 20, nseg, seeder)
        outs.append((c, pg, r))
    c0 = outs[0][0]
    for c, pg, r in outs[1:]:
        for f in StateCotangent.FIELDS:
            a, b = getattr(c, f), getattr(c0, f)
            if a is not None:
                assert np.array_equal(a, b), f
        assert pg.sound_speed == outs[0][1].sound_speed and r.loss == outs[0][2].loss


def test_free_flight_velocity_cotangent():
    """a single free particle (no forces, PIC), seeding x_bar = 1 at step N gives
    v_bar(0) = N dt."""
    s = small_fluid_scene("pic")
    s.mass_epsilon = 1e-15
    from helpers import single_particle_state
    st = single_particle_state(s, [0.513, 0.497], [0.0, 0.0])
    N = 10
    # loss = sum (x - (x_N - 1/2))^2 -> seed 2 (x - target) = 1 per component at step N
    fin = st.copy()
    ctx = Context(s, 1)
    ctx.upload(fin)
    ctx.advance(N)
    fin = ctx.download(fin)
    seeder = {"field": "x", "obs_steps": [N], "sel": None, "target": fin.particles.x[None] - 0.5}
    c, pg, r = ctx.backprop(st, N, 2, seeder)
    assert np.allclose(c.v[0], N * s.config.dt, rtol=1e-10)


def test_finite_difference_initial_velocity():
    """SPEC.md:386 / acceptance 5 (reduced): directional derivative of L(v0) vs central FD, f64."""
    s = small_fluid_scene("flip")
    s.config.gravity = [0.0, -9.8]
    s.geometry[0] = GeometryRegion(lo=[0.3, 0.1], hi=[0.6, 0.4], velocity=VelocityExpr("linear_in_y", alpha=1.0, h0=0.3))
    st = init_scene(s)
    N = 30
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.advance(N)
    tgt = ctx.download(st.copy()).particles.x + 0.003
    seeder = {"field": "x", "obs_steps": [N], "sel": None, "target": tgt[None]}
    c, pg, r = ctx.backprop(st, N, 3, seeder)

    def loss(v0):
        s1 = st.copy()
        s1.particles.v[...] = v0
        ctx.upload(s1)
        ctx.advance(N)
        x = ctx.download(s1).particles.x
        return float(((x - tgt) ** 2).sum())

    rng = np.random.default_rng(5)
    for _ in range(4):
        d = rng.standard_normal(st.particles.v.shape)
        h = 1e-6
        fd = (loss(st.particles.v + h * d) - loss(st.particles.v - h * d)) / (2 * h)
        an = float((c.v * d).sum())
        assert abs(fd - an) <= 1e-5 * (abs(fd) + 1e-12), (fd, an)


@pytest.mark.parametrize("name", ["fluid2-flip", "fluid2-tpic-rate", "dp2-coulomb-obstacle", "dp3-coulomb",
                                  "fluid3-apic"])
@pytest.mark.parametrize("cap", [None, "1"])
def test_backprop_replay_tape_bitwise(name, cap, monkeypatch):
    """The replay tape (the segment replay's sort and grid reused by step_vjp) changes nothing:
    bit-identical to recomputing the forward replay inside every step_vjp. cap=1 forces every
    step's grid to overflow its slot (the recompute fallback)."""
    s = SCENES[name]()
    st = init_scene(s)
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.advance(9)
    seeder = _seeder_final_x(ctx.download(st.copy()), 9)
    ctx.close()
    monkeypatch.setenv("MPM_TAPE", "0")
    ctx0 = Context(s, st.particles.size())
    c_ref, pg_ref, r_ref = ctx0.backprop(st, 9, 2, seeder)
    ctx0.close()
    monkeypatch.setenv("MPM_TAPE", "1")
    if cap:
        monkeypatch.setenv("MPM_TAPE_CAP", cap)
    ctx1 = Context(s, st.particles.size())
    for _ in range(2):  # the second call reuses the persistent tape slots
        c, pg, r = ctx1.backprop(st, 9, 2, seeder)
        for f in StateCotangent.FIELDS:
            a, b = getattr(c, f), getattr(c_ref, f)
            if a is not None:
                assert np.array_equal(a, b), f
        assert r.loss == r_ref.loss
        assert pg.sound_speed == pg_ref.sound_speed and pg.viscosity == pg_ref.viscosity
        for w in range(2 * s.dim):
            if pg_ref.wall_friction[w] is not None:
                assert np.array_equal(pg.wall_friction[w], pg_ref.wall_friction[w])
    ctx1.close()


def _dp3_many_blocks():
    s = dp_block_scene(3, coulomb=True, cells=[200, 100, 110])
    s.config.dh = 0.005  # 2.24 M particles in ~630 occupied blocks: several blocks per CTA
    return s


@pytest.mark.parametrize("name", ["dp3-coulomb", "fluid3-apic", "dp3-many-blocks"])
def test_block_scheduling_bitwise(name, monkeypatch):
    """3-D kernels take occupied blocks heaviest first through work counters (common.cuh).
    Every block's outputs depend only on the block, so the forward state and the backprop
    results are bit-identical to the static CTA stride (MPM_OCC_ORDER=index); a second call
    checks that the counters were reset by the last CTA of every launch."""
    s = _dp3_many_blocks() if name == "dp3-many-blocks" else SCENES[name]()
    st = init_scene(s)
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.advance(9)
    seeder = _seeder_final_x(ctx.download(st.copy()), 9)
    ctx.close()
    out = {}
    for order in ("index", "lpt"):
        monkeypatch.setenv("MPM_OCC_ORDER", order)
        c1 = Context(s, st.particles.size())
        runs = []
        for _ in range(2):
            c1.upload(st)
            c1.advance(7)
            fwd = c1.download(st.copy())
            runs.append((fwd, c1.backprop(st, 9, 2, seeder)))
        c1.close()
        out[order] = runs
    ref_fwd, (c_ref, pg_ref, r_ref) = out["index"][0]
    for fwd, (c, pg, r) in out["index"][1:] + out["lpt"]:
        for f in ("x", "v", "sigma", "rho", "volume", "grad_v"):
            assert np.array_equal(getattr(fwd.particles, f), getattr(ref_fwd.particles, f)), f
        for f in StateCotangent.FIELDS:
            a, b = getattr(c, f), getattr(c_ref, f)
            if a is not None:
                assert np.array_equal(a, b), f
        assert r.loss == r_ref.loss
        assert pg.sound_speed == pg_ref.sound_speed and pg.viscosity == pg_ref.viscosity
        for w in range(2 * s.dim):
            if pg_ref.wall_friction[w] is not None:
                assert np.array_equal(pg.wall_friction[w], pg_ref.wall_friction[w])
