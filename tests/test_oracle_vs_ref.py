"""Pin the restated oracle against the reference itself (compiled unmodified against the
Eigen-API shim, oracle/_ref): bit-identical forward states and adjoint cotangents."""
import numpy as np
import pytest

from helpers import dp_block_scene, fluid_box_scene
from paper_2507_04192_b200 import ParticleSoA, StateCotangent, init_scene

SCENES = {
    "fluid2-pic": lambda: fluid_box_scene(2, kind="pic"),
    "fluid2-flip": lambda: fluid_box_scene(2, kind="flip"),
    "fluid2-blend": lambda: fluid_box_scene(2, kind="blend", alpha=0.3),
    "fluid2-apic": lambda: fluid_box_scene(2, kind="apic"),
    "fluid2-tpic-visc": lambda: fluid_box_scene(2, kind="tpic", visc=0.5, rate_form=True),
    "dp2-noslip": lambda: dp_block_scene(2),
    "dp2-coulomb-obstacle": lambda: dp_block_scene(2, coulomb=True, obstacle=True),
    "dp3": lambda: dp_block_scene(3, cells=[12, 12, 12]),
    "fluid3-apic": lambda: fluid_box_scene(3, kind="apic"),
    "dp2-f32": lambda: dp_block_scene(2, dtype="f32"),
}


def _bits_equal(a, b):
    return a is None or a.size == 0 or np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("name", sorted(SCENES))
def test_forward_bit_identical(orc, ref, name):
    s = SCENES[name]()
    st = init_scene(s)
    a, b = st.copy(), st.copy()
    orc.advance(s, a, 15)
    ref.advance(s, b, 15)
    for f in ParticleSoA.FIELDS:
        assert _bits_equal(getattr(a.particles, f), getattr(b.particles, f)), f
    assert orc.state_hash(s, a) == ref.state_hash(s, b)


@pytest.mark.parametrize("name", sorted(SCENES))
def test_step_vjp_bit_identical(orc, ref, name):
    s = SCENES[name]()
    st = init_scene(s)
    orc.advance(s, st, 10)
    rng = np.random.default_rng(3)
    cot = StateCotangent.zeros_like(st.particles)
    for f in StateCotangent.FIELDS:
        a = getattr(cot, f)
        if a is not None and a.size and f != "eps_eq":
            a[...] = rng.standard_normal(a.shape)
    ci_o, pg_o = orc.step_vjp(s, st, cot)
    ci_r, pg_r = ref.step_vjp(s, st, cot)
    for f in StateCotangent.FIELDS:
        assert _bits_equal(getattr(ci_o, f), getattr(ci_r, f)), f
    assert pg_o.sound_speed == pg_r.sound_speed and pg_o.viscosity == pg_r.viscosity
    for w in range(6):
        assert np.array_equal(pg_o.wall_friction[w], pg_r.wall_friction[w])


@pytest.mark.parametrize("nseg", [1, 3])
def test_backprop_bit_identical(orc, ref, nseg):
    s = dp_block_scene(2, coulomb=True)
    st = init_scene(s)
    fin = st.copy()
    orc.advance(s, fin, 9)
    seeder = {"field": "x", "obs_steps": [5, 9], "sel": None,
              "target": np.stack([fin.particles.x + 0.01, fin.particles.x - 0.02])}
    c_o, pg_o, r_o = orc.backprop(s, st, 9, nseg, seeder)
    c_r, pg_r, r_r = ref.backprop(s, st, 9, nseg, seeder)
    assert r_o.loss == r_r.loss and r_o.peak_replay_states == r_r.peak_replay_states
    for f in StateCotangent.FIELDS:
        assert _bits_equal(getattr(c_o, f), getattr(c_r, f)), f
    assert np.array_equal(pg_o.wall_friction[2], pg_r.wall_friction[2])
