"""Device scene seeding: init_scene on the GPU must give the host init_scene's
particles (which are pinned bit-identical to the reference's init_scene by test_oracle_golden), in
the same order and with the same bits; parabolic_sine differs only through sin."""
from __future__ import annotations

import time

import numpy as np
import pytest

from paper_2507_04192_b200 import init_scene
from paper_2507_04192_b200.presets import c1_column, c3_inverse, c4_column3d, small_fluid_scene
from paper_2507_04192_b200.scene import GeometryRegion, Scene, VelocityExpr, Wall
from paper_2507_04192_b200.solver import init_scene_device

from test_distributed import moving_fluid_scene

pytestmark = pytest.mark.gpu


def cylinder_scene(dtype="f64"):
    from paper_2507_04192_b200.presets import bui_sand

    s = Scene(3, dtype)
    c = s.config
    c.dh, c.cells, c.dt, c.gravity = 0.02, [24, 20, 16], 1e-5, [0.0, -9.8, 0.0]
    c.scheme.kind = "flip"
    s.material = bui_sand()
    s.boundary.walls[2] = Wall("no_slip")
    s.geometry.append(GeometryRegion(shape="cylinder", center=[0.2, 0.2, 0.0], radius=0.12, zmin=0.05, zmax=0.25,
                                     velocity=VelocityExpr("constant", value=[0.5, 0.0, 0.1])))
    s.geometry.append(GeometryRegion(lo=[0.15, 0.05, 0.05], hi=[0.40, 0.15, 0.27],
                                     velocity=VelocityExpr("linear_in_y", alpha=2.0, h0=0.1)))
    return s


def sine_scene():
    s = small_fluid_scene("flip")
    s.geometry[0].velocity = VelocityExpr("parabolic_sine", h0=0.4, amplitude=1.0, perturbation=0.3, frequency=3.0)
    return s


SCENES = {
    "fluid2": lambda: small_fluid_scene("flip"),
    "c1": lambda: c1_column(),
    "c1-f32": lambda: c1_column("f32"),
    "c3-linear": lambda: c3_inverse(),
    "moving3": lambda: moving_fluid_scene(3),
    "cylinder3": lambda: cylinder_scene(),
    "cylinder3-f32": lambda: cylinder_scene("f32"),
}


@pytest.mark.parametrize("name", list(SCENES))
def test_device_seeding_bitwise(name):
    s = SCENES[name]()
    want = init_scene(s)
    eps_host = s.mass_epsilon
    ctx = init_scene_device(s)
    assert s.mass_epsilon == eps_host
    got = ctx.download(want.copy())
    ctx.close()
    for f in ("x", "v", "mass", "volume", "rho", "eps_eq", "sigma", "grad_v"):
        assert np.array_equal(getattr(got.particles, f), getattr(want.particles, f)), f


def test_device_seeding_parabolic_sine_close():
    s = sine_scene()
    want = init_scene(s)
    ctx = init_scene_device(s)
    got = ctx.download(want.copy())
    ctx.close()
    assert np.array_equal(got.particles.x, want.particles.x)
    assert np.allclose(got.particles.v, want.particles.v, rtol=0, atol=1e-15)


def test_device_seeding_c4_speed():
    """C4: 4.2 M particles seeded on the device, identical to the host seeding; the seeding call
    itself (context already created) is timed against the host's"""
    from paper_2507_04192_b200.scene import seeding_capacity
    from paper_2507_04192_b200.solver import Context

    s = c4_column3d()
    t0 = time.perf_counter()
    want = init_scene(s)
    t_host = time.perf_counter() - t0
    ctx = Context(s, seeding_capacity(s))
    ctx.init_scene(s)  # warm (module load)
    t0 = time.perf_counter()
    n = ctx.init_scene(s)
    t_dev = time.perf_counter() - t0
    got = ctx.download(want.copy())
    ctx.close()
    assert n == want.particles.size() == 4194304
    assert np.array_equal(got.particles.x, want.particles.x)
    assert t_dev < t_host
    print(f"C4 seeding: host {t_host * 1e3:.0f} ms, device {t_dev * 1e3:.1f} ms")


def test_device_seeding_capacity_and_cfl():
    from paper_2507_04192_b200.errors import MPMError, ValidationError

    s = small_fluid_scene("flip")
    with pytest.raises(MPMError):
        init_scene_device(s, capacity=10)  # more particles than the context holds
    s.geometry[0].velocity = VelocityExpr("constant", value=[5000.0, 0.0])
    with pytest.raises(ValidationError):
        init_scene_device(s)  # init_scene's CFL refusal


def test_run_async_snapshots_equal_synchronous_downloads():
    """run's snapshots (two asynchronous slots, reused) equal plain downloads at the same steps"""
    from paper_2507_04192_b200.solver import Context, run

    s = c1_column()
    st = init_scene(s)
    res = run(s, st, 40, 5)
    assert [x.step for x in res.snapshots] == list(range(0, 41, 5))
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    for snap in res.snapshots[1:]:
        ctx.advance(5, nan_guard=True)
        want = ctx.download(st.copy())
        assert want.step == snap.step and want.time == snap.time
        for f in ("x", "v", "sigma", "rho", "volume", "grad_v", "eps_eq", "sigma_zz"):
            assert np.array_equal(getattr(snap.particles, f), getattr(want.particles, f)), (snap.step, f)
    ctx.close()
