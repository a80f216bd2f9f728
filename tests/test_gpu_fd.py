"""Gradient correctness by central finite differences (acceptance criterion 5):
a 2-D scene of ~400 particles, 200 steps, f64, >= 20 random directions per parameter class,
relative error against central differences < 1e-5. Run on a fluid scene and a Drucker-Prager
scene, both sliding over a 4-segment Coulomb floor.

Parameter classes (ParamGrads, adjoint.hpp:77-90, and the t = 0 cotangent):
  * the initial velocity field v0 (R^{2N}): 20 random directions;
  * the scalar initial-velocity parameter alpha of v_x(0) = alpha (h0 - y_rel), y_rel measured
    from the region's bottom (config.hpp:92-96; the C3 inverse parameter):
    dL/dalpha = sum_p vbar_x,p(0) v_x,p(0) / alpha, at 20 random alphas;
  * the 4 Coulomb friction segments of the floor (adjoint.hpp:145): 20 random directions in R^4;
  * the fluid sound speed c (adjoint.hpp:153-184, fluid scene only): 20 random values.
The MLP weights of SPEC's third class are out of scope (Mlp::vjp chains the t = 0
cotangent on the host, off the hot path).

Loss: the Lagrangian least-squares seeder on every particle's final position,
run entirely on the device (mpm_backprop); the finite differences re-run the forward on the
device with the perturbed parameter.
"""
import numpy as np
import pytest

from paper_2507_04192_b200 import FluidParams, GeometryRegion, Scene, VelocityExpr, Wall, init_scene
from paper_2507_04192_b200.presets import bui_sand
from paper_2507_04192_b200.solver import Context

pytestmark = pytest.mark.gpu

N_STEPS = 200
N_DIRS = 20
RTOL = 1e-5
H0 = 0.2


def sliding_layer(material: str, alpha=1.0, c=20.0, friction=(0.15, 0.3, 0.2, 0.4)):
    """A 0.9 x 0.075 m layer (432 particles) over a 4-segment Coulomb floor, v_x(0) = alpha (h0 - y)."""
    s = Scene(2, "f64")
    cfg = s.config
    cfg.dh, cfg.cells, cfg.dt, cfg.gravity = 0.025, [40, 40], 1e-4, [0.0, -9.8]
    cfg.scheme.kind = "flip"
    s.material = FluidParams(1000.0, 0.0, c) if material == "fluid" else bui_sand()
    s.boundary.walls[2] = Wall("coulomb", list(friction))
    s.geometry.append(GeometryRegion(lo=[0.05, 0.05], hi=[0.95, 0.125],
                                     velocity=VelocityExpr("linear_in_y", alpha=alpha, h0=H0)))
    init_scene(s)  # sets Scene::mass_epsilon (scene.hpp:107), which the step reads
    return s


def initial_state(s, kind):
    """init_scene, plus for the Drucker-Prager layer a geostatic compression (2 kPa + rho g depth
    on sigma_xx, sigma_yy and the plane-strain sigma_zz): with c = 0 the seeded sigma = 0 is the
    cone's apex, where the return map is not differentiable (adjoint.hpp:234-235 gives it a zero
    cotangent); a compressed layer starts inside the cone and yields by smooth radial returns."""
    st = init_scene(s)
    if kind == "dp":
        p = st.particles
        depth = 0.125 - p.x[:, 1]
        press = 2000.0 + s.material.rho0 * 9.8 * depth
        p.sigma[:, 0, 0] = -press
        p.sigma[:, 1, 1] = -press
        p.sigma_zz[:] = -press
    return st


def final_x(s, st):
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.advance(N_STEPS)
    x = ctx.download(st.copy()).particles.x
    ctx.close()
    return x


def gradient(s, st, target):
    ctx = Context(s, st.particles.size())
    c0, pg, res = ctx.backprop(st, N_STEPS, 4, {"field": "x", "obs_steps": [N_STEPS], "sel": None,
                                                "target": target[None]})
    ctx.close()
    return c0, pg, res.loss


def loss_of(s, st, target):
    return float(((final_x(s, st) - target) ** 2).sum())


def check(fd, an, what):
    assert abs(fd - an) <= RTOL * abs(fd), f"{what}: FD {fd!r} vs adjoint {an!r} (rel {abs(fd - an) / abs(fd):.2e})"


@pytest.fixture(scope="module", params=["fluid", "dp"])
def setup(request):
    s = sliding_layer(request.param)
    st = initial_state(s, request.param)
    assert 400 <= st.particles.size() <= 450
    target = final_x(s, st) + 0.003
    c0, pg, loss = gradient(s, st, target)
    return request.param, s, st, target, c0, pg, loss


def test_fd_initial_velocity_field(setup):
    kind, s, st, target, c0, pg, loss = setup
    assert abs(loss - loss_of(s, st, target)) <= 1e-12 * loss
    rng = np.random.default_rng(613)
    for k in range(N_DIRS):
        d = rng.standard_normal(st.particles.v.shape)
        h = 1e-6
        sp, sm = st.copy(), st.copy()
        sp.particles.v += h * d
        sm.particles.v -= h * d
        fd = (loss_of(s, sp, target) - loss_of(s, sm, target)) / (2 * h)
        check(fd, float((c0.v * d).sum()), f"{kind} v0 direction {k}")


def test_fd_scalar_alpha(setup):
    kind, s, st, target, _, _, _ = setup
    rng = np.random.default_rng(878)
    for k in range(N_DIRS):
        alpha = float(rng.uniform(0.2, 2.0))
        sa = sliding_layer(kind, alpha=alpha)
        sta = initial_state(sa, kind)
        c0, _, _ = gradient(sa, sta, target)
        an = float(np.sum(c0.v[:, 0] * sta.particles.v[:, 0]) / alpha)  # dv_x(0)/dalpha = h0 - y_rel
        h = 1e-6
        fd = (loss_of(sa, initial_state(sliding_layer(kind, alpha=alpha + h), kind), target)
              - loss_of(sa, initial_state(sliding_layer(kind, alpha=alpha - h), kind), target)) / (2 * h)
        check(fd, an, f"{kind} alpha={alpha:.4f}")


def test_fd_friction_segments(setup):
    kind, s, st, target, _, pg, _ = setup
    mu = np.array(s.boundary.walls[2].friction)
    an_grad = np.asarray(pg.wall_friction[2])
    assert an_grad.shape == (4,) and np.count_nonzero(an_grad) == 4, an_grad
    rng = np.random.default_rng(145)
    for k in range(N_DIRS):
        d = rng.standard_normal(4)
        h = 1e-6
        lp = loss_of(sliding_layer(kind, friction=mu + h * d), st, target)
        lm = loss_of(sliding_layer(kind, friction=mu - h * d), st, target)
        check((lp - lm) / (2 * h), float(an_grad @ d), f"{kind} friction direction {k}")


def test_fd_sound_speed(setup):
    kind, s, st, target, _, _, _ = setup
    if kind != "fluid":
        pytest.skip("the reference has no Drucker-Prager parameter gradient (SPEC.md:416)")
    rng = np.random.default_rng(153)
    for k in range(N_DIRS):
        c = float(rng.uniform(15.0, 25.0))
        sc = sliding_layer(kind, c=c)
        _, pg, _ = gradient(sc, st, target)
        h = 1e-5
        fd = (loss_of(sliding_layer(kind, c=c + h), st, target) - loss_of(sliding_layer(kind, c=c - h), st, target)) / (2 * h)
        check(fd, pg.sound_speed, f"fluid c={c:.3f}")
