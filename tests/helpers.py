"""Shared test fixtures: the reference's own scene builders (tests/helpers.hpp) plus parity helpers."""
from __future__ import annotations

import math

import numpy as np

from paper_2507_04192_b200 import (DruckerPragerParams, FluidParams, GeometryRegion, Obstacle, ParticleSoA,
                                   Scene, SimState, VelocityExpr, Wall, init_scene)
from paper_2507_04192_b200.presets import bui_sand, small_fluid_scene  # noqa: F401

# physical floors for relative comparisons (a field that is pure roundoff, e.g. grad v of a
# block in free fall, is compared against this scale instead of its own ~1e-16 magnitude)
FLOORS = {"x": 1.0, "v": 1e-2, "mass": 1e-12, "volume": 1e-12, "rho": 1.0, "eps_eq": 1e-9, "sigma_zz": 1.0,
          "sigma": 1.0, "grad_v": 1.0, "affine": 1e-6, "def_grad": 1.0}


def rel_err(a, b, floor=0.0):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    scale = max(float(np.abs(b).max()), floor, 1e-300)
    return float(np.abs(a - b).max()) / scale


def assert_state_close(got: SimState, ref: SimState, rtol: float, fields=None, what=""):
    fields = fields or [f for f in ParticleSoA.FIELDS if getattr(ref.particles, f) is not None]
    errs = {}
    for f in fields:
        a, b = getattr(got.particles, f), getattr(ref.particles, f)
        if b is None or b.size == 0:
            continue
        errs[f] = rel_err(a, b, FLOORS.get(f, 0.0))
    bad = {k: v for k, v in errs.items() if not v <= rtol}
    assert not bad, f"{what} parity failed (rtol {rtol:g}): " + ", ".join(f"{k}={v:.3e}" for k, v in errs.items())
    return errs


def assert_grid_close(got, ref, rtol, what=""):
    errs = {}
    for f in ("mass", "momentum", "v_old", "v", "force"):
        a, b = getattr(got, f), getattr(ref, f)
        errs[f] = rel_err(a, b, 1e-300)
    bad = {k: v for k, v in errs.items() if not v <= rtol}
    assert not bad, f"{what} grid parity failed (rtol {rtol:g}): " + ", ".join(f"{k}={v:.3e}" for k, v in errs.items())


def random_block(scene, seed, lo=-1.0, hi=1.0):
    """test_transfer.cpp:35-44: init_scene then i.i.d. U(lo, hi) velocities (our RNG)."""
    st = init_scene(scene)
    rng = np.random.default_rng(seed)
    st.particles.v[...] = rng.uniform(lo, hi, st.particles.v.shape)
    return st


def single_particle_state(scene, x, v):
    """tests/helpers.hpp:33-45"""
    st = SimState.zeros(1, scene.dim, scene.np_dtype, scene.config.scheme.uses_affine(), False)
    dh = scene.config.dh
    st.particles.x[0] = x
    st.particles.v[0] = v
    st.particles.mass[0] = 1000.0 * dh * dh / 4
    st.particles.rho[0] = 1000.0
    st.particles.volume[0] = st.particles.mass[0] / 1000.0
    return st


def dp_block_scene(dim=2, dtype="f64", kind="flip", coulomb=False, obstacle=False, cells=None):
    """A D-P block resting on the floor (exercises all three return-map zones)."""
    s = Scene(dim, dtype)
    c = s.config
    c.dh = 0.05
    c.cells = cells or [20] * dim
    c.dt = 1e-5
    c.gravity = [0.0, -9.8] + [0.0] * (dim - 2)
    c.scheme.kind = kind
    s.material = bui_sand()
    s.boundary.walls[2] = Wall("coulomb", [0.1, 0.4, 0.2]) if coulomb else Wall("no_slip")
    hi = [0.5, 0.35, 0.45][:dim]
    s.geometry.append(GeometryRegion(lo=[0.1] * dim, hi=hi, velocity=VelocityExpr("constant", value=[1.5, 0.0, -0.5][:dim])))
    if obstacle:
        s.obstacles.append(Obstacle([0.6, 0.0, 0.0][:dim], [0.8, 0.3, 0.55][:dim]))
    return s


def fluid_box_scene(dim=2, dtype="f64", kind="flip", alpha=0.5, gravity=True, visc=0.0, rate_form=False):
    s = Scene(dim, dtype)
    c = s.config
    c.dh = 0.05
    c.cells = [20] * dim
    c.dt = 1e-4
    c.gravity = ([0.0, -9.8] + [0.0] * (dim - 2)) if gravity else [0.0] * dim
    c.scheme.kind = kind
    c.scheme.alpha_flip = alpha
    s.material = FluidParams(1000.0, visc, 20.0, rate_form)
    s.geometry.append(GeometryRegion(lo=[0.1] * dim, hi=[0.6, 0.5, 0.4][:dim],
                                     velocity=VelocityExpr("constant", value=[0.8, -0.3, 0.2][:dim])))
    return s
