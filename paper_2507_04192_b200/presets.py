"""Scene presets: the reference test fixtures (tests/helpers.hpp) and the BASELINE.json configs
C1-C5 restated in SURVEY.md §8(d)."""
from __future__ import annotations

import math

from .scene import (DruckerPragerParams, FluidParams, GeometryRegion, Scene, VelocityExpr, Wall)

BUI_PHI = 19.8 * math.pi / 180.0


def bui_sand(cohesion=0.0, sigma_t=0.0) -> DruckerPragerParams:
    """test_constitutive.cpp:13-17 / PAPER.md:671 granular material."""
    return DruckerPragerParams.make(2650.0, 0.7e6, 0.3, BUI_PHI, 0.0, cohesion, sigma_t)


def small_fluid_scene(kind="pic", alpha_flip=1.0, dtype="f64") -> Scene:
    """tests/helpers.hpp:11-29: 20x20 cells, dh 0.05, fluid c = 20, no gravity."""
    s = Scene(2, dtype)
    c = s.config
    c.dh, c.cells, c.dt, c.gravity = 0.05, [20, 20], 1e-4, [0.0, 0.0]
    c.scheme.kind, c.scheme.alpha_flip = kind, alpha_flip
    s.material = FluidParams(1000.0, 0.0, 20.0)
    s.geometry.append(GeometryRegion(lo=[0.3, 0.3], hi=[0.7, 0.7]))
    return s


def c1_column(dtype="f64") -> Scene:
    """C1: 2-D Bui column, 0.2 x 0.1 m (100 x 50 cells at dh 0.002) in 128^2, D-P sand,
    FLIP, bottom no-slip, others slip, dt 1e-5 -> 20,000 particles."""
    s = Scene(2, dtype)
    c = s.config
    c.dh, c.cells, c.dt, c.gravity = 0.002, [128, 128], 1e-5, [0.0, -9.8]
    c.scheme.kind = "flip"
    s.material = bui_sand()
    s.boundary.walls[2] = Wall("no_slip")
    s.geometry.append(GeometryRegion(lo=[2 * 0.002, 2 * 0.002], hi=[2 * 0.002 + 0.2, 2 * 0.002 + 0.1]))
    return s


def c2_dam_break(dtype="f64") -> Scene:
    """C2: 2-D water column 0.5 x 0.5 m (250^2 cells at dh 0.002) in 512^2, fluid c 35,
    all slip, FLIP, dt 1e-5 -> 250,000 particles."""
    s = Scene(2, dtype)
    c = s.config
    c.dh, c.cells, c.dt, c.gravity = 0.002, [512, 512], 1e-5, [0.0, -9.8]
    c.scheme.kind = "flip"
    s.material = FluidParams(1000.0, 0.0, 35.0)
    s.geometry.append(GeometryRegion(lo=[0.004, 0.004], hi=[0.004 + 0.5, 0.004 + 0.5]))
    return s


def c3_inverse(alpha=0.1, dtype="f64") -> Scene:
    """C3: §5.1 inverse, H0 = L0 = 0.5 (160^2 cells at dh 1/320) in a 1.5 x 0.6 m domain
    (480 x 192), fluid c 50, all slip, v_x0 = alpha (H0 - y), dt 3e-5 -> 102,400 particles."""
    s = Scene(2, dtype)
    c = s.config
    dh = 1.0 / 320.0
    c.dh, c.cells, c.dt, c.gravity = dh, [480, 192], 3e-5, [0.0, -9.8]
    c.scheme.kind = "flip"
    s.material = FluidParams(1000.0, 0.0, 50.0)
    s.geometry.append(GeometryRegion(lo=[2 * dh, 2 * dh], hi=[2 * dh + 0.5, 2 * dh + 0.5],
                                     velocity=VelocityExpr("linear_in_y", alpha=alpha, h0=0.5)))
    return s


def c4_column3d(dtype="f64", replicas_x: int = 1) -> Scene:
    """C4: 3-D column 0.5 x 0.25 x 0.25 m (128 x 64 x 64 cells, axis 1 vertical) at dh 1/256
    in 256^3 cells, D-P sand, FLIP, bottom no-slip, others slip, dt 1e-5 -> 4,194,304
    particles. replicas_x > 1 gives the weak-scaling domain 256G x 256 x 256 with G columns."""
    s = Scene(3, dtype)
    c = s.config
    dh = 1.0 / 256.0
    c.dh, c.cells, c.dt, c.gravity = dh, [256 * replicas_x, 256, 256], 1e-5, [0.0, -9.8, 0.0]
    c.scheme.kind = "flip"
    s.material = bui_sand()
    s.boundary.walls[2] = Wall("no_slip")
    for r in range(replicas_x):
        x0 = 256 * r * dh + 2 * dh
        s.geometry.append(GeometryRegion(lo=[x0, 2 * dh, 2 * dh], hi=[x0 + 0.5, 2 * dh + 0.25, 2 * dh + 0.25]))
    return s


def c5_landslide(dtype="f64", n_segments=32) -> Scene:
    """C5: 3-D block 1.0 x 0.5 x 0.484 m (256 x 128 x 124 cells) at dh 1/256 in 512 x 256 x 128
    cells, v0 = (2, 0, 0), D-P sand, bottom Coulomb wall with 32 segments along x,
    mu_k = 0.3 + 0.2 sin(2 pi k / 32), others slip, dt 1e-5 -> 32,505,856 particles."""
    s = Scene(3, dtype)
    c = s.config
    dh = 1.0 / 256.0
    c.dh, c.cells, c.dt, c.gravity = dh, [512, 256, 128], 1e-5, [0.0, -9.8, 0.0]
    c.scheme.kind = "flip"
    s.material = bui_sand()
    s.boundary.walls[2] = Wall("coulomb", [0.3 + 0.2 * math.sin(2 * math.pi * k / n_segments)
                                           for k in range(n_segments)])
    s.geometry.append(GeometryRegion(lo=[2 * dh, 2 * dh, 2 * dh], hi=[2 * dh + 1.0, 2 * dh + 0.5, 2 * dh + 0.484375],
                                     velocity=VelocityExpr("constant", value=[2.0, 0.0, 0.0])))
    return s


def c5_landslide_eighth(dtype="f64", n_segments=32) -> Scene:
    """C5 with 1/8 of its particles (4,063,232): the same 512 x 256 x 128 grid, material, dt and
    32-segment Coulomb floor; the block keeps its 1.0 m along x (segments 0-15 under it, as in
    full C5) and v0 = (2, 0, 0), with half the height and a quarter of the width. Used where the
    full scene's 7.3 GB host copies do not fit (parity tests, CPU samples)."""
    s = c5_landslide(dtype, n_segments)
    dh = s.config.dh
    s.geometry[0] = GeometryRegion(lo=[2 * dh, 2 * dh, 2 * dh], hi=[2 * dh + 1.0, 2 * dh + 0.25, 2 * dh + 31 * dh],
                                   velocity=VelocityExpr("constant", value=[2.0, 0.0, 0.0]))
    return s


CONFIGS = {"C1": c1_column, "C2": c2_dam_break, "C3": c3_inverse, "C4": c4_column3d, "C5": c5_landslide,
           "C5/8": c5_landslide_eighth}
