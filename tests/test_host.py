"""Host-side logic: presets, checkpoint plan, scene validation, descriptor packing."""
import math

import numpy as np
import pytest

from paper_2507_04192_b200 import FluidParams, GeometryRegion, Scene, Wall, init_scene
from paper_2507_04192_b200.errors import ValidationError
from paper_2507_04192_b200.presets import c1_column, c2_dam_break, c3_inverse, c5_landslide
from paper_2507_04192_b200.solver import CheckpointPlan


@pytest.mark.parametrize("fn,n", [(c1_column, 20000), (c2_dam_break, 250000), (c3_inverse, 102400)])
def test_preset_particle_counts(fn, n):
    s = fn()
    assert init_scene(s).particles.size() == n
    assert s.mass_epsilon > 0


def test_c5_descriptor_and_count():
    s = c5_landslide()
    d = s.to_desc().desc
    assert d.n_friction[2] == 32 and abs(d.friction[2][8] - 0.5) < 1e-15
    cells = [256, 128, 124]
    assert math.prod(cells) * 8 == 32505856


def test_checkpoint_plan_matches_reference():
    """checkpoint.hpp:15-34 and SPEC make_plan examples"""
    p = CheckpointPlan.make(10, 3)
    assert p.boundaries == [0, 4, 7, 10]
    assert CheckpointPlan.make(10, 1).boundaries == [0, 10]
    assert p.planned_peak_states() == 3 + 4 + 1
    with pytest.raises(ValidationError):
        CheckpointPlan.make(10, 11)
    with pytest.raises(ValidationError):
        CheckpointPlan.make(0, 1)


def test_scene_validation():
    s = Scene(2)
    s.config.dh, s.config.cells, s.config.dt = 0.05, [20, 20], 1e-4
    s.material = FluidParams(1000.0, 0.0, 20.0)
    with pytest.raises(ValidationError):
        init_scene(s)  # no geometry
    s.geometry.append(GeometryRegion(lo=[0.3, 0.3], hi=[0.7, 0.7]))
    s.boundary.walls[2] = Wall("coulomb", [])
    with pytest.raises(ValidationError):
        init_scene(s)
    s.boundary.walls[2] = Wall("coulomb", [0.3])
    s.config.dt = 1.0
    with pytest.raises(ValidationError):
        init_scene(s)  # fluid CFL


def test_f32_seeding_matches_reference_layout():
    s = c1_column("f32")
    st = init_scene(s)
    assert st.particles.x.dtype == np.float32 and st.particles.size() == 20000


def test_presets_build_with_dtype_keyword():
    """bench.py builds every config as CONFIGS[name](dtype=...); C1-C3 seed on the host here"""
    from paper_2507_04192_b200 import init_scene
    from paper_2507_04192_b200.presets import CONFIGS

    for name, make in CONFIGS.items():
        for dt in ("f64", "f32"):
            s = make(dtype=dt)
            assert s.np_dtype == (np.float64 if dt == "f64" else np.float32), name
            if name in ("C1", "C3"):
                n = init_scene(s).particles.size()
                assert n == {"C1": 20000, "C3": 102400}[name]
