"""K1, the incremental cell sort (kernels_sort.cuh, north_star item (1)).

The sort must return exactly the permutation of the full radix sort of (cell key, storage index)
(the canonical order of SPEC.md:149,155): a different order changes every P2G sum at rounding
level. So a context with the incremental sort and one forced onto the radix sort for every step
(MPM_SORT=cub, read when a context is created) must give BIT-IDENTICAL states after many steps,
and bit-identical gradients through backprop_trajectory (the replay tape path).
"""
import os

import numpy as np
import pytest

from helpers import dp_block_scene, fluid_box_scene
from paper_2507_04192_b200 import GeometryRegion, Scene, FluidParams, init_scene
from paper_2507_04192_b200.presets import c1_column
from paper_2507_04192_b200.solver import Context

pytestmark = pytest.mark.gpu

FIELDS = ("x", "v", "sigma", "rho", "volume", "grad_v")


def make_ctx(s, n, sort):
    old = os.environ.get("MPM_SORT")
    os.environ["MPM_SORT"] = sort
    try:
        return Context(s, n)
    finally:
        if old is None:
            del os.environ["MPM_SORT"]
        else:
            os.environ["MPM_SORT"] = old


def run_both(s, st, chunks):
    out = []
    for sort in ("inc", "cub"):
        c = make_ctx(s, st.particles.size(), sort)
        c.upload(st)
        for k in chunks:
            c.advance(k)
        out.append((c.download(st.copy()), c.digest()))
        c.close()
    return out


def assert_bitwise(a, b, what):
    for f in FIELDS:
        assert np.array_equal(getattr(a.particles, f), getattr(b.particles, f)), f"{what}: {f} differs"


def many_movers_scene(dim):
    """Particles crossing cells (and blocks) every step: random velocities of ~0.4 cells/step."""
    s = Scene(dim, "f64")
    c = s.config
    c.dh, c.cells, c.dt, c.gravity = 0.05, [24] * dim, 2e-3, [0.0] * dim
    c.scheme.kind = "pic"
    s.material = FluidParams(1000.0, 0.0, 5.0)
    s.geometry.append(GeometryRegion(lo=[0.3] * dim, hi=[0.9] * dim))
    return s


@pytest.mark.parametrize("case", ["c1", "dp3", "fluid3-apic", "many2", "many3"])
def test_incremental_sort_bitwise_equals_radix_sort(case):
    if case == "c1":
        s = c1_column()
        st = init_scene(s)
        chunks = [1, 40, 59]  # eager first step, graph replays, a second call
    elif case == "dp3":
        s = dp_block_scene(3, cells=[16, 16, 16])
        st = init_scene(s)
        chunks = [100]
    elif case == "fluid3-apic":
        s = fluid_box_scene(3, kind="apic")
        st = init_scene(s)
        chunks = [30, 30]
    else:
        dim = 2 if case == "many2" else 3
        s = many_movers_scene(dim)
        st = init_scene(s)
        rng = np.random.default_rng(11)
        st.particles.v[...] = rng.uniform(-10.0, 10.0, st.particles.v.shape)  # up to 0.4 dh per step
        chunks = [1, 25, 24]
    (a, da), (b, db) = run_both(s, st, chunks)
    assert da == db
    assert_bitwise(a, b, case)


def test_incremental_sort_survives_count_change_and_reupload():
    """Upload / re-upload with a different particle count in between: the stored-order record is
    dropped, so the next sort is a full one and results stay bit-identical to the radix path."""
    s = dp_block_scene(3, cells=[12, 12, 12])
    st = init_scene(s)
    from paper_2507_04192_b200 import SimState
    half = SimState(st.particles.take(np.arange(0, st.particles.size(), 3)))
    res = []
    for sort in ("inc", "cub"):
        c = make_ctx(s, st.particles.size(), sort)
        out = []
        for state in (st, half, st):
            c.upload(state)
            c.advance(6)
            c.advance(5)
            out.append(c.download(state.copy()))
        res.append(out)
        c.close()
    for a, b in zip(*res):
        assert_bitwise(a, b, "reupload")


@pytest.mark.parametrize("nseg", [1, 3])
def test_incremental_sort_backprop_bitwise(nseg):
    """backprop_trajectory: forward sweep, replays (tape sort sets) and VJPs bit-identical."""
    s = dp_block_scene(3, coulomb=True, cells=[16, 12, 12])
    st = init_scene(s)
    N = 12
    got = []
    for sort in ("inc", "cub"):
        c = make_ctx(s, st.particles.size(), sort)
        c.upload(st)
        c.advance(N)
        tgt = c.download(st.copy()).particles.x + 0.01
        c0, pg, r = c.backprop(st, N, nseg, {"field": "x", "obs_steps": [N], "sel": None, "target": tgt[None]})
        got.append((c0, pg, r.loss))
        c.close()
    (a, pa, la), (b, pb, lb) = got
    assert la == lb
    for f in ("x", "v", "sigma", "rho", "volume"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(pa.flat(), pb.flat())
