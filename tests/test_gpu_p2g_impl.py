"""3-D column-march implementations agree bit for bit: the warp-specialized kernels (k_p2g_ws and
K5b's k_adj_scatter_ws: producer warps + consumer warps on mbarriers) against the CTA-barrier
pipelines k_p2g_pipe3 / k_adj_scatter_pipe3 -- same per-particle arithmetic, same partial tiles,
same fixed combine order. The defaults are checked against the oracle elsewhere
(test_gpu_forward.py, test_gpu_adjoint.py), so equality here covers the A/B paths too."""
import numpy as np
import pytest

from paper_2507_04192_b200 import init_scene
from paper_2507_04192_b200.presets import c4_column3d
from paper_2507_04192_b200.scene import FluidParams, Scene
from paper_2507_04192_b200.solver import Context
from paper_2507_04192_b200.state import SimState

from helpers import dp_block_scene, fluid_box_scene

pytestmark = pytest.mark.gpu

FIELDS = ("x", "v", "volume", "rho", "eps_eq", "sigma", "grad_v")


def dense_fluid(dtype, n=30000, seed=3):
    """~117 particles per cell in an 8 x 8 x 4-cell box: levels of ~1900 particles (3 chunks of
    <= 640 per level) in each of 4 blocks -- the chunked path the C4 lattice never takes"""
    s = Scene(3, dtype)
    c = s.config
    c.dh, c.cells, c.dt, c.gravity = 0.05, [20, 20, 20], 1e-4, [0.0, -9.8, 0.0]
    c.scheme.kind, c.scheme.alpha_flip = "flip", 0.9
    s.material = FluidParams(1000.0, 0.0, 20.0)
    rng = np.random.default_rng(seed)
    st = SimState.zeros(n, 3, s.np_dtype)
    p = st.particles
    p.x[...] = rng.uniform([0.2, 0.2, 0.2], [0.6, 0.6, 0.4], (n, 3))
    p.v[...] = rng.uniform(-0.5, 0.5, (n, 3))
    p.mass[...] = 1000.0 * c.dh ** 3 / 8
    p.rho[...] = 1000.0
    p.volume[...] = p.mass / 1000.0
    a = rng.uniform(-50.0, 50.0, (n, 3, 3))
    p.sigma[...] = a + a.transpose(0, 2, 1)
    return s, st


CASES = {
    "dp3": lambda d: (lambda s: (s, init_scene(s)))(dp_block_scene(3, d, cells=[12, 12, 12])),
    "dp3-coulomb-obstacle": lambda d: (lambda s: (s, init_scene(s)))(
        dp_block_scene(3, d, coulomb=True, obstacle=True, cells=[16, 12, 12])),
    "fluid3-flip": lambda d: (lambda s: (s, init_scene(s)))(fluid_box_scene(3, d, kind="flip")),
    "dense-chunks": dense_fluid,
}


def run(s, st, impl, steps, monkeypatch):
    monkeypatch.setenv("MPM_P2G_IMPL", impl)
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.advance(1)
    ctx.advance(steps - 1)
    out = ctx.download(st.copy())
    ctx.close()
    return out


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("case", sorted(CASES))
def test_ws_bitwise_equals_pipe3(case, dtype, monkeypatch):
    s, st = CASES[case](dtype)
    a = run(s, st, "pipe3", 5, monkeypatch)
    b = run(s, st, "ws", 5, monkeypatch)
    for f in FIELDS:
        assert np.array_equal(getattr(a.particles, f), getattr(b.particles, f)), f


def test_ws_bitwise_equals_pipe3_c4(monkeypatch):
    """C4 (4.19 M particles, 1024 occupied blocks over 148 SMs): the work counter, block turnover"""
    s = c4_column3d()
    st = init_scene(s)
    a = run(s, st, "pipe3", 4, monkeypatch)
    b = run(s, st, "ws", 4, monkeypatch)
    for f in FIELDS:
        assert np.array_equal(getattr(a.particles, f), getattr(b.particles, f)), f


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("case", ["dp3-coulomb-obstacle", "fluid3-flip", "dense-chunks"])
def test_k5b_ws_bitwise_equals_pipe3(case, dtype, monkeypatch):
    """backprop_trajectory (forward sweep, replays, VJPs) with K5b on either kernel"""
    s, st = CASES[case](dtype)
    N = 4
    got = []
    for impl in ("ws", "pipe3"):
        monkeypatch.setenv("MPM_K5B", impl)
        c = Context(s, st.particles.size())
        c.upload(st)
        c.advance(N)
        tgt = c.download(st.copy()).particles.x + 0.01
        c0, pg, r = c.backprop(st, N, 2, {"field": "x", "obs_steps": [N], "sel": None, "target": tgt[None]})
        got.append((c0, pg, r.loss))
        c.close()
    (a, pa, la), (b, pb, lb) = got
    assert la == lb
    for f in ("x", "v", "sigma", "rho", "volume"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(pa.flat(), pb.flat())
