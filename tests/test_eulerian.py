"""Eulerian (velocity-monitor) loss seeder, SPEC.md observe_eulerian / PAPER §3.2: the reference
specifies it but does not implement it, so parity is pinned by two independent restatements of the
SPEC formula (the C oracle and EulerianLeastSquares' numpy form), a finite-difference check of the
whole adjoint chain, and the device seeder against the oracle (GPU)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2507_04192_b200 import init_scene
from paper_2507_04192_b200.seeders import EulerianLeastSquares
from paper_2507_04192_b200.state import StateCotangent

from helpers import rel_err
from test_distributed import moving_fluid_scene


def monitors(scene, st, obs, seed=5, empty=True):
    """3x3 monitor boxes over the fluid (+ one empty region far away), targets near the truth"""
    x = st.particles.x
    lo, hi = x.min(0), x.max(0)
    cs = []
    for i in range(3):
        for j in range(3):
            c = lo + (hi - lo) * np.array([0.2 + 0.3 * i, 0.2 + 0.3 * j] + [0.5] * (scene.dim - 2))
            cs.append(c)
    if empty:
        cs.append(np.array([(c - 3) * scene.config.dh for c in scene.config.cells[:scene.dim]]))  # far corner: empty
    cs = np.array(cs)
    rng = np.random.default_rng(seed)
    tgt = rng.standard_normal((len(obs), len(cs), scene.dim)) * 0.05
    mask = np.ones((len(obs), len(cs)), np.uint8)
    mask[0, 1] = 0
    return cs, 0.02, tgt, mask


def numpy_loss_seed(seeder, step, st):
    ids = np.arange(st.particles.size())
    stats = seeder.stats_local(step, st.particles, ids)
    rows, dz = seeder.seed_local(step, st.particles, ids, stats)
    return seeder.loss_from_stats(step, stats), dz


@pytest.mark.parametrize("dim", [2, 3])
def test_oracle_eulerian_seed_matches_numpy(orc, dim):
    s = moving_fluid_scene(dim)
    st = init_scene(s)
    st.particles.v[:] += np.random.default_rng(1).standard_normal(st.particles.v.shape) * 0.1
    cs, half, tgt, mask = monitors(s, st, [0])
    sd = EulerianLeastSquares([0], cs, half, tgt, "v", mask)
    c0, pg, res = orc.backprop(s, st, 2, 1, sd.desc())  # observed only at step 0: c0 = the seed itself
    L, dz = numpy_loss_seed(sd, 0, st)
    assert res.loss == pytest.approx(L, rel=1e-12)
    assert rel_err(c0.v, dz, 1e-300) < 1e-12
    members = sd._members(st.particles)
    assert members[:, -1].sum() == 0  # the empty region contributes nothing
    assert members[:, :-1].sum(0).min() > 0


def test_oracle_eulerian_finite_difference(orc):
    """d L / d v0 through 6 steps of the oracle's adjoint vs central differences of the forward loss"""
    s = moving_fluid_scene(2)
    st = init_scene(s)
    N = 6
    fin = st.copy()
    orc.advance(s, fin, N)
    cs, half, tgt, _ = monitors(s, fin, [N], empty=False)
    sd = EulerianLeastSquares([N], cs, half, tgt, "v")
    c0, _, res = orc.backprop(s, st, N, 2, sd.desc())
    rng = np.random.default_rng(11)

    def loss(v0):
        a = st.copy()
        a.particles.v[...] = v0
        orc.advance(s, a, N)
        return numpy_loss_seed(sd, N, a)[0]

    for _ in range(4):
        d = rng.standard_normal(st.particles.v.shape)
        eps = 1e-6
        fd = (loss(st.particles.v + eps * d) - loss(st.particles.v - eps * d)) / (2 * eps)
        an = float((c0.v * d).sum())
        assert abs(fd - an) <= 1e-5 * (abs(fd) + 1e-12), (fd, an)


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [2, 3])
def test_device_eulerian_backprop_matches_oracle(orc, dim):
    from paper_2507_04192_b200.solver import Context

    s = moving_fluid_scene(dim)
    st = init_scene(s)
    N = 8 if dim == 2 else 4
    mid = st.copy()
    orc.advance(s, mid, N // 2)
    cs, half, tgt, mask = monitors(s, mid, [N // 2, N])
    sd = EulerianLeastSquares([N // 2, N], cs, half, tgt, "v", mask)
    ctx = Context(s, st.particles.size())
    g0, gpg, gres = ctx.backprop(st, N, 2, sd.desc())
    ctx.close()
    w0, wpg, wres = orc.backprop(s, st, N, 2, sd.desc())
    assert gres.loss == pytest.approx(wres.loss, rel=1e-10)
    # fields far below the velocity cotangent's scale (x here: ~1e-17) are compared on that scale
    scale = float(np.abs(w0.v).max())
    for f in ("x", "v", "rho", "volume", "sigma"):
        a, b = getattr(g0, f), getattr(w0, f)
        assert rel_err(a, b, scale) < 1e-8, f
    assert gpg.sound_speed == pytest.approx(wpg.sound_speed, rel=1e-8)


@pytest.mark.gpu
def test_slab_eulerian_backprop_matches_single_context():
    from paper_2507_04192_b200.distributed import GpuSlabDomain, LocalTransport, SlabPlan, slab_backprop_trajectory
    from paper_2507_04192_b200.solver import CheckpointPlan, Context

    s = moving_fluid_scene(2)
    st = init_scene(s)
    N = 10
    cs, half, tgt, mask = monitors(s, st, [5, N])
    sd = EulerianLeastSquares([5, N], cs, half, tgt, "v", mask)
    n = st.particles.size()
    ctx = Context(s, n)
    c0, pg, res = ctx.backprop(st, N, 2, sd.desc())
    ctx.close()
    plan = SlabPlan.make(s, 3, st.particles.x)
    ids = plan.partition(s, st)
    doms = [GpuSlabDomain(s, plan, r, st, ids[r]) for r in range(3)]
    out = slab_backprop_trajectory(s, CheckpointPlan.make(N, 2), sd, doms, LocalTransport(), n)
    assert out.loss == pytest.approx(res.loss, rel=1e-10)
    assert rel_err(out.initial_state_cot.v, c0.v, 1e-300) < 1e-8
    assert rel_err(out.initial_state_cot.x, c0.x, float(np.abs(c0.v).max())) < 1e-8
