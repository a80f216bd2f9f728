"""Slab decomposition on the device through the C ABI's slab entry points.

R contexts share one GPU and are stepped in lock-step by LocalTransport. No rank's kernels wait
on another's. The tests check:
  * a single slab is bit-identical to the plain advance path. The halo-free split P2G + finish
    performs the same operations in the same order.
  * R = 2, 3, 4 slabs match the undecomposed device run and the oracle to round-off. Only the
    summation order on the halo planes differs.
  * the decomposition is deterministic run to run, and migration really happens.
  * an OOD abort on one rank raises on every rank at the same step.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2507_04192_b200 import init_scene
from paper_2507_04192_b200.distributed import (GpuSlabDomain, LocalTransport, SlabPlan, SlabStepper, local_slab_run)
from paper_2507_04192_b200.errors import NumericalError
from paper_2507_04192_b200.solver import Context
from paper_2507_04192_b200.state import SimState

from helpers import assert_state_close
from test_distributed import moving_fluid_scene

pytestmark = pytest.mark.gpu


def plain_gpu(scene, st, steps):
    ctx = Context(scene, st.particles.size())
    ctx.upload(st)
    ctx.advance(steps)
    out = ctx.download(st.copy())
    ctx.close()
    return out


@pytest.mark.parametrize("dim,dtype", [(2, "f64"), (3, "f64"), (2, "f32"), (3, "f32")])
def test_single_slab_bitwise_plain(dim, dtype):
    s = moving_fluid_scene(dim, dtype)
    st = init_scene(s)
    got, stp, _ = local_slab_run(s, st, 1, 12)
    ref = plain_gpu(s, st, 12)
    assert got.step == ref.step == 12
    for f in ("x", "v", "sigma", "rho", "volume", "grad_v", "eps_eq"):
        assert np.array_equal(getattr(got.particles, f), getattr(ref.particles, f)), f


@pytest.mark.parametrize("dim,R", [(2, 2), (2, 3), (2, 4), (3, 2), (3, 4)])
def test_slabs_match_plain_and_oracle(orc, dim, R):
    s = moving_fluid_scene(dim)
    st = init_scene(s)
    steps = 40 if dim == 2 else 20
    got, stp, plan = local_slab_run(s, st, R, steps)
    assert stp.migrated > 0
    assert sum(d.local_count() for d in stp.domains.values()) == st.particles.size()
    ref = plain_gpu(s, st, steps)
    assert_state_close(got, ref, 1e-10, what=f"R={R} vs single context")
    orc_ref = st.copy()
    orc.advance(s, orc_ref, steps)
    assert_state_close(got, orc_ref, 1e-9, what=f"R={R} vs oracle")  # the n-step parity bar (test_gpu_forward)


def test_slabs_f32_close():
    s = moving_fluid_scene(2, "f32")
    st = init_scene(s)
    got, _, _ = local_slab_run(s, st, 3, 30)
    ref = plain_gpu(s, st, 30)
    assert_state_close(got, ref, 2e-4, what="f32 R=3")


def test_slabs_deterministic():
    s = moving_fluid_scene(3)
    st = init_scene(s)
    a, _, _ = local_slab_run(s, st, 4, 15)
    b, _, _ = local_slab_run(s, st, 4, 15)
    for f in ("x", "v", "sigma", "rho", "grad_v"):
        assert np.array_equal(getattr(a.particles, f), getattr(b.particles, f)), f


def test_slabs_dp_column_3d():
    """D-P sand column (C4 material and boundaries, small): decomposition vs single context"""
    from paper_2507_04192_b200.presets import bui_sand
    from paper_2507_04192_b200.scene import GeometryRegion, Scene, Wall

    s = Scene(3, "f64")
    c = s.config
    c.dh, c.cells, c.dt, c.gravity = 1.0 / 64, [64, 32, 32], 1e-5, [0.0, -9.8, 0.0]
    c.scheme.kind = "flip"
    s.material = bui_sand()
    s.boundary.walls[2] = Wall("no_slip")
    dh = c.dh
    s.geometry.append(GeometryRegion(lo=[2 * dh, 2 * dh, 2 * dh], hi=[2 * dh + 0.5, 2 * dh + 0.25, 2 * dh + 0.25]))
    st = init_scene(s)
    got, stp, plan = local_slab_run(s, st, 4, 30)
    ref = plain_gpu(s, st, 30)
    assert_state_close(got, ref, 1e-8, what="D-P column R=4")


def test_abort_stops_all_ranks_like_plain():
    """A particle of rank 0 is thrown into the floor. The plain path raises the compression error
    at step 3 (state step 2). The decomposition must raise the same error during the same step
    attempt, with no rank going on."""
    s = moving_fluid_scene(2)
    st = init_scene(s)
    plan = SlabPlan.make(s, 2, st.particles.x)
    ids = plan.partition(s, st)
    st.particles.v[ids[0][0]] = [0.0, -400.0]
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    with pytest.raises(NumericalError) as plain_err:
        ctx.advance(20)
    err_step = ctx.last_error_step()  # before another call replaces the last error
    plain_done = ctx.download(st.copy()).step
    doms = [GpuSlabDomain(s, plan, r, st, ids[r]) for r in range(2)]
    stp = SlabStepper(doms, LocalTransport())
    with pytest.raises(NumericalError) as slab_err:
        stp.advance(20)
    assert type(slab_err.value) is type(plain_err.value) and str(slab_err.value) == str(plain_err.value)
    got = (stp.steps_done, doms[0].ctx.last_error_step(), doms[1].ctx.last_error_step())
    assert got[:2] == (plain_done, err_step), (got, plain_done, err_step)


# ---- adjoint over slabs (SURVEY §8e adjoint row) -------------------------------------------------
def coulomb_slide_scene(dim=2):
    """the moving fluid on a segmented Coulomb floor: friction gradients on both sides of the slabs"""
    from paper_2507_04192_b200.scene import Wall

    s = moving_fluid_scene(dim)
    s.boundary.walls[2] = Wall("coulomb", [0.2, 0.35, 0.5, 0.3])
    g = s.geometry[0]
    g.lo[1], g.hi[1] = 0.02, 0.02 + (g.hi[1] - g.lo[1])  # on the floor: nodes in the 2-layer friction band
    return s


@pytest.mark.parametrize("dim,R,coulomb", [(2, 2, False), (2, 3, True), (2, 4, True), (3, 2, True), (3, 4, False)])
def test_slab_step_vjp_matches_single_context(dim, R, coulomb):
    from paper_2507_04192_b200.distributed import slab_step_vjp
    from paper_2507_04192_b200.state import ParamGrads

    from test_gpu_adjoint import cot_errs, random_cot

    s = coulomb_slide_scene(dim) if coulomb else moving_fluid_scene(dim)
    st = plain_gpu(s, init_scene(s), 8 if dim == 2 else 4)  # a state with stress and a flow
    cot = random_cot(st, 7)
    ctx = Context(s, st.particles.size())
    pg_ref = ParamGrads(s.boundary)
    want = ctx.step_vjp(st, cot, pg_ref)
    ctx.close()

    plan = SlabPlan.make(s, R, st.particles.x)
    ids = plan.partition(s, st)
    doms = [GpuSlabDomain(s, plan, r, st, ids[r]) for r in range(R)]
    pg = ParamGrads(s.boundary)
    got_r = slab_step_vjp(doms, LocalTransport(), {r: SimState(st.particles.take(ids[r]), st.step, st.time)
                                                   for r in range(R)},
                          {r: cot.take(ids[r]) for r in range(R)}, pg)
    got = want.copy()
    for r in range(R):
        got.put(ids[r], got_r[r])
    # halo-node sums run in a different order than on one context: rounding-level differences,
    # amplified in the x cotangent by the stencil Hessian terms (measured up to 1.1e-9)
    errs = cot_errs(got, want)
    assert all(v < 1e-8 for v in errs.values()), errs
    assert abs(pg.sound_speed - pg_ref.sound_speed) <= 1e-8 * abs(pg_ref.sound_speed) + 1e-300
    if coulomb:
        a, b = pg.wall_friction[2], pg_ref.wall_friction[2]
        assert np.abs(b).max() > 0
        assert np.abs(a - b).max() <= 1e-8 * np.abs(b).max(), (a, b)


@pytest.mark.parametrize("dim,R,nseg", [(2, 2, 3), (2, 3, 1), (3, 2, 2)])
def test_slab_backprop_matches_single_context(dim, R, nseg):
    """backprop_trajectory over slabs vs the single-context device backprop: the initial-state
    cotangent, the ParamGrads (incl. Coulomb friction) and the loss"""
    from paper_2507_04192_b200.distributed import slab_backprop_trajectory
    from paper_2507_04192_b200.seeders import LagrangianLeastSquares
    from paper_2507_04192_b200.solver import CheckpointPlan

    from test_gpu_adjoint import cot_errs

    s = coulomb_slide_scene(dim)
    st = init_scene(s)
    N = 12 if dim == 2 else 6
    n = st.particles.size()
    mid, fin = plain_gpu(s, st, N // 2), plain_gpu(s, st, N)
    rng = np.random.default_rng(3)
    tgt = np.stack([mid.particles.x + 0.002 * rng.standard_normal(mid.particles.x.shape),
                    fin.particles.x + 0.002 * rng.standard_normal(fin.particles.x.shape)])
    seeder = LagrangianLeastSquares([N // 2, N], tgt, "x")
    ctx = Context(s, n)
    c0, pg_ref, res = ctx.backprop(st, N, nseg, seeder.desc())
    ctx.close()

    plan_s = SlabPlan.make(s, R, st.particles.x)
    ids = plan_s.partition(s, st)
    doms = [GpuSlabDomain(s, plan_s, r, st, ids[r]) for r in range(R)]
    out = slab_backprop_trajectory(s, CheckpointPlan.make(N, nseg), seeder, doms, LocalTransport(), n)
    assert out.loss == pytest.approx(res.loss, rel=1e-10)
    errs = cot_errs(out.initial_state_cot, c0)
    assert all(v < 1e-8 for v in errs.values()), errs
    a, b = out.param_grads.wall_friction[2], pg_ref.wall_friction[2]
    assert np.abs(b).max() > 0 and np.abs(a - b).max() <= 1e-8 * np.abs(b).max(), (a, b)
    assert abs(out.param_grads.sound_speed - pg_ref.sound_speed) <= 1e-8 * abs(pg_ref.sound_speed)
    assert out.checkpoints_stored == nseg


def test_gpu_rebalancing_matches_single_context():
    """dynamic slab rebalancing on the device path: even split -> re-planned"""
    s = moving_fluid_scene(2)
    st = init_scene(s)
    plan = SlabPlan.make(s, 3, None)
    ids = plan.partition(s, st)
    doms = [GpuSlabDomain(s, plan, r, st, ids[r]) for r in range(3)]
    stp = SlabStepper(doms, LocalTransport(), rebalance_every=5, imbalance=1.05)
    stp.advance(20)
    assert stp.rebalances >= 1
    c = stp.counts()
    got = stp.gather_local(st)
    from paper_2507_04192_b200.distributed import base_cell_x, block_edge

    col = np.bincount(base_cell_x(s, got.particles.x) // block_edge(2)).max()  # balance is per x-block
    assert max(c.values()) - min(c.values()) <= 2 * col and sum(c.values()) == st.particles.size()
    ref = plain_gpu(s, st, 20)
    assert_state_close(got, ref, 1e-10, what="rebalanced device slabs")
