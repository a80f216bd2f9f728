"""The library-owned slab decomposition (mpm_dist_*, csrc/kernels_dist.cuh): the whole decomposed
step -- incremental sort with device-resident counts, P2G, halo exchange, fixed-order band import,
G2P, fixed-capacity migration messages, the device max-reduction of the abort flag -- runs inside
libmpm_b200 with no host synchronisation inside a call.

On one GPU the R ranks are same-process contexts (mpm_dist_attach_local: device-copy exchanges,
lock-step phases); the NCCL transport is exercised as a 1-rank communicator. Checks:
  * one slab is bit-identical to the plain single-context advance;
  * R = 2, 3, 4 slabs match the single context to round-off (only the halo-plane sums are ordered
    differently) and the oracle to the n-step parity bar, with particles really migrating;
  * bit-identical run to run; the result does not depend on how the steps are split into calls;
  * a rank's failure raises on every rank (its own error on the failing rank);
  * the NCCL rank (nranks = 1) is bit-identical to the plain path.
"""
from __future__ import annotations

import numpy as np
import pytest

from helpers import assert_state_close
from paper_2507_04192_b200 import init_scene
from paper_2507_04192_b200.distributed import LocalSlabGroup, NcclSlabRank, SlabPlan, dist_unique_id
from paper_2507_04192_b200.errors import NumericalError, OutOfDomainError
from paper_2507_04192_b200.presets import c4_column3d
from paper_2507_04192_b200.solver import Context
from paper_2507_04192_b200.state import SimState

from test_distributed import moving_fluid_scene

pytestmark = pytest.mark.gpu

FIELDS = ("x", "v", "sigma", "rho", "volume", "grad_v", "eps_eq")


def plain_gpu(scene, st, steps, chunks=None):
    ctx = Context(scene, st.particles.size())
    ctx.upload(st)
    for k in chunks or [steps]:
        ctx.advance(k)
    out = ctx.download(st.copy())
    ctx.close()
    return out


def dist_run(scene, st, R, chunks, balance=True):
    plan = SlabPlan.make(scene, R, st.particles.x if balance else None)
    g = LocalSlabGroup(scene, plan, st)
    for k in chunks:
        g.advance(k)
    out = g.gather()
    counts = [int(c.lib.mpm_local_count(c.h)) for c in g.ctxs]
    g.close()
    return out, plan, counts


@pytest.mark.parametrize("dim", [2, 3])
def test_single_slab_bitwise_plain(dim):
    s = moving_fluid_scene(dim)
    st = init_scene(s)
    got, _, _ = dist_run(s, st, 1, [1, 11])
    ref = plain_gpu(s, st, 12, [1, 11])
    assert got.step == ref.step == 12
    for f in FIELDS:
        assert np.array_equal(getattr(got.particles, f), getattr(ref.particles, f)), f


@pytest.mark.parametrize("dim,R", [(2, 2), (2, 3), (2, 4), (3, 2), (3, 4)])
def test_slabs_match_plain_and_oracle(orc, dim, R):
    s = moving_fluid_scene(dim)
    st = init_scene(s)
    steps = 40 if dim == 2 else 20
    plan0 = SlabPlan.make(s, R, st.particles.x)
    got, plan, counts = dist_run(s, st, R, [steps])
    assert got.step == steps
    # particles moved between slabs (the block is carried along +x)
    start = [len(ix) for ix in plan0.partition(s, st)]
    assert counts != start
    ref = plain_gpu(s, st, steps)
    assert_state_close(got, ref, 1e-10, what=f"dist R={R} vs single context")
    want = orc.advance(s, st.copy(), steps)
    assert_state_close(got, want, 1e-9, what=f"dist R={R} vs oracle")


def test_slabs_deterministic_and_call_split_invariant():
    s = moving_fluid_scene(3)
    st = init_scene(s)
    a, _, _ = dist_run(s, st, 4, [15])
    b, _, _ = dist_run(s, st, 4, [15])
    c, _, _ = dist_run(s, st, 4, [1, 6, 8])
    for f in FIELDS:
        assert np.array_equal(getattr(a.particles, f), getattr(b.particles, f)), f
        assert np.array_equal(getattr(a.particles, f), getattr(c.particles, f)), f


def test_failure_raises_on_every_rank():
    """a particle thrown out of the domain on one rank: that rank reports its out-of-domain
    error, the others 'another rank aborted'; the call raises"""
    s = moving_fluid_scene(2)
    st = init_scene(s)
    bad = int(np.argmax(st.particles.x[:, 0]))  # on the last rank
    st.particles.v[bad, 0] = 3e4
    plan = SlabPlan.make(s, 3, st.particles.x)
    g = LocalSlabGroup(s, plan, st)
    with pytest.raises((OutOfDomainError, NumericalError)):
        g.advance(5)
    msgs = []
    for c in g.ctxs:
        import ctypes as C
        code = C.c_int()
        buf = C.create_string_buffer(512)
        c.lib.mpm_last_error(c.h, C.byref(code), None, None, buf, 512)
        msgs.append((code.value, buf.value.decode()))
    g.close()
    assert all(code != 0 for code, _ in msgs), msgs
    assert any("another rank" in m for _, m in msgs) and any("another rank" not in m for _, m in msgs), msgs


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("graph", ["1", "0"])
def test_nccl_single_rank_bitwise_plain(dim, graph, monkeypatch):
    """graph "0": the eager step path multi-rank NCCL groups take by default"""
    monkeypatch.setenv("MPM_DIST_GRAPH", graph)
    s = moving_fluid_scene(dim)
    st = init_scene(s)
    plan = SlabPlan([0, s.config.cells[0]], 16 if dim == 2 else 8)
    ids = np.arange(st.particles.size(), dtype=np.int64)
    rk = NcclSlabRank(s, plan, 0, st, ids, dist_unique_id())
    ms = rk.advance(1)
    ms += rk.advance(11)
    parts, gid, (step, _) = rk.gather()
    rk.close()
    assert ms > 0 and step == 12
    got = st.copy()
    got.particles.put(gid, parts)
    ref = plain_gpu(s, st, 12, [1, 11])
    for f in FIELDS:
        assert np.array_equal(getattr(got.particles, f), getattr(ref.particles, f)), f


def test_c4_two_slabs_close_to_single_context():
    """C4 (4.19 M particles) split into two slabs at x = 128 cells, 6 steps"""
    s = c4_column3d()
    st = init_scene(s)
    plan = SlabPlan([0, 128, 256], 8)
    g = LocalSlabGroup(s, plan, st)
    g.advance(1)
    g.advance(5)
    got = g.gather()
    g.close()
    ref = plain_gpu(s, st, 6, [1, 5])
    assert_state_close(got, ref, 1e-10, what="C4 R=2")


# ---- decomposed backprop_trajectory, device-resident (mpm_dist_backprop[_local]) ---------------
def single_backprop(s, st, N, nseg, seeder):
    ctx = Context(s, st.particles.size())
    c0, pg, res = ctx.backprop(st, N, nseg, seeder)
    ctx.close()
    return c0, pg, res


def _lag_seeder(s, st, N):
    ctx = Context(s, st.particles.size())
    ctx.upload(st)
    ctx.advance(N)
    xf = ctx.download(st.copy()).particles.x
    ctx.close()
    rng = np.random.default_rng(4)
    sel = np.sort(rng.choice(len(xf), len(xf) // 3, replace=False)).astype(np.int64)
    return {"field": "x", "obs_steps": [N // 2, N], "sel": sel,
            "target": np.stack([xf[sel] + 0.002, xf[sel] - 0.001])}


def _assert_cot_close(got, want, tol, what):
    from helpers import rel_err
    for f in ("x", "v", "rho", "volume", "sigma"):
        e = rel_err(getattr(got, f), getattr(want, f))
        assert e <= tol, (what, f, e)


@pytest.mark.parametrize("dim,R,nseg", [(2, 1, 1), (2, 2, 1), (2, 3, 2), (3, 2, 3), (3, 4, 1)])
def test_dist_backprop_matches_single_context(dim, R, nseg):
    """migrating fluid block: the decomposed gradient (device-resident, cotangent rows of migrants
    returned to their owners) equals the single context's to round-off"""
    s = moving_fluid_scene(dim)
    st = init_scene(s)
    N = 24 if dim == 2 else 12
    seeder = _lag_seeder(s, st, N)
    want_c0, want_pg, want_res = single_backprop(s, st, N, nseg, seeder)
    plan = SlabPlan.make(s, R, st.particles.x)
    g = LocalSlabGroup(s, plan, st)
    got_c0, got_pg, got_res = g.backprop(N, nseg, seeder)
    after = g.gather()
    g.close()
    assert abs(got_res.loss - want_res.loss) <= 1e-10 * abs(want_res.loss)
    _assert_cot_close(got_c0, want_c0, 1e-8 if R > 1 else 1e-12, f"R={R}")
    assert abs(got_pg.sound_speed - want_pg.sound_speed) <= 1e-8 * abs(want_pg.sound_speed)
    for f in FIELDS:  # the group's state is S^0 again
        assert np.array_equal(getattr(after.particles, f), getattr(st.particles, f)), f


def test_dist_backprop_friction_and_segment_invariance():
    """a fluid block sliding over a 4-segment Coulomb floor in 2 slabs: friction gradients vs the
    single context; the gradient is bit-identical for 1, 2 and 4 checkpoint segments. (A fluid:
    a Drucker-Prager block seeded at sigma = 0 sits on the cone's apex, where round-off differences
    of the halo sums legitimately select other return-map branches in the VJP.)"""
    from paper_2507_04192_b200 import Wall
    s = moving_fluid_scene(3)
    s.boundary.walls[2] = Wall("coulomb", [0.1, 0.3, 0.2, 0.4])
    s.geometry[0].lo[1] = 2 * s.config.dh  # the lowest nodes lie in the wall band
    st = init_scene(s)
    N = 8
    seeder = _lag_seeder(s, st, N)
    want_c0, want_pg, want_res = single_backprop(s, st, N, 1, seeder)
    plan = SlabPlan([0, 16, 32], 8)
    outs = []
    for nseg in (1, 2, 4):
        g = LocalSlabGroup(s, plan, st)
        outs.append(g.backprop(N, nseg, seeder))
        g.close()
    c0, pg, res = outs[0]
    fr_want, fr_got = want_pg.wall_friction[2], pg.wall_friction[2]
    assert np.abs(fr_want).max() > 0
    assert np.abs(fr_got - fr_want).max() <= 1e-8 * np.abs(fr_want).max()
    _assert_cot_close(c0, want_c0, 1e-8, "coulomb fluid R=2")
    for c_k, pg_k, res_k in outs[1:]:
        assert res_k.loss == res.loss
        assert np.array_equal(pg_k.flat(), pg.flat())
        for f in ("x", "v", "sigma"):
            assert np.array_equal(getattr(c_k, f), getattr(c0, f)), f


def test_dist_backprop_nccl_single_rank():
    s = moving_fluid_scene(2)
    st = init_scene(s)
    N = 10
    seeder = _lag_seeder(s, st, N)
    want_c0, want_pg, want_res = single_backprop(s, st, N, 2, seeder)
    plan = SlabPlan([0, s.config.cells[0]], 16)
    ids = np.arange(st.particles.size(), dtype=np.int64)
    rk = NcclSlabRank(s, plan, 0, st, ids, dist_unique_id())
    cot, gid, pg, res = rk.backprop(N, 2, seeder, st.particles.size())
    rk.close()
    got = want_c0.copy()
    got.put(gid, cot)
    assert abs(res.loss - want_res.loss) <= 1e-12 * abs(want_res.loss)
    _assert_cot_close(got, want_c0, 1e-12, "nccl R=1")


@pytest.mark.parametrize("cap", [None, "1"])
def test_dist_backprop_tape_bitwise(cap, monkeypatch):
    """the replay tape (each replay step's sort arrays and forward grid kept for its VJP) changes
    nothing: bit-identical to recomputing the forward replay inside every decomposed step_vjp;
    cap=1 forces every step to overflow its slot (the recompute fallback)"""
    s = moving_fluid_scene(2)
    st = init_scene(s)
    N = 16
    seeder = _lag_seeder(s, st, N)
    plan = SlabPlan.make(s, 3, st.particles.x)
    res = []
    for tape in ("1", "0"):
        monkeypatch.setenv("MPM_TAPE", tape)
        if cap:
            monkeypatch.setenv("MPM_TAPE_CAP", cap)
        g = LocalSlabGroup(s, plan, st)
        res.append(g.backprop(N, 2, seeder))
        g.close()
    (a, pa, ra), (b, pb, rb) = res
    assert ra.loss == rb.loss
    assert np.array_equal(pa.flat(), pb.flat())
    for f in ("x", "v", "sigma", "rho", "volume"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


def test_dist_c2_three_slabs_backprop_and_c5_forward():
    """scale: C2 (250,000 fluid particles) in 3 slabs, a 12-step decomposed backprop against the
    single context; the 1/8-particle C5 (4.06 M particles, 32 Coulomb segments) forward in 2 slabs"""
    from paper_2507_04192_b200.presets import c2_dam_break, c5_landslide_eighth
    s = c2_dam_break()
    st = init_scene(s)
    N = 12
    seeder = _lag_seeder(s, st, N)
    want_c0, want_pg, want_res = single_backprop(s, st, N, 3, seeder)
    g = LocalSlabGroup(s, SlabPlan.make(s, 3, st.particles.x), st)
    got_c0, got_pg, got_res = g.backprop(N, 3, seeder)
    g.close()
    assert abs(got_res.loss - want_res.loss) <= 1e-10 * abs(want_res.loss)
    _assert_cot_close(got_c0, want_c0, 1e-8, "C2 R=3")
    s5 = c5_landslide_eighth()
    st5 = init_scene(s5)
    g5 = LocalSlabGroup(s5, SlabPlan([0, 256, 512], 8), st5)
    g5.advance(1)
    g5.advance(3)
    got5 = g5.gather()
    g5.close()
    ref5 = plain_gpu(s5, st5, 4, [1, 3])
    assert_state_close(got5, ref5, 1e-10, what="C5/8 R=2")
