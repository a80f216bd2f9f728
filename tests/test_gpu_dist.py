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
def test_nccl_single_rank_bitwise_plain(dim):
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
