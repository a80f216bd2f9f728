"""Slab decomposition, CPU side.

These tests cover the plan, the orchestration (halo bands, migration, error propagation), and
two transports: in-process, and torch.distributed gloo at world_size 2. Each rank's physics is
the oracle (tests/slab_oracle.py). The decomposed trajectory must match the undecomposed oracle
to round-off, since only the summation order at the halo nodes differs. Both transports must
give bit-identical results.
"""
from __future__ import annotations

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_04192_b200 import init_scene
from paper_2507_04192_b200.distributed import (LocalTransport, PeerFailure, SlabPlan, SlabStepper, TorchTransport,
                                               base_cell_x, block_edge)
from paper_2507_04192_b200.errors import NumericalError
from paper_2507_04192_b200.scene import FluidParams, GeometryRegion, Scene, VelocityExpr

from helpers import assert_state_close
from slab_oracle import OracleSlabDomain


def moving_fluid_scene(dim=2, dtype="f64", vx=5.0):
    """A fluid block carried along x across slab boundaries (gravity on, slip walls)."""
    s = Scene(dim, dtype)
    c = s.config
    c.dh = 0.01
    c.cells = [64, 32] if dim == 2 else [32, 16, 16]
    c.dt = 1e-4
    c.gravity = [0.0, -9.8] if dim == 2 else [0.0, -9.8, 0.0]
    c.scheme.kind, c.scheme.alpha_flip = "flip", 0.95
    s.material = FluidParams(1000.0, 0.0, 20.0)
    if dim == 2:
        s.geometry.append(GeometryRegion(lo=[0.08, 0.05], hi=[0.40, 0.20],
                                         velocity=VelocityExpr("constant", value=[vx, 0.0])))
    else:
        s.geometry.append(GeometryRegion(lo=[0.04, 0.03, 0.03], hi=[0.22, 0.10, 0.12],
                                         velocity=VelocityExpr("constant", value=[vx, 0.0, 0.0])))
    return s


def oracle_slab_run(scene, state, R, steps, orc, balance=True):
    plan = SlabPlan.make(scene, R, state.particles.x if balance else None)
    ids = plan.partition(scene, state)
    doms = [OracleSlabDomain(scene, plan, r, state, ids[r], orc) for r in range(R)]
    stp = SlabStepper(doms, LocalTransport())
    stp.advance(steps)
    return stp.gather_local(state), stp, plan


# ---- plan --------------------------------------------------------------------------------------
def test_plan_even_and_balanced():
    s = moving_fluid_scene()
    st = init_scene(s)
    B = block_edge(2)
    for R in (1, 2, 3, 4):
        for x in (None, st.particles.x):
            p = SlabPlan.make(s, R, x)
            assert p.n_ranks == R and p.bounds[0] == 0 and p.bounds[-1] == s.config.cells[0]
            assert all(b % B == 0 for b in p.bounds[:-1])
            assert all(p.bounds[k] < p.bounds[k + 1] for k in range(R))
            parts = p.partition(s, st)
            allids = np.sort(np.concatenate(parts))
            assert np.array_equal(allids, np.arange(st.particles.size()))
            bx = base_cell_x(s, st.particles.x)
            for r, ids in enumerate(parts):
                assert np.all((bx[ids] >= p.lo(r)) & (bx[ids] < p.hi(r)))
    # balanced plan: counts within one x-block column of each other
    p = SlabPlan.make(s, 2, st.particles.x)
    sizes = [len(i) for i in p.partition(s, st)]
    col = np.bincount(base_cell_x(s, st.particles.x) // B).max()
    assert abs(sizes[0] - sizes[1]) <= col
    with pytest.raises(ValueError):
        SlabPlan.make(s, 5, None)  # 64 cells / 16 = 4 blocks


# ---- in-process decomposition vs the undecomposed oracle -----------------------------------
@pytest.mark.parametrize("dim,R", [(2, 2), (2, 3), (2, 4), (3, 2), (3, 4)])
def test_local_decomposition_matches_oracle(orc, dim, R):
    s = moving_fluid_scene(dim)
    st = init_scene(s)
    steps = 30 if dim == 2 else 15
    got, stp, plan = oracle_slab_run(s, st, R, steps, orc)
    ref = st.copy()
    orc.advance(s, ref, steps)
    assert got.step == ref.step == steps
    assert stp.migrated > 0, "the scene must move particles across slab boundaries"
    assert_state_close(got, ref, 1e-10, what=f"slab R={R} vs oracle")


def test_single_slab_is_bitwise_oracle(orc):
    s = moving_fluid_scene(2)
    st = init_scene(s)
    got, stp, _ = oracle_slab_run(s, st, 1, 10, orc)
    ref = st.copy()
    orc.advance(s, ref, 10)
    for f in ("x", "v", "sigma", "rho", "volume", "grad_v"):
        assert np.array_equal(getattr(got.particles, f), getattr(ref.particles, f)), f


def test_error_propagates_to_all_ranks(orc):
    """a NaN on one rank aborts every rank at the same step (stepper.hpp:106-109)"""
    s = moving_fluid_scene(2)
    st = init_scene(s)
    plan = SlabPlan.make(s, 2, st.particles.x)
    ids = plan.partition(s, st)
    st.particles.v[ids[1][0], 1] = np.nan
    doms = [OracleSlabDomain(s, plan, r, st, ids[r], orc) for r in range(2)]
    stp = SlabStepper(doms, LocalTransport())
    with pytest.raises(NumericalError) as ei:
        stp.step(nan_guard=True)
    assert not isinstance(ei.value, PeerFailure)  # the failing rank's own error is raised
    assert len({d.sub.step for d in doms}) == 1 and stp.migrated == 0  # no rank went past the abort


# ---- torch.distributed gloo, world_size 2 ------------------------------------------------------
def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _gloo_worker(rank, world, port, out_path, dim, steps):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import CpuOracle

        orc = CpuOracle("orc")
        s = moving_fluid_scene(dim)
        st = init_scene(s)
        plan = SlabPlan.make(s, world, st.particles.x)
        ids = plan.partition(s, st)
        dom = OracleSlabDomain(s, plan, rank, st, ids[rank], orc)
        stp = SlabStepper([dom], TorchTransport())
        stp.advance(steps)
        sub, pid, _ = dom.gather()
        parts = [None] * world if rank == 0 else None
        dist.gather_object((sub, pid, stp.migrated), parts, dst=0)
        if rank == 0:
            out = st.copy()
            mig = 0
            for sp, ip, m in parts:
                out.particles.put(ip, sp)
                mig += m
            np.savez(out_path, x=out.particles.x, v=out.particles.v, sigma=out.particles.sigma,
                     rho=out.particles.rho, mig=mig)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dim", [2, 3])
def test_gloo_world2_matches_local_bitwise(orc, dim):
    steps = 20 if dim == 2 else 10
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "out.npz")
        mp.start_processes(_gloo_worker, args=(2, _free_port(), path, dim, steps), nprocs=2, join=True,
                           start_method="spawn")
        g = np.load(path)
        s = moving_fluid_scene(dim)
        st = init_scene(s)
        loc, stp, _ = oracle_slab_run(s, st, 2, steps, orc)
        assert int(g["mig"]) == stp.migrated > 0
        for f in ("x", "v", "sigma", "rho"):
            assert np.array_equal(g[f], getattr(loc.particles, f)), f"gloo vs in-process differ on {f}"
        ref = st.copy()
        orc.advance(s, ref, steps)
        assert_state_close(loc, ref, 1e-10)


class _FakeDom:
    def __init__(self, rank, per=5, dim=2):
        self.rank, self.per, self.dim, self.device = rank, per, dim, torch.device("cpu")

    def empty_halo(self, n):
        return torch.empty((n * self.per, 1 + 2 * self.dim), dtype=torch.float64)

    def empty_halo_cot(self, n):
        return torch.empty((n * self.per, 2 * self.dim), dtype=torch.float64)


def _gloo_adjoint_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = TorchTransport()
        d = _FakeDom(rank)
        mk = lambda v: torch.full((2 * d.per, 2 * d.dim), float(v), dtype=torch.float64)  # noqa: E731
        sends = {rank: (mk(10 * rank + 1) if rank > 0 else None, mk(10 * rank + 2) if rank + 1 < world else None)}
        recv = tr.exchange(sends, {rank: d}, "halo_cot")[rank]
        tot = tr.sum_ordered({rank: np.array([0.1 * (rank + 1), 1e-17 * rank])})
        objs = tr.allgather_obj({rank: ("ids", rank)})
        res = {"from_lo": None if recv[0] is None else float(recv[0][0, 0]),
               "from_hi": None if recv[1] is None else float(recv[1][0, 0]), "tot": tot.tolist(),
               "objs": [objs[q][1] for q in range(world)]}
        np.save(out_path + f".{rank}.npy", np.array([res], dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


def test_gloo_adjoint_transport_primitives():
    """the cotangent halo band, the rank-ordered ParamGrads sum and the object gather over gloo"""
    world = 3
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "adj")
        mp.start_processes(_gloo_adjoint_worker, args=(world, _free_port(), path), nprocs=world, join=True,
                           start_method="spawn")
        res = [np.load(path + f".{r}.npy", allow_pickle=True)[0] for r in range(world)]
    for r in range(world):
        assert res[r]["from_lo"] == (None if r == 0 else 10 * (r - 1) + 2)  # lower neighbour's upper band
        assert res[r]["from_hi"] == (None if r == world - 1 else 10 * (r + 1) + 1)
        assert res[r]["objs"] == list(range(world))
        assert res[r]["tot"] == res[0]["tot"]  # identical bits on every rank
    want = 0.1 * 1
    for r in range(1, world):
        want = want + 0.1 * (r + 1)  # rank order
    assert res[0]["tot"][0] == want


@pytest.mark.parametrize("dim,R", [(2, 3), (3, 2)])
def test_rebalancing_keeps_physics_and_balances(orc, dim, R):
    """an even block split of a block sitting on one side is badly unbalanced; the
    stepper re-plans from the global histogram, moves particles to their new owners, and the
    trajectory still matches the undecomposed oracle"""
    s = moving_fluid_scene(dim)
    st = init_scene(s)
    plan = SlabPlan.make(s, R, None)  # even split: unbalanced for this scene
    ids = plan.partition(s, st)
    c0 = [len(i) for i in ids]
    assert max(c0) > 1.3 * (sum(c0) / R)
    doms = [OracleSlabDomain(s, plan, r, st, ids[r], orc) for r in range(R)]
    stp = SlabStepper(doms, LocalTransport(), rebalance_every=4, imbalance=1.05)
    steps = 16 if dim == 2 else 8
    stp.advance(steps)
    assert stp.rebalances >= 1
    counts = stp.counts()
    B = block_edge(dim)
    col = np.bincount(base_cell_x(s, stp.gather_local(st).particles.x) // B).max()
    assert max(counts.values()) - min(counts.values()) <= 2 * col
    assert sum(counts.values()) == st.particles.size()
    for r, d in stp.domains.items():  # every particle sits in its (new) slab
        bx = base_cell_x(s, d.sub.particles.x)
        assert np.all((bx >= d.plan.lo(r)) & ((bx < d.plan.hi(r)) | (r == R - 1)))
    got = stp.gather_local(st)
    ref = st.copy()
    orc.advance(s, ref, steps)
    assert_state_close(got, ref, 1e-10, what="rebalanced slabs vs oracle")
