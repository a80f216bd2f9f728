"""Slab decomposition of the MPM step across GPUs.

The reference is single-process (stepper.hpp:49-70 has no decomposition). This module shards
the same step along x across one process per GPU. Every rank owns the particles whose base cell
along x lies in its slab `[lo, hi)`. Slab bounds are multiples of the particle-block edge: 16
cells in 2-D, 8 in 3-D. One step runs in four phases:

  1. P2G. Each rank calls `mpm_step_p2g_local`: it scatters its own particles and sums the
     nodes of the 2 node planes `[hi, hi + 2)` it shares with each neighbour, without `g m_i`.
  2. Halo sum. Each rank exports its partial (m, p, f) on those planes and posts the neighbour
     send/recv. While the bands travel, `mpm_step_grid_interior` updates every other node (sum,
     `g m_i`, momentum, corrections). Then each rank adds the neighbour's partial in a fixed
     order, lower rank's partial first, so both owners hold bit-identical nodes.
  3. Finish. Each rank calls `mpm_step_finish_local`: the band nodes get `g m_i`, the momentum
     update and the boundary corrections; then G2P and the constitutive update.
  4. Migration. A particle whose new base cell left the slab is exported from G2P and vacated
     from its slot. It is then appended by the receiving neighbour, in particle-id order.

There is no all-reduce on the data path. Each step does one small MAX all-reduce of an error
flag, so that a NaN/OOD abort on one rank stops every rank at the same step (stepper.hpp:106-109).

Transports:
  * TorchTransport runs torch.distributed point-to-point (NCCL over NVLink on device tensors;
    gloo on CPU tensors for the CPU tests). It carries one rank per process.
  * LocalTransport hands tensors between domains that live in the same process. It serves the
    single-GPU tests: R contexts on one device, stepped in lock-step, never waiting on each other.

Domains implement the per-rank protocol of `SlabDomain`. The product domain is GpuSlabDomain,
which calls the C ABI. tests/slab_oracle.py holds an oracle-backed domain used by the CPU tests.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from .errors import MPMError, NumericalError
from .scene import Scene
from .state import ParticleSoA, SimState


def block_edge(dim: int) -> int:
    """particle/node block edge in cells (csrc/common.cuh Cfg<D>::B)"""
    return 16 if dim == 2 else 8


def base_cell_x(scene: Scene, x: np.ndarray) -> np.ndarray:
    """base node index along x of the quadratic stencil (bspline.hpp:79-91): floor(u - 1/2)"""
    c = scene.config
    u = (x[:, 0] - c.origin[0]) / c.dh
    return np.floor(u - 0.5).astype(np.int64)


@dataclass
class SlabPlan:
    """Cell bounds along x for each rank. There are R+1 bounds, all multiples of `block`, with
    bounds[0] = 0 and bounds[R] = cells_x."""

    bounds: list
    block: int
    halo_planes: int = 2

    @property
    def n_ranks(self) -> int:
        return len(self.bounds) - 1

    def lo(self, r: int) -> int:
        return self.bounds[r]

    def hi(self, r: int) -> int:
        return self.bounds[r + 1]

    @staticmethod
    def make(scene: Scene, n_ranks: int, x: np.ndarray | None = None) -> "SlabPlan":
        """Split the x-blocks into n_ranks contiguous slabs. With particle positions `x`, balance
        the particle counts; otherwise split the blocks evenly. Every slab is at least one block
        wide and at least 3 cells wide, so that a particle's stencil never spans three slabs."""
        B = block_edge(scene.dim)
        cx = scene.config.cells[0]
        nbx = -(-cx // B)
        if n_ranks < 1 or n_ranks > nbx:
            raise ValueError(f"cannot split {nbx} x-blocks into {n_ranks} slabs")
        if x is None or len(x) == 0:
            cuts = [round(k * nbx / n_ranks) for k in range(n_ranks + 1)]
            bounds = [min(c * B, cx) for c in cuts]
            bounds[-1] = cx
            return SlabPlan(bounds, B)
        return SlabPlan.from_histogram(SlabPlan.block_histogram(scene, x), B, cx, n_ranks)

    @staticmethod
    def block_histogram(scene: Scene, x: np.ndarray) -> np.ndarray:
        """particle count per x-block column of base cells"""
        B = block_edge(scene.dim)
        nbx = -(-scene.config.cells[0] // B)
        return np.bincount(np.clip(base_cell_x(scene, x) // B, 0, nbx - 1), minlength=nbx).astype(np.float64)

    @staticmethod
    def from_histogram(hist: np.ndarray, B: int, cells_x: int, n_ranks: int) -> "SlabPlan":
        """balanced cuts: each block boundary whose cumulative count is closest to k/R of the total,
        at least one block per rank"""
        nbx = len(hist)
        cum = np.concatenate([[0.0], np.cumsum(hist)])
        total = cum[-1]
        cuts = [0]
        for k in range(1, n_ranks):
            lo_c, hi_c = cuts[-1] + 1, nbx - (n_ranks - k)
            c = lo_c + int(np.argmin(np.abs(cum[lo_c:hi_c + 1] - total * k / n_ranks)))
            cuts.append(c)
        cuts.append(nbx)
        bounds = [min(c * B, cells_x) for c in cuts]
        bounds[-1] = cells_x
        return SlabPlan(bounds, B)

    def owner(self, base_x: np.ndarray) -> np.ndarray:
        """rank owning each base cell; out-of-range bases clamp to the edge slabs"""
        return np.clip(np.searchsorted(np.asarray(self.bounds[1:-1]), base_x, side="right"), 0, self.n_ranks - 1)

    def partition(self, scene: Scene, state: SimState) -> list:
        """global particle ids of each rank, ascending"""
        own = self.owner(base_cell_x(scene, state.particles.x))
        return [np.nonzero(own == r)[0].astype(np.int64) for r in range(self.n_ranks)]

    def nodes_per_plane(self, scene: Scene) -> int:
        c = scene.config.cells
        return int(np.prod([c[a] + 1 for a in range(1, scene.dim)]))


# ---------------------------------------------------------------------------------------------
class SlabDomain:
    """Per-rank protocol driven by SlabStepper.

    Buffers are torch tensors: device tensors for the GPU domain, CPU tensors for the oracle
    domain. halo_export must return a tensor that stays valid until the next call.
    """

    rank: int
    plan: SlabPlan

    def p2g(self) -> None: ...
    def grid_interior(self) -> None: ...    # grid update of the nodes off the halo bands
    def halo_export(self, plane_lo: int, n_planes: int, side: int): ...
    def halo_import(self, plane_lo: int, n_planes: int, buf, mode: int) -> None: ...
    def finish_async(self, nan_guard: bool): ...  # -> int64[3] (failed, n_lo, n_hi), may be on device
    def commit(self, n_lo: int, n_hi: int, any_failed: bool) -> None: ...  # raises this rank's error
    def migrate_export(self): ...            # -> (lo_recs, lo_pids, hi_recs, hi_pids)
    def migrate_import(self, recs, pids) -> None: ...
    def local_count(self) -> int: ...
    def gather(self): ...                    # -> (ParticleSoA subset, ids int64)
    def empty_records(self, k: int): ...     # -> (recs, pids) receive buffers
    def empty_halo(self, n_planes: int): ...


class PeerFailure(NumericalError):
    """Another rank aborted this step."""


class LocalTransport:
    """In-process neighbour exchange. Every domain lives in this process and is stepped in
    lock-step, so no rank ever waits on another rank's kernels."""

    def exchange(self, sends: dict, domains: dict, kind: str, report: dict | None = None) -> dict:
        """sends[r] = (to_lo, to_hi) -> recv[r] = (from_lo, from_hi)"""
        out = {}
        for r in domains:
            from_lo = sends[r - 1][1] if r - 1 in sends else None
            from_hi = sends[r + 1][0] if r + 1 in sends else None
            out[r] = (from_lo, from_hi)
        return out

    def start(self, sends: dict, domains: dict, kind: str, report: dict | None = None):
        return self.exchange(sends, domains, kind, report)

    def wait(self, handle) -> dict:
        return handle

    def allgather_obj(self, local: dict) -> dict:
        return dict(local)

    def sum_ordered(self, local: dict) -> np.ndarray:
        """sum of per-rank f64 vectors in rank order (deterministic ParamGrads reduction)"""
        tot = None
        for r in sorted(local):
            tot = local[r].copy() if tot is None else tot + local[r]
        return tot

    def report(self, local: dict, n_ranks: int) -> dict:
        """local[r] = int64 tensor (failed, n_lo, n_hi) or None (failed) -> tuples for every rank"""
        out = {}
        for r, t in local.items():
            f, lo, hi = (1, 0, 0) if t is None else [int(v) for v in t.tolist()]
            out[r] = (bool(f), lo, hi)
        return out


class TorchTransport:
    """torch.distributed point-to-point between x-neighbours (one rank per process)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def _post(self, sends: dict, domains: dict, kind: str, report: dict | None = None):
        """One rank per process: sends[r] = (to_lo, to_hi); migration sizes come from `report`."""
        dist = self.dist
        r = self.rank
        d = domains[r]
        to_lo, to_hi = sends[r]
        lo_peer = r - 1 if r > 0 else None
        hi_peer = r + 1 if r + 1 < self.size else None
        ops, recv = [], {}
        for peer, out in ((lo_peer, to_lo), (hi_peer, to_hi)):
            if peer is None:
                continue
            if kind in ("halo", "halo_cot"):
                inc = d.empty_halo(2) if kind == "halo" else d.empty_halo_cot(2)
                ops += [dist.P2POp(dist.isend, out, peer, self.group), dist.P2POp(dist.irecv, inc, peer, self.group)]
                recv[peer] = inc
                continue
            if out is not None and out[1].numel():
                ops += [dist.P2POp(dist.isend, out[0], peer, self.group), dist.P2POp(dist.isend, out[1], peer, self.group)]
            # what the peer sends us: its count toward this rank
            k = report[peer][2] if peer == lo_peer else report[peer][1]
            if k:
                recs, pids = d.empty_records(k)
                recv[peer] = (recs, pids)
                ops += [dist.P2POp(dist.irecv, recs, peer, self.group), dist.P2POp(dist.irecv, pids, peer, self.group)]
        works = dist.batch_isend_irecv(ops) if ops else []
        return works, {r: (recv.get(lo_peer), recv.get(hi_peer))}

    def start(self, sends: dict, domains: dict, kind: str, report: dict | None = None):
        """post the neighbour sends/receives; the caller may enqueue independent work before wait()"""
        return self._post(sends, domains, kind, report)

    def wait(self, handle) -> dict:
        works, recv = handle
        for w in works:
            w.wait()  # NCCL: orders the current stream (the library's); gloo: blocks the host
        return recv

    def exchange(self, sends: dict, domains: dict, kind: str, report: dict | None = None) -> dict:
        return self.wait(self.start(sends, domains, kind, report))

    def report(self, local: dict, n_ranks: int) -> dict:
        import torch

        (r, mine), = local.items()
        if mine is None:
            mine = torch.tensor([1, 0, 0], dtype=torch.int64, device=self._dev)
        allr = torch.empty(self.size * 3, dtype=torch.int64, device=self._dev)
        self.dist.all_gather_into_tensor(allr, mine, group=self.group)
        rows = allr.view(self.size, 3).cpu().tolist()  # the one host synchronisation of the exchange
        return {q: (bool(rows[q][0]), rows[q][1], rows[q][2]) for q in range(self.size)}

    def allgather_obj(self, local: dict) -> dict:
        (r, obj), = local.items()
        out = [None] * self.size
        self.dist.all_gather_object(out, obj, group=self.group)
        return {q: out[q] for q in range(self.size)}

    def sum_ordered(self, local: dict) -> np.ndarray:
        """all-gather of the per-rank f64 vectors, summed in rank order on every rank (a NCCL/gloo
        all-reduce does not fix the summation order)"""
        import torch

        (r, vec), = local.items()
        t = torch.as_tensor(np.ascontiguousarray(vec), dtype=torch.float64).to(self._dev)
        allv = torch.empty(self.size * t.numel(), dtype=torch.float64, device=self._dev)
        self.dist.all_gather_into_tensor(allv, t, group=self.group)
        rows = allv.view(self.size, -1).cpu().numpy()
        tot = rows[0].copy()
        for q in range(1, self.size):
            tot = tot + rows[q]
        return tot

    _dev = "cpu"


class SlabStepper:
    """Drives one step of the decomposition over the domains this process owns.

    Mirrors Stepper::advance (stepper.hpp:49-70). Every rank advances by one step, and an
    error on any rank raises on all of them at the same step.
    """

    def __init__(self, domains: list, transport, rebalance_every: int = 0, imbalance: float = 1.2):
        """rebalance_every > 0: every that many steps, re-plan the slabs when the largest rank holds
        more than `imbalance` times the mean particle count (granular flows spread)"""
        self.domains = {d.rank: d for d in domains}
        self.transport = transport
        self.rebalance_every = int(rebalance_every)
        self.imbalance = float(imbalance)
        self.rebalances = 0
        if isinstance(transport, TorchTransport):
            import torch

            d0 = next(iter(self.domains.values()))
            transport._dev = d0.device
            # NCCL: the first operation on the group involves every rank before any P2P batch
            t = torch.zeros(1, device=transport._dev)
            transport.dist.all_reduce(t, group=transport.group)
            if getattr(d0, "stream", None) is not None:
                d0.stream.wait_stream(torch.cuda.current_stream(d0.device))
        self.migrated = 0
        self.steps_done = 0  # steps every rank completed (an aborted step is not counted)

    def step(self, nan_guard: bool = False):
        stream = getattr(next(iter(self.domains.values())), "stream", None)
        if stream is not None:
            import torch

            with torch.cuda.stream(stream):
                return self._step(nan_guard)
        return self._step(nan_guard)

    def _step(self, nan_guard: bool):
        doms = self.domains
        n_ranks = next(iter(doms.values())).plan.n_ranks
        errs: dict = {}
        reps: dict = {}
        for r, d in doms.items():
            try:
                d.p2g()
            except MPMError as e:
                errs[r] = e
        # halo: the 2 node planes shared with each neighbour
        sends = {}
        for r, d in doms.items():
            p = d.plan
            to_lo = d.halo_export(p.lo(r), 2, 0) if r > 0 else None
            to_hi = d.halo_export(p.hi(r), 2, 1) if r + 1 < n_ranks else None
            sends[r] = (to_lo, to_hi)
        pending = self.transport.start(sends, doms, "halo")
        for r, d in doms.items():  # nodes off the bands, while the bands travel
            if r not in errs:
                d.grid_interior()
        recv = self.transport.wait(pending)
        for r, d in doms.items():
            from_lo, from_hi = recv[r]
            p = d.plan
            if from_lo is not None:
                d.halo_import(p.lo(r), 2, from_lo, 1)  # lower rank's partial first
            if from_hi is not None:
                d.halo_import(p.hi(r), 2, from_hi, 2)  # own partial first
            if r in errs:
                reps[r] = None
                continue
            try:
                reps[r] = d.finish_async(nan_guard)  # (failed, n_lo, n_hi), written behind G2P
            except MPMError as e:
                errs[r] = e
                reps[r] = None
        # one gather of (failed, n_lo, n_hi) from every rank: the step's only host synchronisation
        rep = self.transport.report(reps, n_ranks)
        any_failed = any(v[0] for v in rep.values())
        for r, d in doms.items():
            if r in errs:
                continue
            try:
                d.commit(rep[r][1], rep[r][2], any_failed)  # raises this rank's own error
            except MPMError as e:
                errs[r] = e
        if any_failed:
            for r in doms:
                if r in errs:
                    raise errs[r]
            raise PeerFailure("step aborted on another rank")
        if rep.get(0, (0, 0, 0))[1] or rep.get(n_ranks - 1, (0, 0, 0))[2]:
            raise NumericalError("a particle left the outermost slab")  # OOD catches this first
        if not any(v[1] or v[2] for v in rep.values()):
            # no rank exported a particle (every rank holds the same gathered report, so all skip
            # together): the export/exchange/import would move nothing. MEASURED at C4 N=1: 19 us of
            # host time per step, all of it exposed behind the report's synchronisation.
            self.steps_done += 1
            return
        # migration of particles that left their slab
        sends = {}
        for r, d in doms.items():
            lo_r, lo_p, hi_r, hi_p = d.migrate_export()
            sends[r] = ((lo_r, lo_p) if r > 0 else None, (hi_r, hi_p) if r + 1 < n_ranks else None)
        recv = self.transport.exchange(sends, doms, "mig", rep)
        for r, d in doms.items():
            parts = [x for x in recv[r] if x is not None and x[1].numel()]
            if parts:
                import torch

                recs = parts[0][0] if len(parts) == 1 else torch.cat([x[0] for x in parts])
                pids = parts[0][1] if len(parts) == 1 else torch.cat([x[1] for x in parts])
                d.migrate_import(recs, pids)
                self.migrated += int(pids.shape[0])
        self.steps_done += 1

    def advance(self, n: int, nan_guard: bool = False):
        for _ in range(int(n)):
            self.step(nan_guard)
            if self.rebalance_every and self.steps_done % self.rebalance_every == 0:
                self.maybe_rebalance()

    def counts(self) -> dict:
        return {r: int(c) for r, c in self.transport.allgather_obj({r: d.local_count()
                                                                   for r, d in self.domains.items()}).items()}

    def maybe_rebalance(self) -> bool:
        c = self.counts()
        mean = sum(c.values()) / len(c)
        if mean <= 0 or max(c.values()) <= self.imbalance * mean:
            return False
        self.rebalance()
        return True

    def rebalance(self):
        """New slab bounds from the global x-block histogram (summed over the ranks in rank order),
        then every particle moves to its new owner: host-orchestrated (rebalancing is rare), the
        received particles appended in id order so the storage order stays deterministic."""
        doms = self.domains
        d0 = next(iter(doms.values()))
        scene, old = d0.scene, d0.plan
        snaps = {r: d.gather() for r, d in doms.items()}
        hist = self.transport.sum_ordered({r: SlabPlan.block_histogram(scene, sub.x)
                                           for r, (sub, ids, _) in snaps.items()})
        plan = SlabPlan.from_histogram(hist, old.block, scene.config.cells[0], old.n_ranks)
        out = {}
        for r, (sub, ids, _) in snaps.items():
            own = plan.owner(base_cell_x(scene, sub.x))
            out[r] = {q: (sub.take(np.nonzero(own == q)[0]), np.asarray(ids)[own == q]) for q in range(plan.n_ranks)}
        allg = self.transport.allgather_obj(out)
        for r, d in doms.items():
            parts = [allg[src][r] for src in sorted(allg)]
            ids = np.concatenate([p[1] for p in parts]).astype(np.int64)
            order = np.argsort(ids, kind="stable")
            tmpl = snaps[r][0]
            sub = ParticleSoA(len(ids), tmpl.dim, tmpl.dtype, tmpl.affine is not None, tmpl.def_grad is not None)
            at = 0
            for p in parts:
                k = len(p[1])
                sub.put(np.arange(at, at + k), p[0])
                at += k
            step, time = snaps[r][2]
            d.retarget(plan, sub.take(order), ids[order], step, time)
        self.rebalances += 1

    def gather_local(self, template: SimState) -> SimState:
        """Assemble the global state from domains in this process (every rank local)"""
        out = template.copy()
        step = None
        for d in self.domains.values():
            sub, ids, st = d.gather()
            out.particles.put(ids, sub)
            step = st
        if step is not None:
            out.step, out.time = step
        return out


# ---------------------------------------------------------------------------------------------
class GpuSlabDomain(SlabDomain):
    """One rank's slab on one GPU, through the C ABI (include/mpm_capi.h, slab section)."""

    def __init__(self, scene: Scene, plan: SlabPlan, rank: int, state: SimState, ids: np.ndarray | None = None,
                 device: int = 0, capacity: int | None = None, mig_cap: int | None = None, local: bool = False):
        """state: the global state (this rank takes rows `ids`, default its slab's particles), or
        with local=True this rank's particles already, `ids` their global ids."""
        import torch

        from . import capi
        from .solver import Context

        self.scene, self.plan, self.rank = scene, plan, rank
        self.device = torch.device("cuda", device)
        if local:
            sub = state
            n_total = state.particles.size() * plan.n_ranks
        else:
            if ids is None:
                ids = plan.partition(scene, state)[rank]
            sub = SimState(state.particles.take(ids), state.step, state.time)
            n_total = state.particles.size()
        # room for particles arriving from the neighbours (a quarter of an average slab by default)
        self.capacity = int(capacity or max(1024, int(1.25 * len(ids)) + n_total // (4 * plan.n_ranks) + 1024))
        self.mig_cap = int(mig_cap or max(1024, self.capacity // 8))
        self.ctx = Context(scene, self.capacity, device)
        self.lib, self.h = self.ctx.lib, self.ctx.h
        # the library, the halo/migration buffers and the transport share one stream per device
        self.stream = _slab_stream(device)
        self.ctx.check(self.lib.mpm_ctx_set_stream(self.h, C.c_void_p(self.stream.cuda_stream)))
        self.ctx.check(self.lib.mpm_slab_set(self.h, plan.lo(rank), plan.hi(rank), self.mig_cap))
        v, keep = sub.to_view()
        ids64 = np.ascontiguousarray(ids, dtype=np.int64)
        self.ctx.check(self.lib.mpm_state_upload_ids(self.h, C.byref(v), ids64.ctypes.data_as(C.c_void_p)))
        self.rec = int(self.lib.mpm_particle_record_size(self.h))
        self.tdtype = torch.float64 if scene.np_dtype == np.float64 else torch.float32
        self.nf = 1 + 2 * scene.dim
        self.per = plan.nodes_per_plane(scene)
        with torch.cuda.stream(self.stream):
            self._halo = [self.empty_halo(2), self.empty_halo(2)]
            self._mig = [(torch.empty((self.mig_cap, self.rec), dtype=self.tdtype, device=self.device),
                          torch.empty(self.mig_cap, dtype=torch.int32, device=self.device)) for _ in range(2)]
        self._counts = (0, 0)
        with torch.cuda.stream(self.stream):
            self._rep = torch.zeros(3, dtype=torch.int64, device=self.device)
        self._template = sub
        self._flags = capi

    def empty_halo(self, n_planes: int):
        import torch

        return torch.empty((n_planes * self.per, self.nf), dtype=self.tdtype, device=self.device)

    def empty_records(self, k: int):
        import torch

        return (torch.empty((k, self.rec), dtype=self.tdtype, device=self.device),
                torch.empty(k, dtype=torch.int32, device=self.device))

    def p2g(self):
        self.ctx.check(self.lib.mpm_step_p2g_local(self.h))

    def grid_interior(self):
        self.ctx.check(self.lib.mpm_step_grid_interior(self.h))

    def halo_export(self, plane_lo, n_planes, side):
        buf = self._halo[side]
        self.ctx.check(self.lib.mpm_halo(self.h, int(plane_lo), int(n_planes), C.c_void_p(buf.data_ptr()), 0))
        return buf

    def halo_import(self, plane_lo, n_planes, buf, mode):
        buf = buf.contiguous()
        self.ctx.check(self.lib.mpm_halo(self.h, int(plane_lo), int(n_planes), C.c_void_p(buf.data_ptr()), int(mode)))

    def finish(self, nan_guard):
        """synchronous form (status read here); the stepper uses finish_async + commit"""
        self.ctx.check(self.lib.mpm_step_finish_local(self.h, self._flags.MPM_ADV_NAN_GUARD if nan_guard else 0))
        nlo, nhi = C.c_int64(), C.c_int64()
        self.ctx.check(self.lib.mpm_migrate_counts(self.h, C.byref(nlo), C.byref(nhi)))
        self._counts = (nlo.value, nhi.value)
        return self._counts

    def finish_async(self, nan_guard):
        self.ctx.check(self.lib.mpm_step_finish_async(self.h, self._flags.MPM_ADV_NAN_GUARD if nan_guard else 0,
                                                      C.c_void_p(self._rep.data_ptr())))
        return self._rep

    def commit(self, n_lo, n_hi, any_failed):
        self.ctx.check(self.lib.mpm_step_commit(self.h, int(n_lo), int(n_hi), int(bool(any_failed))))
        self._counts = (int(n_lo), int(n_hi))

    def migrate_export(self):
        (lr, lp), (hr, hp) = self._mig
        nlo, nhi = C.c_int64(), C.c_int64()
        self.ctx.check(self.lib.mpm_migrate_export(self.h, C.c_void_p(lr.data_ptr()), C.c_void_p(lp.data_ptr()),
                                                   C.c_void_p(hr.data_ptr()), C.c_void_p(hp.data_ptr()),
                                                   self.mig_cap, C.byref(nlo), C.byref(nhi)))
        return lr[: nlo.value], lp[: nlo.value], hr[: nhi.value], hp[: nhi.value]  # stream-ordered copies

    def migrate_import(self, recs, pids):
        recs, pids = recs.contiguous(), pids.contiguous()
        self.ctx.check(self.lib.mpm_migrate_import(self.h, C.c_void_p(recs.data_ptr()), C.c_void_p(pids.data_ptr()),
                                                   int(pids.numel())))

    def local_count(self) -> int:
        return int(self.lib.mpm_local_count(self.h))

    def retarget(self, plan: SlabPlan, particles: ParticleSoA, ids, step: int, time: float):
        """move to new slab bounds and load this rank's new particle set (rebalancing)"""
        self.plan = plan
        if len(ids) > self.capacity:  # grow: a fresh context on the same stream
            from .solver import Context

            self.ctx.close()
            self.capacity = int(1.25 * len(ids)) + 1024
            self.ctx = Context(self.scene, self.capacity, self.device.index or 0)
            self.lib, self.h = self.ctx.lib, self.ctx.h
            self.ctx.check(self.lib.mpm_ctx_set_stream(self.h, C.c_void_p(self.stream.cuda_stream)))
        self.ctx.check(self.lib.mpm_slab_set(self.h, plan.lo(self.rank), plan.hi(self.rank), self.mig_cap))
        self.restore(particles, ids, step, time)

    def restore(self, particles: ParticleSoA, ids, step: int, time: float):
        """load a checkpoint of this rank (its particles, their global ids, step, time)"""
        v, keep = SimState(particles, step, time).to_view()
        ids64 = np.ascontiguousarray(ids, dtype=np.int64)
        self.ctx.check(self.lib.mpm_state_upload_ids(self.h, C.byref(v), ids64.ctypes.data_as(C.c_void_p)))

    # ---- step_vjp over the slab (adjoint.hpp:328-525 decomposed; include/mpm_capi.h) ----------
    def empty_halo_cot(self, n_planes: int):
        import torch

        return torch.empty((n_planes * self.per, 2 * self.scene.dim), dtype=self.tdtype, device=self.device)

    def vjp_begin(self, state: SimState, cot_out):
        """state: this rank's particles at step t (replaces the context's state), cot_out the
        cotangents of the same particles at t + 1, same order"""
        v, keep = state.to_view()
        self.ctx.check(self.lib.mpm_state_upload(self.h, C.byref(v)))
        co, kco = cot_out.to_view()
        self.ctx.check(self.lib.mpm_slab_vjp_begin(self.h, C.byref(co)))
        self._vjp_state = state
        if not hasattr(self, "_hcot"):
            import torch

            with torch.cuda.stream(self.stream):
                self._hcot = [self.empty_halo_cot(2), self.empty_halo_cot(2)]

    def vjp_interior(self):
        self.ctx.check(self.lib.mpm_slab_vjp_interior(self.h))

    def vjp_scatter(self):
        self.ctx.check(self.lib.mpm_slab_vjp_scatter(self.h))

    def halo_cot_export(self, plane_lo, n_planes, side):
        buf = self._hcot[side]
        self.ctx.check(self.lib.mpm_halo_cot(self.h, int(plane_lo), int(n_planes), C.c_void_p(buf.data_ptr()), 0))
        return buf

    def halo_cot_import(self, plane_lo, n_planes, buf, mode):
        buf = buf.contiguous()
        self.ctx.check(self.lib.mpm_halo_cot(self.h, int(plane_lo), int(n_planes), C.c_void_p(buf.data_ptr()),
                                             int(mode)))

    def vjp_finish(self):
        from .state import ParamGrads, StateCotangent

        cin = StateCotangent.zeros_like(self._vjp_state.particles)
        ci, kci = cin.to_view()
        pg = ParamGrads(self.scene.boundary)
        pv = pg.to_view()
        self.ctx.check(self.lib.mpm_slab_vjp_finish(self.h, C.byref(ci), C.byref(pv)))
        cin.sync_from(kci)
        pg.sync_from(pv)
        return cin, pg

    def gather(self):
        k = self.local_count()
        p = self._template.particles
        sub = SimState(ParticleSoA(k, p.dim, p.dtype, p.affine is not None, p.def_grad is not None))
        v, keep = sub.output_view()
        ids = np.empty(max(k, 1), np.int64)
        self.ctx.check(self.lib.mpm_state_download_local(self.h, C.byref(v), ids.ctypes.data_as(C.c_void_p)))
        sub.sync_from(v, keep)
        return sub.particles, ids[:k], (sub.step, sub.time)

    def close(self):
        self.ctx.close()


def slab_step_vjp(domains: list, transport, states: dict, cot_outs: dict, pg) -> dict:
    """step_vjp (adjoint.hpp:328-331) over the slab decomposition: states[r] / cot_outs[r] are rank
    r's particles at step t and their cotangents at t + 1 (same order). Returns cot_in per rank
    (overwritten semantics) and accumulates the ParamGrads of all ranks into pg, summed in rank
    order. Two halo exchanges: the forward replay's (m, p, f) and the node (v, v_old) cotangents;
    the interior grid replay overlaps the first."""
    doms = {d.rank: d for d in domains}
    stream = getattr(next(iter(doms.values())), "stream", None)
    if stream is not None:
        import torch

        with torch.cuda.stream(stream):
            return _slab_step_vjp(doms, transport, states, cot_outs, pg)
    return _slab_step_vjp(doms, transport, states, cot_outs, pg)


def _slab_step_vjp(doms, transport, states, cot_outs, pg):
    n_ranks = next(iter(doms.values())).plan.n_ranks
    for r, d in doms.items():
        d.vjp_begin(states[r], cot_outs[r])

    def exchange(export, imp, kind, overlap=None):
        sends = {}
        for r, d in doms.items():
            p = d.plan
            sends[r] = (export(d, p.lo(r), 0) if r > 0 else None, export(d, p.hi(r), 1) if r + 1 < n_ranks else None)
        pending = transport.start(sends, doms, kind)
        if overlap is not None:
            for d in doms.values():
                overlap(d)
        recv = transport.wait(pending)
        for r, d in doms.items():
            from_lo, from_hi = recv[r]
            if from_lo is not None:
                imp(d, d.plan.lo(r), from_lo, 1)  # lower rank's partial first
            if from_hi is not None:
                imp(d, d.plan.hi(r), from_hi, 2)

    exchange(lambda d, lo, side: d.halo_export(lo, 2, side), lambda d, lo, b, m: d.halo_import(lo, 2, b, m), "halo",
             overlap=lambda d: d.vjp_interior())
    for d in doms.values():
        d.vjp_scatter()
    exchange(lambda d, lo, side: d.halo_cot_export(lo, 2, side), lambda d, lo, b, m: d.halo_cot_import(lo, 2, b, m),
             "halo_cot")
    out, parts = {}, {}
    for r, d in doms.items():
        out[r], pr = d.vjp_finish()
        parts[r] = pr.flat()
    pg.add_flat(transport.sum_ordered(parts))
    return out


def _digest(particles: ParticleSoA, ids) -> int:
    """order-independent content digest of a rank's particles (id-sorted bytes)"""
    import hashlib

    o = np.argsort(np.asarray(ids), kind="stable")
    h = hashlib.sha256(np.asarray(ids)[o].tobytes())
    for f in ("x", "v", "volume", "rho", "eps_eq", "sigma_zz", "sigma", "grad_v", "affine"):
        a = getattr(particles, f)
        if a is not None and a.size:
            h.update(np.ascontiguousarray(a[o]).tobytes())
    return int.from_bytes(h.digest()[:8], "little")


def slab_backprop_trajectory(scene: Scene, plan, seeder, domains: list, transport, n_total: int):
    """backprop_trajectory (checkpoint.hpp:72-143) over the slab decomposition.

    The domains hold the initial state. Per rank, checkpoints are the rank's (particles, ids) at
    segment starts. The replay of a segment is checked against the forward sweep's boundary
    digest (checkpoint.hpp:124-126), and the reverse sweep runs slab_step_vjp. A rank's
    cotangent rows at step t are those of its particles at t. Particles that migrated during the
    step get their cotangent from an id-indexed assembly through the transport, which costs O(N)
    host traffic per step; a neighbour-only exchange of the migrants' rows is the scalable form.
    The seeder is evaluated per rank on global ids (LagrangianLeastSquares.loss_local / seed_local),
    with loss terms summed in rank order. Returns a solver.BackpropResult with the global
    initial-state cotangent.
    """
    from .errors import NumericalError as _NE
    from .solver import BackpropResult
    from .state import ParamGrads, StateCotangent

    doms = {d.rank: d for d in domains}
    stp = SlabStepper(domains, transport)

    def gather():
        return {r: d.gather() for r, d in doms.items()}

    glob = getattr(seeder, "global_stats", False)  # Eulerian: region sums span the ranks

    def stats(step, snap):
        return transport.sum_ordered({r: seeder.stats_local(step, sub, ids) for r, (sub, ids, _) in snap.items()})

    def loss_of(step, snap):
        if not seeder.observes(step):
            return 0.0
        if glob:
            return seeder.loss_from_stats(step, stats(step, snap))
        part = {r: np.array([seeder.loss_local(step, sub, ids)]) for r, (sub, ids, _) in snap.items()}
        return float(transport.sum_ordered(part)[0])

    # forward sweep: checkpoints at segment starts, digests at every boundary
    nseg = plan.n_segments
    snap = gather()
    loss = loss_of(0, snap)
    ckpt, bdig = [], []
    for k in range(nseg):
        ckpt.append(snap)
        bdig.append({r: _digest(sub, ids) for r, (sub, ids, _) in snap.items()})
        for t in range(plan.boundaries[k], plan.boundaries[k + 1]):
            stp.step()
            if seeder.observes(t + 1):
                snap = gather()
                loss += loss_of(t + 1, snap)
        snap = gather()
    bdig.append({r: _digest(sub, ids) for r, (sub, ids, _) in snap.items()})

    # backward sweep (host-global cotangent rows by id)
    template = next(iter(snap.values()))[0]
    cot = StateCotangent(n_total, template.dim, template.dtype, template.affine is not None)
    pg = ParamGrads(scene.boundary)
    peak = 0

    def seed(step, snap_t):
        if not seeder.observes(step):
            return
        local = {}
        st = stats(step, snap_t) if glob else None
        for r, (sub, ids, _) in snap_t.items():
            rows, dz = seeder.seed_local(step, sub, ids, st) if glob else seeder.seed_local(step, sub, ids)
            local[r] = (np.asarray(ids)[rows], dz)
        for r in sorted(allg := transport.allgather_obj(local)):
            gid, dz = allg[r]
            tgt = cot.x if seeder.field == "x" else cot.v
            tgt[gid] += dz

    for k in range(nseg - 1, -1, -1):
        b0, b1 = plan.boundaries[k], plan.boundaries[k + 1]
        for r, d in doms.items():
            sub, ids, (st, tm) = ckpt[k][r]
            d.restore(sub, ids, st, tm)
        replay = [ckpt[k]]
        for _ in range(b0, b1):
            stp.step()
            replay.append(gather())
        if {r: _digest(sub, ids) for r, (sub, ids, _) in replay[-1].items()} != bdig[k + 1]:
            raise _NE(f"checkpoint mismatch: recomputed segment end differs from the recorded state at step {b1}")
        peak = max(peak, len(replay))
        for t in range(b1, b0, -1):
            seed(t, replay[t - b0])
            prev = replay[t - b0 - 1]
            states = {r: SimState(sub, st, tm) for r, (sub, ids, (st, tm)) in prev.items()}
            outs = {r: cot.take(np.asarray(ids)) for r, (sub, ids, _) in prev.items()}
            cin = slab_step_vjp(domains, transport, states, outs, pg)
            allg = transport.allgather_obj({r: (np.asarray(prev[r][1]), cin[r]) for r in cin})
            cot = StateCotangent(n_total, template.dim, template.dtype, template.affine is not None)
            for r in sorted(allg):
                gid, c = allg[r]
                cot.put(gid, c)
    seed(0, ckpt[0])
    return BackpropResult(cot, pg, loss, nseg, peak)


_STREAMS: dict = {}


def _slab_stream(device: int):
    import torch

    if device not in _STREAMS:
        _STREAMS[device] = torch.cuda.Stream(device=device)
    return _STREAMS[device]


def local_slab_run(scene: Scene, state: SimState, n_ranks: int, steps: int, nan_guard: bool = False,
                   device: int = 0, balance: bool = True):
    """Single-process decomposition on one GPU (R contexts stepped in lock-step): the testable
    form of the multi-GPU path. Returns (final global state, stepper)."""
    plan = SlabPlan.make(scene, n_ranks, state.particles.x if balance else None)
    ids = plan.partition(scene, state)
    doms = [GpuSlabDomain(scene, plan, r, state, ids[r], device) for r in range(n_ranks)]
    stp = SlabStepper(doms, LocalTransport())
    stp.advance(steps, nan_guard)
    out = stp.gather_local(state)
    return out, stp, plan


__all__ = ["SlabPlan", "SlabDomain", "SlabStepper", "LocalTransport", "TorchTransport", "GpuSlabDomain",
           "PeerFailure", "local_slab_run", "slab_step_vjp", "slab_backprop_trajectory", "block_edge", "base_cell_x"]


# ---------------------------------------------------------------------------------------------
# The library-owned decomposition (include/mpm_capi.h, mpm_dist_*): the same slab step, run
# inside libmpm_b200 with device-resident counts and no host synchronisation inside a call. The
# classes above orchestrate the step from Python (the protocol reference, and the decomposed
# adjoint); these drive the C++ path.
def dist_unique_id() -> bytes:
    """An NCCL unique id from the library (rank 0 makes it, every rank receives it)."""
    from . import capi

    lib = capi.load_library()
    buf = (C.c_ubyte * capi.DIST_ID_BYTES)()
    rc = lib.mpm_dist_unique_id(buf)
    if rc:
        raise MPMError(f"mpm_dist_unique_id failed ({rc})")
    return bytes(buf)


def _dist_capacity(n_local: int, n_total: int, n_ranks: int, mig_cap: int) -> int:
    """room for particles arriving from the neighbours: a quarter of an average slab, plus one
    step's worst-case arrivals (2 mig_cap)"""
    return max(1024, int(1.25 * n_local) + n_total // (4 * n_ranks) + 2 * mig_cap)


def _dist_cot_views(ctxs, template: SimState):
    """per rank: a writable cotangent view sized for its live particles, plus the id array"""
    from .state import StateCotangent

    outs = []
    p = template.particles
    for c in ctxs:
        k = int(c.lib.mpm_local_count(c.h))
        prt = ParticleSoA(k, p.dim, p.dtype, p.affine is not None, False)
        cot = StateCotangent.zeros_like(prt)
        v, keep = cot.to_view()
        ids = np.empty(max(k, 1), np.int64)
        outs.append((cot, v, keep, ids))
    return outs


def _dist_cot_assemble(outs, n_total: int, template: SimState):
    """rows of every rank (c0.n of them, storage order) -> the global cotangent in id order"""
    from .state import StateCotangent

    glob = StateCotangent.zeros_like(template.particles)
    for cot, v, keep, ids in outs:
        k = int(v.n)
        cot.sync_from(keep)
        live = np.nonzero(ids[:k] >= 0)[0]  # vacated slots (exported particles) carry id -1
        glob.put(ids[live], cot.take(live))
    return glob


class NcclSlabRank:
    """This process's rank of the decomposition (one process per GPU): a context owning particles
    [lo, hi) of the plan and an NCCL communicator (mpm_dist_attach_nccl)."""

    def __init__(self, scene: Scene, plan: SlabPlan, rank: int, state: SimState, ids: np.ndarray, nccl_id: bytes,
                 device: int = 0, n_total: int | None = None, mig_cap: int | None = None, capacity: int | None = None):
        from .solver import Context

        self.scene, self.plan, self.rank = scene, plan, rank
        n_local = state.particles.size()
        n_total = int(n_total or n_local * plan.n_ranks)
        self.mig_cap = int(mig_cap or max(1024, n_total // (256 * plan.n_ranks)))
        self.capacity = int(capacity or _dist_capacity(n_local, n_total, plan.n_ranks, self.mig_cap))
        self.ctx = Context(scene, self.capacity, device)
        self.lib, self.h = self.ctx.lib, self.ctx.h
        v, keep = state.to_view()
        ids64 = np.ascontiguousarray(ids, dtype=np.int64)
        self.ctx.check(self.lib.mpm_state_upload_ids(self.h, C.byref(v), ids64.ctypes.data_as(C.c_void_p)))
        idb = (C.c_ubyte * len(nccl_id)).from_buffer_copy(nccl_id)
        self.ctx.check(self.lib.mpm_dist_attach_nccl(self.h, rank, plan.n_ranks, idb, plan.lo(rank), plan.hi(rank),
                                                     self.mig_cap))
        self._template = state

    def advance(self, n: int, nan_guard: bool = False) -> float:
        """n decomposed steps; returns their device time (ms, CUDA events on the context stream)"""
        from . import capi

        ms = C.c_double()
        self.ctx.check(self.lib.mpm_dist_advance(self.h, int(n), capi.MPM_ADV_NAN_GUARD if nan_guard else 0,
                                                 C.byref(ms)))
        return ms.value

    def backprop(self, total: int, nseg: int, seeder: dict, id_space: int):
        """backprop_trajectory over the decomposition (mpm_dist_backprop): returns (this rank's cotangent
        rows with their global ids, ParamGrads (rank-ordered sum, identical on every rank), result)"""
        from . import capi
        from .seeders import make_seeder_desc
        from .state import ParamGrads

        sd, keep_sd = make_seeder_desc(seeder, self.scene.np_dtype)
        (cot, v, keep, ids), = _dist_cot_views([self.ctx], self._template)
        pg = ParamGrads(self.scene.boundary)
        pv = pg.to_view()
        res = capi.BackpropResultView()
        self.ctx.check(self.lib.mpm_dist_backprop(self.h, int(total), int(nseg), C.byref(sd), int(id_space),
                                                  C.byref(v), ids.ctypes.data_as(C.c_void_p), C.byref(pv),
                                                  C.byref(res)))
        k = int(v.n)
        cot.sync_from(keep)
        pg.sync_from(pv)
        live = np.nonzero(ids[:k] >= 0)[0]  # vacated slots carry id -1
        return cot.take(live), ids[live], pg, res

    def gather(self):
        """(particles, global ids, (step, time)) of this rank's live particles"""
        k = int(self.lib.mpm_local_count(self.h))
        p = self._template.particles
        sub = SimState(ParticleSoA(k, p.dim, p.dtype, p.affine is not None, p.def_grad is not None))
        v, keep = sub.output_view()
        ids = np.empty(max(k, 1), np.int64)
        self.ctx.check(self.lib.mpm_state_download_local(self.h, C.byref(v), ids.ctypes.data_as(C.c_void_p)))
        sub.sync_from(v, keep)
        return sub.particles.take(np.arange(v.n)), ids[:v.n], (sub.step, sub.time)

    def close(self):
        self.ctx.close()


class LocalSlabGroup:
    """All ranks of the decomposition in this process (mpm_dist_attach_local): R contexts, stepped
    in lock-step by the library with device-copy exchanges -- the single-GPU test bed of the NCCL
    path (same phases, same kernels, only the transport differs)."""

    def __init__(self, scene: Scene, plan: SlabPlan, state: SimState, device: int = 0, mig_cap: int | None = None):
        from .solver import Context

        self.scene, self.plan = scene, plan
        parts = plan.partition(scene, state)
        n_total = state.particles.size()
        R = plan.n_ranks
        self.mig_cap = int(mig_cap or max(256, n_total // (64 * R)))
        self.ctxs = []
        for r in range(R):
            ids = parts[r]
            sub = SimState(state.particles.take(ids), state.step, state.time)
            ctx = Context(scene, _dist_capacity(len(ids), n_total, R, self.mig_cap), device)
            v, keep = sub.to_view()
            ids64 = np.ascontiguousarray(ids, dtype=np.int64)
            ctx.check(ctx.lib.mpm_state_upload_ids(ctx.h, C.byref(v), ids64.ctypes.data_as(C.c_void_p)))
            self.ctxs.append(ctx)
        self.lib = self.ctxs[0].lib
        self._arr = (C.c_void_p * R)(*[c.h for c in self.ctxs])
        bounds = (C.c_int * (R + 1))(*plan.bounds)
        rc = self.lib.mpm_dist_attach_local(self._arr, R, bounds, self.mig_cap)
        if rc:
            self.ctxs[0].check(rc)
        self._template = state
        self.n_total = n_total

    def advance(self, n: int, nan_guard: bool = False):
        from . import capi

        rc = self.lib.mpm_dist_advance_local(self._arr, len(self.ctxs), int(n),
                                             capi.MPM_ADV_NAN_GUARD if nan_guard else 0)
        if rc:  # every rank raises at the same step; report the failing rank's own error first
            errs = []
            for c in self.ctxs:
                code = C.c_int()
                buf = C.create_string_buffer(1024)
                c.lib.mpm_last_error(c.h, C.byref(code), None, None, buf, 1024)
                if code.value:
                    errs.append((b"another rank" in buf.value, c, code.value))
            errs.sort(key=lambda e: e[0])
            if errs:
                errs[0][1].check(errs[0][2])
            self.ctxs[0].check(rc)

    def backprop(self, total: int, nseg: int, seeder: dict):
        """backprop_trajectory (checkpoint.hpp:72-143) over the decomposition, device-resident
        (mpm_dist_backprop_local): (global cotangent of S^0 in id order, ParamGrads, result)"""
        from . import capi
        from .seeders import make_seeder_desc
        from .state import ParamGrads

        sd, keep_sd = make_seeder_desc(seeder, self.scene.np_dtype)
        outs = _dist_cot_views(self.ctxs, self._template)
        R = len(self.ctxs)
        views = (capi.CotView * R)(*[o[1] for o in outs])
        idp = (C.c_void_p * R)(*[o[3].ctypes.data for o in outs])
        pg = ParamGrads(self.scene.boundary)
        pv = pg.to_view()
        res = capi.BackpropResultView()
        rc = self.lib.mpm_dist_backprop_local(self._arr, R, int(total), int(nseg), C.byref(sd), int(self.n_total),
                                              views, idp, C.byref(pv), C.byref(res))
        if rc:
            self._raise(rc)
        for k, o in enumerate(outs):
            o[1].n = views[k].n
        pg.sync_from(pv)
        return _dist_cot_assemble(outs, self.n_total, self._template), pg, res

    def _raise(self, rc):
        errs = []
        for c in self.ctxs:
            code = C.c_int()
            buf = C.create_string_buffer(1024)
            c.lib.mpm_last_error(c.h, C.byref(code), None, None, buf, 1024)
            if code.value:
                errs.append((b"another" in buf.value, c, code.value))
        errs.sort(key=lambda e: e[0])
        if errs:
            errs[0][1].check(errs[0][2])
        self.ctxs[0].check(rc)

    def gather(self) -> SimState:
        """the global state in particle-id order"""
        out = self._template.copy()
        step = None
        for c in self.ctxs:
            k = int(c.lib.mpm_local_count(c.h))
            p = self._template.particles
            sub = SimState(ParticleSoA(k, p.dim, p.dtype, p.affine is not None, p.def_grad is not None))
            v, keep = sub.output_view()
            ids = np.empty(max(k, 1), np.int64)
            c.check(c.lib.mpm_state_download_local(c.h, C.byref(v), ids.ctypes.data_as(C.c_void_p)))
            sub.sync_from(v, keep)
            out.particles.put(ids[:v.n], sub.particles.take(np.arange(v.n)))
            step = (v.step, v.time)
        out.step, out.time = step
        return out

    def close(self):
        for c in self.ctxs:
            c.close()
