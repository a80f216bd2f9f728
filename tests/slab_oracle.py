"""Oracle-backed slab domain: TEST INFRASTRUCTURE ONLY.

This implements the per-rank protocol of paper_2507_04192_b200.distributed.SlabDomain on top of
the CPU oracle's phase functions. The phases follow the reference's Stepper::advance
(stepper.hpp:59-69), run on one rank's particle subset:
  - p2g: the reference's p2g with `g m_i` inside the scatter (transfer.hpp:62);
  - halo sum;
  - grid_momentum_update, apply_grid_corrections, g2p, constitutive_update;
  - migration.
It lets the CPU suite exercise the decomposition's orchestration: the plan, the halo bands,
migration, the transports, and gloo world_size 2. The product domain is GpuSlabDomain.
"""
from __future__ import annotations

import numpy as np
import torch

from paper_2507_04192_b200.distributed import SlabDomain, SlabPlan, base_cell_x
from paper_2507_04192_b200.state import ParticleSoA, SimState


class OracleSlabDomain(SlabDomain):
    def __init__(self, scene, plan: SlabPlan, rank: int, state: SimState, ids, orc):
        self.scene, self.plan, self.rank, self.orc = scene, plan, rank, orc
        self.device = torch.device("cpu")
        self.sub = SimState(state.particles.take(ids), state.step, state.time)
        self.ids = np.asarray(ids, np.int64)
        self.grid = None
        self.nf = 1 + 2 * scene.dim
        self.per = plan.nodes_per_plane(scene)
        self.tdtype = torch.float64 if scene.np_dtype == np.float64 else torch.float32
        self._out = None

    # ---- grid phases -----------------------------------------------------------------------
    def p2g(self):
        if self.sub.particles.size():
            self.grid = self.orc.p2g(self.scene, self.sub)
        else:
            self.grid = self.orc.new_grid(self.scene)

    def grid_interior(self):
        pass  # the oracle's p2g already formed the whole grid; nothing to overlap

    def _band(self, plane_lo, n_planes):
        return slice(plane_lo * self.per, (plane_lo + n_planes) * self.per)

    def halo_export(self, plane_lo, n_planes, side):
        g, sl = self.grid, self._band(plane_lo, n_planes)
        a = np.concatenate([g.mass[sl, None], g.momentum[sl], g.force[sl]], axis=1)
        return torch.from_numpy(np.ascontiguousarray(a))

    def halo_import(self, plane_lo, n_planes, buf, mode):
        g, sl = self.grid, self._band(plane_lo, n_planes)
        b = buf.numpy()
        d = self.scene.dim
        for arr, cols in ((g.mass, slice(0, 1)), (g.momentum, slice(1, 1 + d)), (g.force, slice(1 + d, 1 + 2 * d))):
            own = arr[sl].reshape(-1, cols.stop - cols.start)
            rec = b[:, cols]
            tot = rec + own if mode == 1 else own + rec
            arr[sl] = tot.reshape(arr[sl].shape)

    def empty_halo(self, n_planes):
        return torch.empty((n_planes * self.per, self.nf), dtype=self.tdtype)

    def finish(self, nan_guard):
        sc, st = self.scene, self.sub
        self.orc.grid_momentum_update(sc, self.grid)
        self.orc.grid_corrections(sc, self.grid)
        if st.particles.size():
            self.orc.g2p(sc, self.grid, st)
            self.orc.constitutive(sc, st)
        st.step += 1
        T = sc.np_dtype
        st.time = float(T(st.step) * T(sc.config.dt))
        if nan_guard and not st.particles.all_finite():
            from paper_2507_04192_b200.errors import NumericalError

            raise NumericalError(f"run: non-finite particle field detected at step {st.step}")
        bx = base_cell_x(self.scene, st.particles.x)
        self._lo_idx = np.nonzero(bx < self.plan.lo(self.rank))[0]
        self._hi_idx = np.nonzero(bx >= self.plan.hi(self.rank))[0]
        return len(self._lo_idx), len(self._hi_idx)

    def finish_async(self, nan_guard):
        self._err = None
        try:
            lo, hi = self.finish(nan_guard)
            return torch.tensor([0, lo, hi], dtype=torch.int64)
        except Exception as e:  # reported through the gather, raised by commit
            self._err = e
            return torch.tensor([1, 0, 0], dtype=torch.int64)

    def commit(self, n_lo, n_hi, any_failed):
        if any_failed and self._err is not None:
            raise self._err

    # ---- migration ---------------------------------------------------------------------------
    def _pack(self, idx):
        p = self.sub.particles
        k, d = len(idx), p.dim
        cols = [p.x[idx], p.v[idx], p.mass[idx, None], p.volume[idx, None], p.rho[idx, None], p.eps_eq[idx, None],
                p.sigma_zz[idx, None] if d == 2 else np.zeros((k, 1), p.dtype),
                p.sigma[idx].reshape(k, d * d), p.grad_v[idx].reshape(k, d * d)]
        if p.affine is not None:
            cols.append(p.affine[idx].reshape(k, d * d))
        if p.def_grad is not None:
            cols.append(p.def_grad[idx].reshape(k, d * d))
        return torch.from_numpy(np.ascontiguousarray(np.concatenate(cols, axis=1)))

    def _unpack(self, recs: np.ndarray) -> ParticleSoA:
        p = self.sub.particles
        k, d = len(recs), p.dim
        out = ParticleSoA(k, d, p.dtype, p.affine is not None, p.def_grad is not None)
        q = 0

        def take(w):
            nonlocal q
            a = recs[:, q:q + w]
            q += w
            return a

        out.x[...] = take(d)
        out.v[...] = take(d)
        out.mass[...] = take(1)[:, 0]
        out.volume[...] = take(1)[:, 0]
        out.rho[...] = take(1)[:, 0]
        out.eps_eq[...] = take(1)[:, 0]
        szz = take(1)[:, 0]
        if d == 2:
            out.sigma_zz[...] = szz
        out.sigma[...] = take(d * d).reshape(k, d, d)
        out.grad_v[...] = take(d * d).reshape(k, d, d)
        if out.affine is not None:
            out.affine[...] = take(d * d).reshape(k, d, d)
        if out.def_grad is not None:
            out.def_grad[...] = take(d * d).reshape(k, d, d)
        return out

    def rec_size(self):
        return int(self._pack(np.zeros(0, np.int64)).shape[1])

    def empty_records(self, k):
        return torch.empty((k, self.rec_size()), dtype=self.tdtype), torch.empty(k, dtype=torch.int32)

    def migrate_export(self):
        lo_idx, hi_idx = self._lo_idx, self._hi_idx
        out = (self._pack(lo_idx), torch.from_numpy(self.ids[lo_idx].astype(np.int32)),
               self._pack(hi_idx), torch.from_numpy(self.ids[hi_idx].astype(np.int32)))
        keep = np.ones(self.sub.particles.size(), bool)
        keep[lo_idx] = False
        keep[hi_idx] = False
        keep_idx = np.nonzero(keep)[0]
        self.sub.particles = self.sub.particles.take(keep_idx)
        self.ids = self.ids[keep_idx]
        return out

    def migrate_import(self, recs, pids):
        pids = pids.numpy().astype(np.int64)
        order = np.argsort(pids, kind="stable")  # append in particle-id order, as the device does
        new = self._unpack(recs.numpy()[order])
        old = self.sub.particles
        merged = ParticleSoA(old.size() + new.size(), old.dim, old.dtype, old.affine is not None,
                             old.def_grad is not None)
        merged.put(np.arange(old.size()), old)
        merged.put(np.arange(old.size(), merged.size()), new)
        self.sub.particles = merged
        self.ids = np.concatenate([self.ids, pids[order]])

    def local_count(self):
        return self.sub.particles.size()

    def retarget(self, plan, particles, ids, step, time):
        self.plan = plan
        self.sub = SimState(particles, step, time)
        self.ids = np.asarray(ids, np.int64)

    def gather(self):
        return self.sub.particles, self.ids, (self.sub.step, self.sub.time)
