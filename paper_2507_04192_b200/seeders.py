"""Built-in device loss seeders (SPEC.md observe_lagrangian + masked least-squares loss), the
Seeder protocol of backprop_trajectory (checkpoint.hpp:63-66) without host round-trips."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi


class LagrangianLeastSquares:
    """L = sum_{t in obs_steps} sum_{l in sel} || z_l(t) - target[t][l] ||^2, z = x or v.

    `sel` = particle ids (None = all, in id order); `target` = [n_obs, n_sel, dim]."""

    def __init__(self, obs_steps, target, field: str = "x", sel=None):
        self.obs_steps = list(int(s) for s in obs_steps)
        self.target = np.asarray(target)
        self.field = field
        self.sel = None if sel is None else np.asarray(sel, np.int64)

    def desc(self) -> dict:
        return {"field": self.field, "obs_steps": self.obs_steps, "sel": self.sel, "target": self.target}

    # ---- the same seeder on one rank's particles (slab decomposition; global ids) --------------
    def observes(self, step: int) -> bool:
        return int(step) in self.obs_steps

    def _local(self, step, particles, ids):
        k = self.obs_steps.index(int(step))
        ids = np.asarray(ids, np.int64)
        if self.sel is None:
            rows, l = np.arange(len(ids)), ids
        else:
            if not hasattr(self, "_inv") or len(self._inv) <= (ids.max() if len(ids) else 0):
                n = int(max(self.sel.max() + 1, (ids.max() + 1) if len(ids) else 0))
                self._inv = np.full(n, -1, np.int64)
                self._inv[self.sel] = np.arange(len(self.sel))
            l = self._inv[ids] if len(ids) else ids
            rows = np.nonzero(l >= 0)[0]
            l = l[rows]
        z = (particles.x if self.field == "x" else particles.v)[rows]
        return rows, z - self.target[k][l]

    def loss_local(self, step, particles, ids) -> float:
        """this rank's share of loss_at (checkpoint.hpp:63-66)"""
        _, r = self._local(step, particles, ids)
        return float((r.astype(np.float64) ** 2).sum())

    def seed_local(self, step, particles, ids):
        """(rows, d z) of this rank's share of seed: cot.z[rows] += 2 (z - target)"""
        rows, r = self._local(step, particles, ids)
        return rows, 2 * r


class EulerianLeastSquares:
    """Velocity-monitor supervision (SPEC.md observe_eulerian, PAPER §3.2 and §5.1 "sparse
    velocity-monitor supervision"): region l is the closed box |x - centers[l]| <= half[l];
    Q_l(t) = mean of z over the particles inside; L = sum_t sum_l m[t][l] ||Q_l(t) - target[t][l]||^2,
    an empty region carries no term (mask 0). `half` may be a scalar, per region or per region and
    axis; `mask` = [n_obs, n_regions] of {0, 1} or None."""

    def __init__(self, obs_steps, centers, half, target, field: str = "v", mask=None):
        self.obs_steps = list(int(s) for s in obs_steps)
        self.centers = np.atleast_2d(np.asarray(centers, np.float64))
        nreg, dim = self.centers.shape
        h = np.asarray(half, np.float64)
        self.half = np.broadcast_to(h.reshape(-1, 1) if h.ndim == 1 else h, (nreg, dim)).copy()
        self.target = np.asarray(target)
        self.field = field
        self.mask = None if mask is None else np.asarray(mask, np.uint8)

    def desc(self) -> dict:
        return {"kind": "eulerian", "field": self.field, "obs_steps": self.obs_steps, "centers": self.centers,
                "half": self.half, "target": self.target, "mask": self.mask}

    # ---- slab decomposition: region statistics are summed over the ranks before Q is formed ----
    global_stats = True

    def observes(self, step: int) -> bool:
        return int(step) in self.obs_steps

    def _members(self, particles):
        x = particles.x
        return np.all(np.abs(x[:, None, :] - self.centers[None]) <= self.half[None], axis=2)  # [n, nreg]

    def stats_local(self, step, particles, ids) -> np.ndarray:
        """per region (sum z, count) of this rank's particles, flattened"""
        inm = self._members(particles)
        z = particles.x if self.field == "x" else particles.v
        s = np.concatenate([inm.T.astype(np.float64) @ z.astype(np.float64), inm.sum(0)[:, None]], axis=1)
        return s.reshape(-1)

    def _coef(self, step, stats):
        k = self.obs_steps.index(int(step))
        nreg, dim = self.centers.shape
        st = stats.reshape(nreg, dim + 1)
        cnt = st[:, dim]
        on = cnt > 0
        if self.mask is not None:
            on &= self.mask[k].astype(bool)
        q = np.where(on[:, None], st[:, :dim] / np.where(on, cnt, 1)[:, None], 0.0)
        r = np.where(on[:, None], q - self.target[k], 0.0)
        return r, cnt, on

    def loss_from_stats(self, step, stats) -> float:
        r, _, _ = self._coef(step, stats)
        return float((r ** 2).sum())

    def seed_local(self, step, particles, ids, stats):
        r, cnt, on = self._coef(step, stats)
        g = np.where(on[:, None], 2 * r / np.where(on, cnt, 1)[:, None], 0.0)
        dz = self._members(particles).astype(np.float64) @ g
        return np.arange(len(ids)), dz.astype(particles.x.dtype)


def make_seeder_desc(seeder: dict | None, T):
    sd = capi.SeederDesc()
    if not seeder:
        sd.kind = capi.MPM_SEEDER_NONE
        return sd, {}
    if seeder.get("kind") == "eulerian":
        obs = np.ascontiguousarray(np.asarray(seeder["obs_steps"], np.int64))
        cen = np.ascontiguousarray(np.asarray(seeder["centers"], T))
        half = np.ascontiguousarray(np.asarray(seeder["half"], T))
        tgt = np.ascontiguousarray(np.asarray(seeder["target"], T))
        mask = seeder.get("mask")
        mask = None if mask is None else np.ascontiguousarray(np.asarray(mask, np.uint8))
        sd.kind = capi.MPM_SEEDER_EULERIAN_LS
        sd.field = 0 if seeder.get("field", "v") == "x" else 1
        sd.n_obs = len(obs)
        sd.obs_steps = obs.ctypes.data_as(C.POINTER(C.c_int64))
        sd.n_sel = 0
        sd.target = tgt.ctypes.data
        sd.n_regions = len(cen)
        sd.centers = cen.ctypes.data
        sd.half = half.ctypes.data
        sd.mask = None if mask is None else mask.ctypes.data_as(C.POINTER(C.c_ubyte))
        return sd, {"obs": obs, "cen": cen, "half": half, "tgt": tgt, "mask": mask}
    obs = np.ascontiguousarray(np.asarray(seeder["obs_steps"], np.int64))
    sel = seeder.get("sel")
    sel = None if sel is None else np.ascontiguousarray(np.asarray(sel, np.int64))
    tgt = np.ascontiguousarray(np.asarray(seeder["target"], T))
    sd.kind = capi.MPM_SEEDER_LAGRANGIAN_LS
    sd.field = 0 if seeder.get("field", "x") == "x" else 1
    sd.n_obs = len(obs)
    sd.obs_steps = obs.ctypes.data_as(C.POINTER(C.c_int64))
    sd.n_sel = 0 if sel is None else len(sel)
    sd.sel = None if sel is None else sel.ctypes.data_as(C.POINTER(C.c_int64))
    sd.target = tgt.ctypes.data
    return sd, {"obs": obs, "sel": sel, "tgt": tgt}
