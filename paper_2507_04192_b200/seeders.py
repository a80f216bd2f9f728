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


def make_seeder_desc(seeder: dict | None, T):
    sd = capi.SeederDesc()
    if not seeder:
        sd.kind = capi.MPM_SEEDER_NONE
        return sd, {}
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
