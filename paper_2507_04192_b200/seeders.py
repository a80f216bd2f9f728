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
