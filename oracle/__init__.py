"""CPU oracle loader -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package, and only as the checker or the timed CPU baseline -- never on the product
path (paper_2507_04192_b200 fails loudly when its CUDA library is missing).

    CpuOracle("orc")  the restatement          oracle/_build/liboracle.so  (oracle/mpm_oracle.cpp)
    CpuOracle("ref")  the reference, unmodified oracle/_ref/libmpm_ref.so  (oracle/ref_capi.cpp)

Both expose the same stateless ABI (oracle/mpm_oracle.h) over the product's host types
(paper_2507_04192_b200.state / .scene).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

from paper_2507_04192_b200 import capi
from paper_2507_04192_b200.errors import raise_for
from paper_2507_04192_b200.state import Grid, ParamGrads, SimState, StateCotangent

HERE = Path(__file__).resolve().parent
LIBS = {"orc": HERE / "_build" / "liboracle.so", "ref": HERE / "_ref" / "libmpm_ref.so",
        "ref_v3": HERE / "_ref" / "libmpm_ref_v3.so"}  # the reference at -march=x86-64-v3


class OrcRegion(C.Structure):
    _fields_ = [
        ("shape", C.c_int),
        ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("center", C.c_double * 3),
        ("radius", C.c_double), ("zmin", C.c_double), ("zmax", C.c_double),
        ("vel_kind", C.c_int), ("value", C.c_double * 3),
        ("alpha", C.c_double), ("h0", C.c_double), ("amplitude", C.c_double),
        ("perturbation", C.c_double), ("frequency", C.c_double),
    ]


def build(quiet: bool = True) -> None:
    """make -C oracle (restatement always; the reference too when /root/reference exists)."""
    out = subprocess.run(["make", "-C", str(HERE), "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])


def available(kind: str) -> bool:
    return LIBS[kind].exists()


_VELK = {"constant": 0, "linear_in_y": 1, "parabolic_sine": 2}


def _regions(scene):
    arr = (OrcRegion * max(1, len(scene.geometry)))()
    for i, g in enumerate(scene.geometry):
        r = arr[i]
        r.shape = 0 if g.shape == "box" else 1
        for a in range(scene.dim):
            if g.lo is not None:
                r.lo[a] = g.lo[a]
            if g.hi is not None:
                r.hi[a] = g.hi[a]
            if g.center is not None:
                r.center[a] = g.center[a]
            if g.velocity.value is not None:
                r.value[a] = g.velocity.value[a]
        r.radius, r.zmin, r.zmax = g.radius, g.zmin, g.zmax
        ve = g.velocity
        r.vel_kind = _VELK[ve.kind]
        r.alpha, r.h0, r.amplitude, r.perturbation, r.frequency = (
            ve.alpha, ve.h0, ve.amplitude, ve.perturbation, ve.frequency)
    return arr


class CpuOracle:
    def __init__(self, kind: str = "orc"):
        if kind not in LIBS:
            raise ValueError(kind)
        if not LIBS[kind].exists():
            raise RuntimeError(f"oracle library {LIBS[kind]} missing; run `make -C oracle`")
        self.kind = kind
        lib = C.CDLL(str(LIBS[kind]))
        P = "ref_" if kind.startswith("ref") else "orc_"
        sig = {
            "last_error": (C.c_int, [C.POINTER(C.c_int64), C.c_char_p, C.c_size_t]),
            "dp_make": (C.c_int, [C.POINTER(capi.SceneDesc)] + [C.c_double] * 7),
            "init_scene_count": (C.c_int64, [C.POINTER(capi.SceneDesc), C.c_void_p, C.c_int]),
            "init_scene": (C.c_int, [C.POINTER(capi.SceneDesc), C.c_void_p, C.c_int, C.POINTER(capi.StateView),
                                     C.POINTER(C.c_double)]),
            "advance": (C.c_int, [C.POINTER(capi.SceneDesc), C.POINTER(capi.StateView), C.c_int64, C.c_int]),
            "p2g": (C.c_int, [C.POINTER(capi.SceneDesc), C.POINTER(capi.StateView), C.POINTER(capi.GridView)]),
            "grid_momentum_update": (C.c_int, [C.POINTER(capi.SceneDesc), C.POINTER(capi.GridView)]),
            "grid_corrections": (C.c_int, [C.POINTER(capi.SceneDesc), C.POINTER(capi.GridView)]),
            "g2p": (C.c_int, [C.POINTER(capi.SceneDesc), C.POINTER(capi.GridView), C.POINTER(capi.StateView)]),
            "constitutive": (C.c_int, [C.POINTER(capi.SceneDesc), C.POINTER(capi.StateView)]),
            "step_vjp": (C.c_int, [C.POINTER(capi.SceneDesc), C.POINTER(capi.StateView), C.POINTER(capi.CotView),
                                   C.POINTER(capi.CotView), C.POINTER(capi.ParamGradsView)]),
            "backprop": (C.c_int, [C.POINTER(capi.SceneDesc), C.POINTER(capi.StateView), C.c_int64, C.c_int,
                                   C.POINTER(capi.SeederDesc), C.POINTER(capi.CotView),
                                   C.POINTER(capi.ParamGradsView), C.POINTER(capi.BackpropResultView)]),
            "state_hash": (C.c_uint64, [C.POINTER(capi.SceneDesc), C.POINTER(capi.StateView)]),
            "run_seconds_per_1000": (C.c_double, [C.POINTER(capi.SceneDesc), C.POINTER(capi.StateView), C.c_int64]),
        }
        self.f = {}
        for k, (res, args) in sig.items():
            fn = getattr(lib, P + k)
            fn.restype, fn.argtypes = res, args
            self.f[k] = fn
        self._lib = lib

    # -- errors --------------------------------------------------------------------------
    def _check(self, rc):
        if rc != 0:
            p = C.c_int64(-1)
            buf = C.create_string_buffer(512)
            self.f["last_error"](C.byref(p), buf, 512)
            raise_for(rc, p.value, buf.value.decode(errors="replace"))

    # -- scene -----------------------------------------------------------------------------
    def dp_make(self, rho0, K, nu, phi, psi, cohesion, sigma_t):
        from paper_2507_04192_b200.scene import DruckerPragerParams
        d = capi.SceneDesc()
        self._check(self.f["dp_make"](C.byref(d), rho0, K, nu, phi, psi, cohesion, sigma_t))
        return DruckerPragerParams(**{k: getattr(d, k) for k in (
            "rho0", "K", "nu", "G", "phi", "psi", "cohesion", "sigma_t", "q_phi", "k_phi", "q_psi", "tau_P",
            "alpha_P")})

    def init_scene(self, scene) -> SimState:
        dh = scene.to_desc()
        regs = _regions(scene)
        n = self.f["init_scene_count"](dh.ref, regs, len(scene.geometry))
        if n < 0:
            meps = C.c_double()
            self._check(self.f["init_scene"](dh.ref, regs, len(scene.geometry), None, C.byref(meps)))
        cfg = scene.config
        st = SimState.zeros(n, scene.dim, scene.np_dtype, cfg.scheme.uses_affine(), cfg.track_def_grad)
        v, keep = st.output_view()
        meps = C.c_double()
        self._check(self.f["init_scene"](dh.ref, regs, len(scene.geometry), C.byref(v), C.byref(meps)))
        st.sync_from(v, keep)
        scene.mass_epsilon = meps.value
        return st

    # -- forward -------------------------------------------------------------------------
    def advance(self, scene, state: SimState, n: int = 1, nan_guard: bool = False):
        dh = scene.to_desc()
        v, keep = state.to_view()
        rc = self.f["advance"](dh.ref, C.byref(v), n, int(nan_guard))
        state.sync_from(v, {k: (a.reshape(-1) if a is not None else None) for k, a in keep.items()})
        self._check(rc)
        return state

    def new_grid(self, scene) -> Grid:
        c = scene.config
        return Grid(c.cells, c.dh, c.origin, scene.np_dtype, scene.dim)

    def p2g(self, scene, state: SimState) -> Grid:
        g = self.new_grid(scene)
        v, keep = state.to_view()
        self._check(self.f["p2g"](scene.to_desc().ref, C.byref(v), C.byref(g.to_view())))
        return g

    def grid_momentum_update(self, scene, g: Grid) -> Grid:
        self._check(self.f["grid_momentum_update"](scene.to_desc().ref, C.byref(g.to_view())))
        return g

    def grid_corrections(self, scene, g: Grid) -> Grid:
        self._check(self.f["grid_corrections"](scene.to_desc().ref, C.byref(g.to_view())))
        return g

    def g2p(self, scene, g: Grid, state: SimState) -> SimState:
        v, keep = state.to_view()
        self._check(self.f["g2p"](scene.to_desc().ref, C.byref(g.to_view()), C.byref(v)))
        state.sync_from(v, {k: (a.reshape(-1) if a is not None else None) for k, a in keep.items()})
        return state

    def constitutive(self, scene, state: SimState) -> SimState:
        v, keep = state.to_view()
        rc = self.f["constitutive"](scene.to_desc().ref, C.byref(v))
        state.sync_from(v, {k: (a.reshape(-1) if a is not None else None) for k, a in keep.items()})
        self._check(rc)
        return state

    # -- adjoint -------------------------------------------------------------------------
    def step_vjp(self, scene, state: SimState, cot_out: StateCotangent, pg: ParamGrads | None = None):
        pg = pg or ParamGrads(scene.boundary)
        v, keep = state.to_view()
        co, kco = cot_out.to_view()
        cin = StateCotangent.zeros_like(state.particles)
        ci, kci = cin.to_view()
        pv = pg.to_view()
        self._check(self.f["step_vjp"](scene.to_desc().ref, C.byref(v), C.byref(co), C.byref(ci), C.byref(pv)))
        cin.sync_from({k: (a.reshape(-1) if a is not None else None) for k, a in kci.items()})
        pg.sync_from(pv)
        return cin, pg

    def backprop(self, scene, state: SimState, total_steps: int, n_segments: int, seeder: dict):
        """seeder: {"field": "x"|"v", "obs_steps": [...], "sel": ids or None, "target": [n_obs, n_sel, dim]}"""
        sd, keep_sd = make_seeder(seeder, scene.np_dtype)
        v, keep = state.to_view()
        c0 = StateCotangent.zeros_like(state.particles)
        cv, kc = c0.to_view()
        pg = ParamGrads(scene.boundary)
        pv = pg.to_view()
        res = capi.BackpropResultView()
        self._check(self.f["backprop"](scene.to_desc().ref, C.byref(v), total_steps, n_segments, C.byref(sd),
                                       C.byref(cv), C.byref(pv), C.byref(res)))
        c0.sync_from({k: (a.reshape(-1) if a is not None else None) for k, a in kc.items()})
        pg.sync_from(pv)
        return c0, pg, res

    def state_hash(self, scene, state: SimState) -> int:
        v, keep = state.to_view()
        return int(self.f["state_hash"](scene.to_desc().ref, C.byref(v)))

    def run_seconds_per_1000(self, scene, state: SimState, n: int) -> float:
        v, keep = state.to_view()
        secs = self.f["run_seconds_per_1000"](scene.to_desc().ref, C.byref(v), n)
        state.sync_from(v, {k: (a.reshape(-1) if a is not None else None) for k, a in keep.items()})
        return secs


def make_seeder(seeder: dict | None, T):
    """Builds an mpm_seeder_desc (Lagrangian or Eulerian least squares) plus its keep-alive arrays;
    the descriptor layout is the product ABI's (include/mpm_capi.h), so the package builds it."""
    from paper_2507_04192_b200.seeders import make_seeder_desc

    return make_seeder_desc(seeder, T)
