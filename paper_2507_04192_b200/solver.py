"""Python mirror of the reference solver API (stepper.hpp, adjoint.hpp, checkpoint.hpp) over the
C ABI of libmpm_b200.so. Names, argument meaning and error behaviour follow the reference:

    Stepper(scene).advance(state)                    stepper.hpp:49-70
    run(scene, state, n, stride, force, observer)    stepper.hpp:91-122
    step_vjp(scene, state, cot_out, cot_in, pg, ws)  adjoint.hpp:328-525
    backprop_trajectory(scene, s0, plan, seeder)     checkpoint.hpp:72-143
    CheckpointPlan.make(N_t, n)                      checkpoint.hpp:15-34

Every call runs on the GPU through the in-tree CUDA library; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import time as _time
from dataclasses import dataclass, field

import numpy as np

from . import capi
from .errors import ValidationError, raise_for
from .scene import Scene, cfl_report
from .state import Grid, ParamGrads, SimState, StateCotangent


class Context:
    """Owns one device context (mpm_ctx) for a scene; the device-side Stepper."""

    def __init__(self, scene: Scene, max_particles: int, device: int = 0):
        self.lib = capi.load_library()
        self.scene = scene
        self._desc = scene.to_desc()
        h = C.c_void_p()
        rc = self.lib.mpm_ctx_create(C.byref(self._desc.desc), int(max_particles), device, C.byref(h))
        if rc != 0:
            raise_for(rc, -1, f"mpm_ctx_create failed (status {rc}); an sm_100 GPU is required")
        self.h = h
        self.max_particles = int(max_particles)

    def close(self):
        if getattr(self, "h", None):
            self.lib.mpm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- errors -----------------------------------------------------------------------------
    def check(self, rc: int):
        if rc != 0:
            code, p, s = C.c_int(), C.c_int64(), C.c_int64()
            buf = C.create_string_buffer(1024)
            self.lib.mpm_last_error(self.h, C.byref(code), C.byref(p), C.byref(s), buf, 1024)
            raise_for(rc, p.value, buf.value.decode(errors="replace"))

    def last_error_step(self) -> int:
        code, p, s = C.c_int(), C.c_int64(), C.c_int64()
        self.lib.mpm_last_error(self.h, C.byref(code), C.byref(p), C.byref(s), None, 0)
        return s.value

    # -- state --------------------------------------------------------------------------------
    def upload(self, state: SimState):
        v, keep = state.to_view()
        self.check(self.lib.mpm_state_upload(self.h, C.byref(v)))

    def init_scene(self, scene: Scene) -> int:
        """init_scene (scene.hpp:55-116) seeded on the device into this context:
        the same particles, order and bits as scene.init_scene (except parabolic_sine's sin).
        Returns the particle count; sets scene.mass_epsilon like init_scene."""
        from .scene import seeding_constants

        regs, mass, volume, rho0 = seeding_constants(scene)
        arr = (capi.Region * len(regs))(*regs)
        n = C.c_int64()
        self.check(self.lib.mpm_init_scene(self.h, arr, len(regs), mass, volume, rho0, C.byref(n)))
        return n.value

    def snapshot_begin(self, slot: int):
        self.check(self.lib.mpm_snapshot_begin(self.h, int(slot)))

    def snapshot_fetch(self, slot: int, template: SimState) -> SimState:
        out = template.copy()
        v, keep = out.output_view()
        self.check(self.lib.mpm_snapshot_fetch(self.h, int(slot), C.byref(v)))
        out.sync_from(v, keep)
        return out

    def download(self, state: SimState) -> SimState:
        v, keep = state.output_view()
        self.check(self.lib.mpm_state_download(self.h, C.byref(v)))
        state.sync_from(v, keep)
        return state

    def advance(self, n: int, nan_guard: bool = False, store_grid: bool = False):
        flags = (capi.MPM_ADV_NAN_GUARD if nan_guard else 0) | (capi.MPM_ADV_STORE_GRID if store_grid else 0)
        self.check(self.lib.mpm_advance(self.h, int(n), flags))

    def advance_timed(self, n: int, nan_guard: bool = False) -> float:
        """advance n steps; returns the device time (ms) from CUDA events on the context stream"""
        ms = C.c_double()
        self.check(self.lib.mpm_advance_timed(self.h, int(n), capi.MPM_ADV_NAN_GUARD if nan_guard else 0,
                                              C.byref(ms)))
        return ms.value

    def digest(self) -> int:
        d = C.c_uint64()
        self.check(self.lib.mpm_state_digest(self.h, C.byref(d)))
        return d.value

    def max_speed(self) -> float:
        v = C.c_double()
        self.check(self.lib.mpm_max_speed(self.h, C.byref(v)))
        return v.value

    def new_grid(self) -> Grid:
        c = self.scene.config
        return Grid(c.cells, c.dh, c.origin, self.scene.np_dtype, self.scene.dim)

    def grid_download(self, g: Grid | None = None) -> Grid:
        g = g or self.new_grid()
        self.check(self.lib.mpm_grid_download(self.h, C.byref(g.to_view())))
        return g

    def grid_upload(self, g: Grid):
        self.check(self.lib.mpm_grid_upload(self.h, C.byref(g.to_view())))

    # -- phases -------------------------------------------------------------------------------
    def p2g(self):
        self.check(self.lib.mpm_p2g(self.h))

    def grid_momentum_update(self):
        self.check(self.lib.mpm_grid_momentum_update(self.h))

    def grid_corrections(self):
        self.check(self.lib.mpm_grid_corrections(self.h))

    def g2p(self):
        self.check(self.lib.mpm_g2p(self.h))

    def constitutive(self):
        self.check(self.lib.mpm_constitutive(self.h))

    # -- instrumentation ------------------------------------------------------------------------
    def profile(self, enable: bool):
        self.check(self.lib.mpm_profile_enable(self.h, int(enable)))

    def profile_reset(self):
        self.check(self.lib.mpm_profile_reset(self.h))

    def profile_query(self, name: str = "") -> tuple[float, int]:
        ms, k = C.c_double(), C.c_int64()
        self.check(self.lib.mpm_profile_query(self.h, name.encode(), C.byref(ms), C.byref(k)))
        return ms.value, k.value

    def launch_count(self) -> int:
        return int(self.lib.mpm_launch_count(self.h))

    def grid_stats(self) -> tuple[int, int, int]:
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        self.check(self.lib.mpm_grid_stats(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    # -- adjoint ----------------------------------------------------------------------------------
    def step_vjp(self, state: SimState, cot_out: StateCotangent, pg: ParamGrads) -> StateCotangent:
        v, keep = state.to_view()
        co, kco = cot_out.to_view()
        cin = StateCotangent.zeros_like(state.particles)
        ci, kci = cin.to_view()
        pv = pg.to_view()
        self.check(self.lib.mpm_step_vjp(self.h, C.byref(v), C.byref(co), C.byref(ci), C.byref(pv)))
        cin.sync_from(kci)
        pg.sync_from(pv)
        return cin

    def backprop(self, state: SimState, total: int, nseg: int, seeder: dict | None):
        from .seeders import make_seeder_desc
        sd, keep_sd = make_seeder_desc(seeder, self.scene.np_dtype)
        v, keep = state.to_view()
        c0 = StateCotangent.zeros_like(state.particles)
        cv, kc = c0.to_view()
        pg = ParamGrads(self.scene.boundary)
        pv = pg.to_view()
        res = capi.BackpropResultView()
        self.check(self.lib.mpm_backprop(self.h, C.byref(v), int(total), int(nseg), C.byref(sd), C.byref(cv),
                                         C.byref(pv), C.byref(res)))
        c0.sync_from(kc)
        pg.sync_from(pv)
        return c0, pg, res


# -------------------------------------------------------------------------------------------
_CTX_CACHE: dict = {}


def init_scene_device(scene: Scene, device: int = 0, capacity: int | None = None) -> Context:
    """init_scene (scene.hpp:55-116) seeded directly on the device: returns a
    Context holding the seeded state, with the same CFL refusal as init_scene for fluids."""
    from .scene import FluidParams, seeding_capacity, seeding_constants

    seeding_constants(scene)  # validates and sets mass_epsilon before the context copies the scene
    ctx = Context(scene, capacity or seeding_capacity(scene), device)
    ctx.n = ctx.init_scene(scene)
    if isinstance(scene.material, FluidParams):
        courant = cfl_report(scene.config, scene.material, ctx.max_speed())
        if courant > 1:
            ctx.close()
            raise ValidationError(f"scene: CFL violation, Courant number {courant} > 1 (reduce dt or coarsen the grid)")
    return ctx


def _context_for(scene: Scene, n: int) -> Context:
    """One cached context per (scene identity, capacity)."""
    key = id(scene)
    ctx = _CTX_CACHE.get(key)
    if ctx is None or ctx.max_particles < n or ctx.scene is not scene or _scene_changed(ctx, scene):
        if ctx is not None:
            ctx.close()
        ctx = Context(scene, max(n, 1))
        _CTX_CACHE[key] = ctx
    return ctx


def _scene_changed(ctx: Context, scene: Scene) -> bool:
    return bytes(scene.to_desc().desc) != bytes(ctx._desc.desc)


class Stepper:
    """stepper.hpp:49-70. `grid` is a host mirror refreshed on demand (the device grid is
    derived data, so poisoning this copy between steps changes nothing, as in the reference)."""

    def __init__(self, scene: Scene):
        self.scene = scene
        c = scene.config
        self.grid = Grid(c.cells, c.dh, c.origin, scene.np_dtype, scene.dim)
        self._ctx: Context | None = None

    def advance(self, state: SimState):
        n = state.particles.size()
        if self._ctx is None or self._ctx.max_particles < n or _scene_changed(self._ctx, self.scene):
            self._ctx = Context(self.scene, n)
        self._ctx.upload(state)
        self._ctx.advance(1, store_grid=True)
        self._ctx.download(state)

    def fetch_grid(self) -> Grid:
        if self._ctx is not None:
            self._ctx.grid_download(self.grid)
        return self.grid


@dataclass
class RunResult:
    """stepper.hpp:72-76"""
    snapshots: list = field(default_factory=list)
    seconds_per_1000_steps: float = 0.0


def max_particle_speed(state: SimState) -> float:
    """stepper.hpp:78-85"""
    return float(np.sqrt((state.particles.v.astype(np.float64) ** 2).sum(axis=1)).max()) if state.particles.size() else 0.0


def run(scene: Scene, state: SimState, num_steps: int, stride: int, force: bool = False, observer=None) -> RunResult:
    """stepper.hpp:91-122: CFL refusal, NaN guard every step, snapshots at the stride, the
    reference's own timer. Steps between snapshots run as one device call."""
    courant = cfl_report(scene.config, scene.material, max_particle_speed(state))
    if courant > 1 and not force:
        raise ValidationError(f"run: Courant number {courant} > 1; refusing to start (use force to override)")
    state = state.copy()
    res = RunResult()
    res.snapshots.append(state.copy())
    ctx = Context(scene, state.particles.size())
    ctx.upload(state)
    t0 = _time.perf_counter()
    s = 0
    pending = []  # snapshot slots in flight (their D2H copies overlap the following steps)

    def take():
        res.snapshots.append(ctx.snapshot_fetch(pending.pop(0), state))

    while s < num_steps:
        if observer is not None:
            chunk = 1
        elif stride > 0:
            chunk = min(num_steps - s, stride - (state.step + s) % stride if (state.step + s) % stride else stride)
        else:
            chunk = num_steps - s
        ctx.advance(chunk, nan_guard=True, store_grid=observer is not None)
        s += chunk
        cur_step = state.step + s
        if observer is not None:
            st = ctx.download(state.copy())
            observer(st, ctx.grid_download())
        if stride > 0 and cur_step % stride == 0 and cur_step != num_steps:
            free = ({0, 1} - set(pending))
            if not free:
                take()
                free = ({0, 1} - set(pending))
            slot = min(free)
            ctx.snapshot_begin(slot)
            pending.append(slot)
    t1 = _time.perf_counter()
    while pending:
        take()
    if num_steps > 0:
        res.snapshots.append(ctx.download(state.copy()))
        res.seconds_per_1000_steps = (t1 - t0) / num_steps * 1000.0
    ctx.close()
    return res


def constitutive_update(scene: Scene, state: SimState):
    """stepper.hpp:15-43 on the device (phase function)."""
    ctx = _context_for(scene, state.particles.size())
    ctx.upload(state)
    ctx.constitutive()
    ctx.download(state)


# ---- adjoint ----------------------------------------------------------------------------------
class AdjointWorkspace:
    """adjoint.hpp:297-322: here it just caches the device context."""

    def __init__(self):
        self.ctx: Context | None = None


def step_vjp(scene: Scene, state: SimState, cot_out: StateCotangent, cot_in: StateCotangent | None,
             pg: ParamGrads, ws: AdjointWorkspace | None = None) -> StateCotangent:
    """adjoint.hpp:328-525: cot_in is overwritten, pg accumulated. Returns cot_in."""
    ws = ws or AdjointWorkspace()
    n = state.particles.size()
    if ws.ctx is None or ws.ctx.max_particles < n or _scene_changed(ws.ctx, scene):
        ws.ctx = Context(scene, n)
    res = ws.ctx.step_vjp(state, cot_out, pg)
    if cot_in is not None:
        for f in StateCotangent.FIELDS:
            a = getattr(cot_in, f)
            if a is not None:
                a[...] = getattr(res, f)
        return cot_in
    return res


@dataclass
class CheckpointPlan:
    """checkpoint.hpp:10-51"""
    total_steps: int
    n_segments: int
    boundaries: list

    @staticmethod
    def make(total_steps: int, n_segments: int) -> "CheckpointPlan":
        if total_steps < 1:
            raise ValidationError("checkpoint plan: need at least one step")
        if n_segments < 1 or n_segments > total_steps:
            raise ValidationError("checkpoint plan: n_segments must lie in [1, N_t]")
        base, rem = divmod(total_steps, n_segments)
        b, at = [0], 0
        for k in range(n_segments):
            at += base + (1 if k < rem else 0)
            b.append(at)
        return CheckpointPlan(total_steps, n_segments, b)

    def segment_length(self, k):
        return self.boundaries[k + 1] - self.boundaries[k]

    def max_segment_length(self):
        return max(self.segment_length(k) for k in range(self.n_segments))

    def planned_peak_states(self):
        return self.n_segments + self.max_segment_length() + 1


@dataclass
class BackpropResult:
    """checkpoint.hpp:53-61"""
    initial_state_cot: StateCotangent
    param_grads: ParamGrads
    loss: float
    checkpoints_stored: int
    peak_replay_states: int

    def measured_peak_states(self):
        return self.checkpoints_stored + self.peak_replay_states


def backprop_trajectory(scene: Scene, initial: SimState, plan: CheckpointPlan, seeder) -> BackpropResult:
    """checkpoint.hpp:72-143 with a built-in device seeder (paper_2507_04192_b200.seeders)."""
    ctx = Context(scene, initial.particles.size())
    c0, pg, res = ctx.backprop(initial, plan.total_steps, plan.n_segments, seeder.desc() if seeder else None)
    ctx.close()
    return BackpropResult(c0, pg, res.loss, res.checkpoints_stored, res.peak_replay_states)
