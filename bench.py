#!/usr/bin/env python
"""Benchmark of the B200 MPM step (BASELINE.json metric: particle-steps/s, fwd, with HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config C4] [--dtype f64]

Workload (N=1): C4 -- 3-D granular column collapse, Drucker-Prager sand, FLIP, 128x64x64-cell
column = 4,194,304 particles on a 256^3 grid, f64 (the reference's precision), synthetic input
from init_scene. A "step" is one forward MPM step Phi over all particles.
  value      particle-steps/s over K steps timed with CUDA events on the library's stream,
             state resident in HBM (1.4 GB >> 126 MB L2: no flush needed), max over ranks.
  e2e        the same metric through the reference-facing C ABI with HOST buffers: one
             `run`-style call = mpm_state_upload (pinned host -> device) + mpm_advance(K) +
             mpm_state_download, wall-clock, so host<->device copies are inside the region.
  roofline   dominant kernel (largest share of the step) measured live with CUDA events:
             algorithmic bytes per launch / mean launch time vs MEASURED_PEAKS.json hbm_gbs;
             plus the whole-step figure N_p * B_fwd / t_step (B_fwd from SURVEY.md §8d).
  cpu_baseline  the reference compiled unmodified (oracle/_ref, "reference") -- or the oracle
             restatement ("port") if absent -- on a bounded sample of the same workload, one
             process per host core.
N>1 (torchrun): weak scaling through the slab decomposition of SURVEY.md §8e
(paper_2507_04192_b200/distributed.py). The C4 domain becomes 256N x 256 x 256 cells with one
column per rank, and rank r owns the slab x in [256r, 256(r+1)). Every step does a real NCCL halo
exchange of the 2 shared node planes and migrates particles that cross a slab. The time is
max-over-ranks device time (CUDA events around K steps). `--mode slab` runs the same path at N=1.
--impl reference: the reference's own CPU implementation of the step on all host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "particle-steps/sec (fwd)"
UNIT = "particle-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-workloads", action="store_true", help="skip the C2/C3/C5 sub-lines")
    ap.add_argument("--slab-adj", action="store_true",
                    help="slab mode: also time the host-orchestrated decomposed backprop (slow; DESIGN.md §7)")
    ap.add_argument("--adj-steps", type=int, default=20, help="fwd+adjoint sample: backprop steps (0: skip)")
    ap.add_argument("--long-adj", type=int, default=1000,
                    help="also time a backprop over this many steps with the HBM-sized checkpoint plan (0: skip)")
    ap.add_argument("--adj-segments", type=int, default=0,
                    help="checkpoint segments of the fwd+adjoint sample (0: fewest that fit in HBM)")
    ap.add_argument("--mode", default="auto", choices=["auto", "plain", "slab", "pyslab"],
                    help="auto: one context at N=1, the library's slab decomposition (mpm_dist_*, NCCL) for "
                         "N>1; slab: that path at any N; pyslab: the Python-orchestrated protocol reference")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1 with C4: weak = one C4 column per GPU (256N x 256 x 256 domain); strong = the one "
                         "C4 scene split into N slabs")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---- algorithmic bytes ------------------------------------------------------
def gv_dead(scene) -> bool:
    """FLIP / PIC / blend without F tracking never read the stored grad v: inside one advance()
    call only the last step writes it"""
    return scene.config.scheme.kind not in ("apic", "tpic") and not scene.config.track_def_grad


def bytes_model(scene, n_particles, active_nodes, steps_per_call=1):
    """B_fwd = (IN + OUT) s + (A/N_p) 2 (1 + 2d) s, IN/OUT per SURVEY §8d (D-P adds eps, 2-D sigma_zz).
    This is SURVEY §8d's figure (the one the roofline is scored on), with OUT holding grad v. With
    steps_per_call > 1 and gv_dead(), grad v is stored once per advance() call instead, and the
    return value is the traffic the implementation actually needs (reported beside it)."""
    d = scene.dim
    s = 8 if scene.dtype == "f64" else 4
    ns = 3 if d == 2 else 6
    dp = scene.material.__class__.__name__ == "DruckerPragerParams"
    IN = 2 * d + 2 + 1 + ns + (1 if dp else 0) + (1 if (dp and d == 2) else 0)    # x v m V rho sig (+eps, +szz)
    OUT = 2 * d + 2 + ns + d * d + (1 if dp else 0) + (1 if (dp and d == 2) else 0)  # x v V rho sig gradv (+eps, +szz)
    if gv_dead(scene):
        OUT -= d * d * (1 - 1 / steps_per_call)
    per_particle = (IN + OUT) * s
    grid = 2 * (1 + 2 * d) * s * active_nodes / n_particles
    return per_particle + grid, IN, OUT


def kernel_bytes(scene, n, active_nodes, occupied_blocks):
    """Per launch of the two particle kernels: SURVEY §8(d)'s COMPULSORY bytes ("algorithmic":
    every particle field the kernel must read or write, once, and each active node's fields once)
    next to the bytes the implementation actually moves ("moved": + the sort permutation / keys /
    particle ids and the (B+2)^d partial tiles of every occupied block instead of the active nodes).
      k_p2g  reads x v m V sigma; writes the active nodes' m p f once
      k_g2p  reads x v V rho sigma (+eps, +sigma_zz) and the active nodes' v v_old; writes
             x v V rho sigma grad v (+eps, +sigma_zz) -- grad v counted as SURVEY does
             ("needed" drops it: FLIP stores it only on a call's last step)"""
    d = scene.dim
    s = 8 if scene.dtype == "f64" else 4
    ns = 3 if d == 2 else 6
    dp = scene.material.__class__.__name__ == "DruckerPragerParams"
    B = 16 if d == 2 else 8
    tile = (B + 2) ** d
    nf = 1 + 2 * d
    extra = (1 if dp else 0) + (1 if (dp and d == 2) else 0)  # eps (+ sigma_zz)
    p2g_in = 2 * d + 2 + ns
    g2p_in = 2 * d + 2 + ns + extra
    g2p_out = g2p_in + d * d
    alg = {"k_p2g": n * p2g_in * s + active_nodes * nf * s,
           "k_g2p": n * (g2p_in + g2p_out) * s + active_nodes * 2 * d * s}
    need = {"k_p2g": alg["k_p2g"], "k_g2p": alg["k_g2p"] - (n * d * d * s if gv_dead(scene) else 0)}
    moved = {"k_p2g": n * (p2g_in * s + 8) + occupied_blocks * tile * nf * s,
             "k_g2p": n * ((g2p_in + 1 + g2p_out) * s + 4 * 4) + occupied_blocks * tile * 2 * d * s}
    return alg, need, moved


# particle counts of the configs' init_scene seeding (pinned by tests/test_gpu_configs.py)
N_PARTICLES = {"C1": 20_000, "C2": 250_000, "C3": 102_400, "C4": 4_194_304, "C5": 32_505_856}
GRID = {"C1": [128, 128], "C2": [512, 512], "C3": [480, 192], "C4": [256, 256, 256], "C5": [512, 256, 128]}
DESC = {"C4": "3-D D-P granular column collapse, FLIP, 128x64x64-cell column on a 256^3 grid, dt 1e-5, f64",
        "C1": "2-D D-P column (Bui), 20k particles, 128^2", "C2": "2-D dam break, fluid, 250k particles, 512^2",
        "C3": "2-D inverse-velocity scene, fluid, 102k particles, 480x192",
        "C5": "3-D landslide, D-P + 32-segment Coulomb floor, 32.5M particles, 512x256x128"}


def run_mode(a, world):
    if a.mode == "pyslab":
        return "pyslab"
    return "dist" if (a.mode == "slab" or (a.mode == "auto" and world > 1)) else "plain"


def workload_config(a, world):
    """The line's `config`: the static description of the workload, identical in both arms
    (--impl b200 and --impl reference) at the same N. Measured quantities (active nodes, bytes,
    slab bounds after balancing, migration counts) live in `roofline` / `slab`, not here."""
    mode = run_mode(a, world)
    n = N_PARTICLES[a.config]
    cells = list(GRID[a.config])
    l2 = "inputs larger than the 126 MB L2 (state >= 0.9 GB f64 per GPU at C4); no flush"
    if mode == "plain":
        return {"workload": f"{a.config}: {DESC[a.config]}", "particles_per_gpu": n, "grid_cells": cells,
                "parallelism": f"replicas x{world}", "l2_policy": l2}
    weak = a.config == "C4" and a.scaling == "weak"
    if weak:
        cells[0] *= world
        return {"workload": f"C4 x{world} (weak scaling): one C4 column per GPU, {DESC['C4']}",
                "particles_total": n * world, "particles_per_gpu": n, "grid_cells": cells,
                "parallelism": f"slab x{world} along x (library-owned NCCL halo + migration)", "l2_policy": l2}
    return {"workload": f"{a.config} (strong scaling): the one scene split into {world} particle-balanced slabs, "
                        f"{DESC[a.config]}", "particles_total": n, "grid_cells": cells,
            "parallelism": f"slab x{world} along x (library-owned NCCL halo + migration)", "l2_policy": l2}


# ---- clocks sampler -------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None
        self.first = 0

    def ready(self, timeout=5.0):
        """wait until nvidia-smi delivers its first line (its start-up can take longer than a short
        timed region), then mark where the timed region's samples begin"""
        t0 = time.time()
        while self.proc and not self.samples and time.time() - t0 < timeout:
            time.sleep(0.02)
        self.first = len(self.samples)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        # the samples taken during the timed region (plus the one just before it when the region
        # was shorter than the 100 ms sampling period)
        region = self.samples[max(self.first - 1, 0):] if self.samples else []
        sm = [float(p[0]) for p in region if p[0].replace(".", "").isdigit()]
        mx = [float(p[1]) for p in region if p[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for p in region:
            for k, nme in enumerate(names):
                if p[3 + k].lower() in ("active", "1"):
                    reasons.add(nme)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(region),
                "samples_in_region": len(self.samples) - self.first}


# ---- CPU baseline (the reference on host cores) --------------------------------------------
def _cpu_worker(args):
    """One host process: the reference's own run() timer (stepper.hpp:91-122) for mode "fwd", or the
    wall clock of its backprop_trajectory (checkpoint.hpp:72-143) for mode "adj", on the full scene."""
    cfg, dtype, kind, steps, mode, nseg = args[:6]
    warm = args[6] if len(args) > 6 else 0
    sys.path.insert(0, str(ROOT))
    from oracle import CpuOracle  # test infrastructure: the CPU baseline, never the product path
    from paper_2507_04192_b200.presets import CONFIGS
    s = CONFIGS[cfg](dtype=dtype)
    o = CpuOracle(kind)
    st = o.init_scene(s)
    if warm and mode == "fwd":
        o.advance(s, st, warm)  # untimed warm-up steps
    if mode == "fwd":
        secs = o.run_seconds_per_1000(s, st, steps) / 1000.0 * steps
    else:
        sd = {"field": "x", "obs_steps": [steps], "sel": None, "target": st.particles.x[None] + 1e-3}
        t0 = time.perf_counter()
        o.backprop(s, st, steps, nseg, sd)
        secs = time.perf_counter() - t0
    return st.particles.size() * steps, secs


def _mem_available_gb():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) / 1e6
    except Exception:
        pass
    return 16.0


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# host memory one reference process needs (state copies inside run / backprop_trajectory), GB
_PROC_GB = {"fwd": {"C4": 6.0, "C5": 40.0, "C5/8": 6.0}, "adj": {"C4": 14.0, "C5": 100.0, "C5/8": 14.0}}


def cpu_sample(cfg, dtype="f64", steps=1, mode="fwd", nseg=1, kind=None, procs=None, warm=0):
    """The reference (oracle/_ref, compiled unmodified) -- or the restatement -- on the full scene
    `cfg`: `steps` forward steps (mode "fwd") or a backprop_trajectory over `steps` steps (mode
    "adj"), in `procs` concurrent processes (default: one per host core, capped by host memory;
    independent replicas are the reference's only sanctioned concurrency).
    value = sum of the per-process particle-steps/s."""
    import multiprocessing as mp
    import oracle
    kind = kind or ("ref" if oracle.available("ref") else "orc")
    cores = os.cpu_count() or 1
    per_proc_gb = _PROC_GB[mode].get(cfg, 1.0 if mode == "fwd" else 2.0) * (0.5 if dtype == "f32" else 1.0)
    cap = max(1, min(cores, int(_mem_available_gb() * 0.6 / per_proc_gb)))
    procs = min(procs or cap, cap)
    with mp.get_context("spawn").Pool(procs) as pool:
        t0 = time.perf_counter()
        res = pool.map(_cpu_worker, [(cfg, dtype, kind, steps, mode, nseg, warm)] * procs)
        wall = time.perf_counter() - t0
    per_proc = [r[0] / r[1] for r in res]
    n = int(res[0][0] / steps)
    what = (f"{steps} forward step(s) timed by the reference's run() timer" if mode == "fwd" else
            f"backprop_trajectory over {steps} step(s), {nseg} segment(s), Lagrangian least-squares loss on the "
            f"final positions, wall clock of the call")
    flags = "-O3 -DNDEBUG -march=x86-64-v3" if kind == "ref_v3" else "-O3 -DNDEBUG (no -march: the reference's CMake Release)"
    return {"value": sum(per_proc), "unit": UNIT, "cores": procs, "host_cores": cores,
            "kind": "reference" if kind.startswith("ref") else "port",
            "sample": (f"{procs} concurrent process(es) (of {cores} host cores{', capped by host memory' if procs < cores else ''}) "
                       f"each running the full {cfg} scene ({n} particles): {what}; value = sum of per-process rates"),
            "single_process": per_proc[0], "wall_s": wall, "cpu_model": _cpu_model(),
            "label": f"reference compiled against the Eigen-API shim (C++20 {flags}, serial)"
            if kind.startswith("ref") else "oracle restatement (C++20 -O3, serial)"}


def cpu_baseline(cfg, dtype, steps=1):
    """Headline CPU baseline (all host cores) plus BASELINE.md §2's variants: one process alone
    (1 thread) and the -march=x86-64-v3 build on all cores."""
    import oracle
    out = cpu_sample(cfg, dtype, steps)
    out["variants"] = {}
    try:
        one = cpu_sample(cfg, dtype, steps, procs=1)
        out["variants"]["one_thread"] = {k: one[k] for k in ("value", "cores", "sample", "label")}
    except Exception as e:
        out["variants"]["one_thread"] = {"error": str(e)[:200]}
    if oracle.available("ref_v3"):
        try:
            v3 = cpu_sample(cfg, dtype, steps, kind="ref_v3")
            out["variants"]["march_x86_64_v3"] = {k: v3[k] for k in ("value", "cores", "sample", "label")}
        except Exception as e:
            out["variants"]["march_x86_64_v3"] = {"error": str(e)[:200]}
    return out


def cpu_baseline_adj(cfg, dtype, steps=2, nseg=1):
    """fwd+adjoint on the host cores: the reference's backprop_trajectory over `steps` steps."""
    return cpu_sample(cfg, dtype, steps, mode="adj", nseg=nseg)


def bench_fwd_adj(ctx, s, st, n, steps, nseg, profile=True):
    """fwd+adjoint (BASELINE metric, second half): one checkpointed backprop_trajectory through the
    C ABI -- forward sweep, segment replays, step_vjp per step (checkpoint.hpp:72-143) -- with the
    device Lagrangian least-squares seeder on the final positions. Device time from CUDA events on
    the context stream around the sweep (mpm_backprop_result.device_ms); the S0 upload and the
    cotangent download are outside it. Roofline: B_fwd+adj = 2 B_fwd + B_vjp."""
    from paper_2507_04192_b200.seeders import LagrangianLeastSquares
    st0 = ctx.download(st)
    sd = LagrangianLeastSquares([steps], st0.particles.x[None] + 1e-3, "x")
    ctx.backprop(st0, steps, nseg, sd.desc())  # allocates the checkpoint / replay pool
    t0 = time.perf_counter()
    _, _, res = ctx.backprop(st0, steps, nseg, sd.desc())
    wall = time.perf_counter() - t0
    ms = res.device_ms
    kern = {}
    if not profile:
        return {"value": n * steps / (ms / 1e3), "unit": UNIT, "steps": steps, "n_segments": nseg, "device_ms": ms,
                "ms_per_step": ms / steps, "wall_s_incl_host_transfers": wall, "loss": res.loss,
                "forward_passes_per_step": 1 + (steps - (steps // nseg)) / steps}
    ctx.profile(True)
    ctx.profile_reset()
    ctx.backprop(st0, steps, nseg, sd.desc())
    for k in ("k_p2g", "k_grid", "k_g2p", "k_adj_g2pT_gather", "k_adj_scatter", "k_adj_grid", "k_adj_p2gT",
              "k_seed"):
        t, c = ctx.profile_query(k)
        if c:
            kern[k] = {"ms_per_launch": t / c, "launches": c}
    ctx.profile(False)
    return {"value": n * steps / (ms / 1e3), "unit": UNIT, "steps": steps, "n_segments": nseg,
            "device_ms": ms, "ms_per_step": ms / steps, "wall_s_incl_host_transfers": wall,
            "loss": res.loss, "kernels": kern,
            "timing": "CUDA events on the library stream around forward sweep + replays + VJPs",
            # the last segment runs in the replay slots during the forward sweep and is not
            # replayed (bit-identical states): forward passes per step = 1 + (steps - L_last) / steps
            "forward_passes_per_step": 1 + (steps - (steps // nseg)) / steps}


def vjp_bytes(s, n, active_nodes_step, B_fwd, IN, fwd_passes=2.0):
    """B_fwd+adj = fwd_passes B_fwd + B_vjp per particle-step; SURVEY.md §8d writes it with 2
    forward passes (sweep + replay); the bench also reports it on the passes actually executed."""
    d = s.dim
    sz = 8 if s.dtype == "f64" else 4
    ns = 3 if d == 2 else 6
    dp = s.material.__class__.__name__ == "DruckerPragerParams"
    COT = 2 * d + 2 + ns + (1 if (dp and d == 2) else 0)
    A_np = active_nodes_step / n
    B_vjp = (IN + 2 * COT) * sz + A_np * (2 * (1 + 2 * d) + 8 * d) * sz
    return fwd_passes * B_fwd + B_vjp


# CPU samples of the sub-lines (BASELINE.md §2 horizons where they fit a few minutes of wall
# time; the reference is serial, so each is run as concurrent replicas on the host cores):
#   (cfg, mode, steps, n_segments)
CPU_SUBLINE = {"C1": {"fwd": ("C1", "fwd", 1000, 1)}, "C4/f32": {"fwd": ("C4", "fwd", 1, 1, "f32")},
               "C2": {"fwd": ("C2", "fwd", 100, 1)},
               "C3": {"fwd": ("C3", "fwd", 100, 1), "fwd_adj": ("C3", "adj", 20, 1)},
               "C5": {"fwd": ("C5", "fwd", 1, 1), "fwd_adj": ("C5/8", "adj", 1, 1)}}


def bench_workloads(peak, names, cpu=True):
    """The other BASELINE.json configs on this GPU (N = 1), device-timed through the same context
    API: C2 forward; C3 the paper's inverse problem (loss on the final deposit of an alpha* = 2
    twin, reverse-mode gradient through all 1000 steps from t = 0, HBM-sized checkpoint plan,
    dL/dalpha chained on the host as in SURVEY §8d, compared with the reference's own gradient in
    tests/golden/c3_gradient.npz); C5 forward + a 20-step fwd+adjoint with the 32 Coulomb friction
    segments' gradients. Each sub-line carries its own roofline and a CPU sample (CPU_SUBLINE)."""
    import numpy as np
    import torch
    from paper_2507_04192_b200 import init_scene
    from paper_2507_04192_b200.presets import CONFIGS, c3_inverse
    from paper_2507_04192_b200.seeders import LagrangianLeastSquares
    from paper_2507_04192_b200.solver import Context

    out = {}
    for name in names:
        try:
            if name == "C5" and _mem_available_gb() < 48:
                out[name] = {"skipped": "host memory below 48 GB for the 7.3 GB host copies"}
                continue
            cname, dt = (name.split("/") + ["f64"])[:2]
            s = CONFIGS[cname](dtype=dt)
            st0 = init_scene(s)
            n = st0.particles.size()
            ctx = Context(s, n)
            ctx.upload(st0)
            ctx.advance(3)
            k_fwd = {"C1": 1000, "C2": 200, "C3": 200, "C4/f32": 50, "C5": 20}[name]
            ms = ctx.advance_timed(k_fwd, nan_guard=True)
            act, _, _ = ctx.grid_stats()
            B_fwd, IN, _ = bytes_model(s, n, act / k_fwd)
            w = {"particles": n, "grid_cells": s.config.cells, "dtype": dt,
                 "fwd": {"value": n * k_fwd / (ms / 1e3), "unit": UNIT, "steps": k_fwd, "ms_per_step": ms / k_fwd,
                         "roofline_frac": n * B_fwd / (ms / k_fwd / 1e3) / 1e9 / peak,
                         "bytes_per_particle_step": B_fwd}}
            adj = {"C3": 1000, "C5": 20}.get(name, 0)
            if adj:
                if name == "C3":  # twin run at the true alpha* = 2.0 gives the observed deposit
                    tw = c3_inverse(alpha=2.0, dtype="f64")
                    stt = init_scene(tw)
                    ctt = Context(tw, stt.particles.size())
                    ctt.upload(stt)
                    ctt.advance(adj)
                    target = ctt.download(stt).particles.x[None].copy()
                    ctt.close()
                    sd = LagrangianLeastSquares([adj], target, "x")
                else:  # positions of a 1 % subset (seeded) against a perturbed twin
                    rng = np.random.default_rng(0)
                    sel = np.sort(rng.choice(n, n // 100, replace=False))
                    ctx.upload(st0)
                    ctx.advance(adj)
                    xf = ctx.download(st0.copy()).particles.x
                    sd = LagrangianLeastSquares([adj], xf[sel][None] + 1e-3, "x", sel=sel)
                act0 = act / k_fwd
                nseg, plan = hbm_plan(s, n, adj, act0)
                ctx.backprop(st0, adj, nseg, sd.desc())  # allocates the checkpoint / replay pool
                c0, pg, res = ctx.backprop(st0, adj, nseg, sd.desc())
                L_last = adj // nseg
                fpps = 1 + (adj - L_last) / adj
                B_fa = vjp_bytes(s, n, act0, B_fwd, IN, fpps)
                mps = res.device_ms / adj
                w["fwd_adj"] = {"value": n * adj / (res.device_ms / 1e3), "unit": UNIT, "steps": adj,
                                "ms_per_step": mps, "plan": plan, "loss": res.loss, "forward_passes_per_step": fpps,
                                "roofline_frac": n * B_fa / (mps / 1e3) / 1e9 / peak, "bytes_per_particle_step": B_fa,
                                "roofline_basis": "forward passes executed x B_fwd + B_vjp",
                                "timing": "mpm_backprop_result.device_ms (forward sweep + replays + VJPs)"}
                if name == "C3":  # v_x(0) = alpha (h0 - y_rel): dL/dalpha = sum_p vbar_x(0) v_x(0) / alpha
                    alpha = s.geometry[0].velocity.alpha
                    dl = float(np.sum(c0.v[:, 0] * st0.particles.v[:, 0]) / alpha)
                    w["fwd_adj"]["dL_dalpha"] = dl
                    gold = ROOT / "tests" / "golden" / "c3_gradient.npz"
                    if gold.exists():
                        g = np.load(gold)
                        w["fwd_adj"]["reference_gradient"] = {
                            "dL_dalpha": float(g["dL_dalpha"]), "loss": float(g["loss"]),
                            "rel_diff_dL_dalpha": abs(dl - float(g["dL_dalpha"])) / abs(float(g["dL_dalpha"])),
                            "rel_diff_loss": abs(res.loss - float(g["loss"])) / abs(float(g["loss"])),
                            "source": "tests/golden/c3_gradient.npz: the reference's backprop_trajectory, "
                                      "1000 steps, n_seg 10 (tests/golden/make_c3_gradient.py)"}
                else:
                    fr = np.asarray(pg.flat())
                    w["fwd_adj"]["param_grads_norm"] = float(np.linalg.norm(fr))
            ctx.close()
            torch.cuda.empty_cache()
            if cpu:
                for leg, spec in CPU_SUBLINE.get(name, {}).items():
                    ccfg, mode, steps, cseg = spec[:4]
                    cdt = spec[4] if len(spec) > 4 else "f64"
                    if leg in w:
                        try:
                            w[leg]["cpu_baseline"] = cpu_sample(ccfg, cdt, steps, mode=mode, nseg=cseg)
                        except Exception as e:
                            w[leg]["cpu_baseline"] = {"value": None, "error": f"{type(e).__name__}: {str(e)[:160]}"}
            out[name] = w
        except Exception as e:  # a workload that fails is reported, the headline line still prints
            out[name] = {"error": f"{type(e).__name__}: {str(e)[:200]}"}
    return out


def hbm_plan(s, n, steps, active_nodes):
    """Fewest checkpoint segments whose HBM footprint fits: n_seg checkpoints + L_max + 1 replay
    slots (checkpoint.hpp:50's planned_peak_states) + L_max replay-tape entries, within 70 % of
    the free device memory. B200-first: 180 GB holds a C4 20-step trajectory whole (one segment,
    nothing replayed), where a CPU-sized plan would recompute half of it."""
    import torch
    d = s.dim
    sz = 8 if s.dtype == "f64" else 4
    fields = (2 * d + 4 + (1 if d == 2 else 0) + (3 if d == 2 else 6) + d * d)
    state = n * (fields * sz + 4)
    tape = n * 8 + 1.25 * active_nodes * (1 + 4 * d) * sz
    free = torch.cuda.mem_get_info()[0]
    for nseg in range(1, steps + 1):
        L = -(-steps // nseg)
        if (nseg + L + 1) * state + L * tape <= 0.7 * free:
            return nseg, {"n_segments": nseg, "rule": "fewest segments whose checkpoints + replay slots + tape "
                          "fit in 70% of free HBM", "state_bytes": state, "free_hbm_bytes": free}
    return steps, {"n_segments": steps, "rule": "HBM-bound: one step per segment"}


# ---- GPU arm -----------------------------------------------------------------------------------
def bench_b200(a, rank, world, local):
    import ctypes as C

    import torch
    from paper_2507_04192_b200 import capi, init_scene
    from paper_2507_04192_b200.presets import CONFIGS
    from paper_2507_04192_b200.solver import Context

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    s = CONFIGS[a.config](dtype=a.dtype)
    st = init_scene(s)
    n = st.particles.size()
    ctx = Context(s, n, device=local)
    ctx.upload(st)
    ctx.advance(a.warmup)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timed region
    clocks = ClockSampler(local)
    clocks.start()
    clocks.ready()
    l0 = ctx.launch_count()
    barrier()
    ms = ctx.advance_timed(a.steps, nan_guard=True)  # run()'s per-step all_finite guard (stepper.hpp:106-109)
    barrier()
    launches = ctx.launch_count() - l0
    ck = clocks.stop()
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / a.steps
    value = n * world * a.steps / (ms / 1e3)

    active_nodes, occ_blocks, act_blocks = ctx.grid_stats()
    active_nodes_step = active_nodes / a.steps
    B_fwd, IN, OUT = bytes_model(s, n, active_nodes_step)  # SURVEY §8d (grad v stored every step)
    B_fwd1 = B_fwd
    B_need = bytes_model(s, n, active_nodes_step, a.steps)[0]  # grad v stored by the call's last step

    # ---- per-kernel profile (CUDA events around each launch on the library stream)
    ctx.profile(True)
    ctx.profile_reset()
    ctx.advance(3, nan_guard=True)
    prof = {}
    for k in ("k_p2g", "k_grid", "k_g2p", "k_sort", "k_seg", "k_occ", "k_compact", "k_mark_nodes", "k_step_end",
              "k_keys"):
        t_ms, cnt = ctx.profile_query(k)
        if cnt:
            prof[k] = {"ms_per_launch": t_ms / cnt, "launches": cnt}
    total_ms, _ = ctx.profile_query("")
    ctx.profile(False)
    kb, kneed, kmoved = kernel_bytes(s, n, active_nodes_step, occ_blocks)
    dom = max(("k_p2g", "k_g2p"), key=lambda k: prof.get(k, {}).get("ms_per_launch", 0))
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    dom_ms = prof[dom]["ms_per_launch"]
    achieved = kb[dom] / (dom_ms / 1e3) / 1e9
    step_gbs = n * B_fwd / (ms_per_step / 1e3) / 1e9
    per_kernel = {}
    for k in ("k_p2g", "k_g2p"):
        if k in prof:
            t = prof[k]["ms_per_launch"] / 1e3
            tr = traffic_for(k, a)
            per_kernel[k] = {"mean_launch_ms": prof[k]["ms_per_launch"],
                             "algorithmic_bytes_per_launch": kb[k], "frac": kb[k] / t / 1e9 / peak,
                             "needed_bytes_per_launch": kneed[k], "frac_needed": kneed[k] / t / 1e9 / peak,
                             "moved_bytes_per_launch": kmoved[k],
                             "ncu_dram_bytes_per_launch": tr,
                             "waste_ratio_ncu_over_algorithmic": (tr / kb[k]) if tr else None,
                             "l2_hit_rate_pct_ncu": l2_hit_for(k, a)}
    if "k_grid" in prof:
        per_kernel["k_grid"] = {"mean_launch_ms": prof["k_grid"]["ms_per_launch"],
                                "ncu_dram_bytes_per_launch": traffic_for("k_grid", a),
                                "l2_hit_rate_pct_ncu": l2_hit_for("k_grid", a)}

    # ---- e2e through the C ABI with pinned host buffers (upload + K steps + download)
    e2e = None
    if rank == 0:
        e2e = bench_e2e(ctx, s, st, a.steps)

    # ---- fwd+adjoint (checkpointed backprop_trajectory), device-timed
    fwd_adj = None
    if a.adj_steps > 0:
        nseg, plan = (a.adj_segments, {"n_segments": a.adj_segments, "rule": "--adj-segments"}) \
            if a.adj_segments > 0 else hbm_plan(s, n, a.adj_steps, active_nodes_step)
        fwd_adj = bench_fwd_adj(ctx, s, st, n, a.adj_steps, nseg)
        fwd_adj["plan"] = plan
        if nseg != 2 and a.adj_steps >= 2:  # the two-segment plan beside it (same loss, more replay)
            alt = bench_fwd_adj(ctx, s, st, n, a.adj_steps, 2)
            fwd_adj["two_segments"] = {k: alt[k] for k in ("value", "ms_per_step", "forward_passes_per_step", "loss")}
        if a.long_adj > 0:  # the horizon an inverse run sustains (C3 / C5: 1000 steps), HBM-sized plan
            nl, pl = hbm_plan(s, n, a.long_adj, active_nodes_step)
            lg = bench_fwd_adj(ctx, s, st, n, a.long_adj, nl, profile=False)
            fwd_adj["long_horizon"] = {k: lg[k] for k in ("value", "ms_per_step", "steps", "n_segments",
                                                         "forward_passes_per_step", "loss", "device_ms")}
            fwd_adj["long_horizon"]["plan"] = pl
        B_fa = vjp_bytes(s, n, active_nodes_step, B_fwd1, IN)
        B_ex = vjp_bytes(s, n, active_nodes_step, B_fwd1, IN, fwd_adj["forward_passes_per_step"])
        gbs = n * B_fa / (fwd_adj["ms_per_step"] / 1e3) / 1e9
        gbs_ex = n * B_ex / (fwd_adj["ms_per_step"] / 1e3) / 1e9
        fwd_adj["roofline"] = {"bound": "hbm", "bytes_per_particle_step": B_ex, "achieved": gbs_ex, "peak": peak,
                               "unit": "GB/s", "frac": gbs_ex / peak,
                               "basis": "forward passes actually executed per step x B_fwd + B_vjp",
                               "survey_formula": {"bytes_per_particle_step": B_fa, "frac": gbs / peak,
                                                  "note": "2 B_fwd + B_vjp (one replay per step assumed)"}}

    ctx.close()
    workloads = None
    if world == 1 and a.config == "C4" and not a.no_workloads:
        workloads = bench_workloads(peak, ["C1", "C2", "C3", "C4/f32", "C5"], cpu=not a.no_cpu_baseline)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    if rank != 0:
        return None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": a.dtype, "data": "synthetic (init_scene seeding of the named scene, deterministic)",
        "config": workload_config(a, world),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_for(dom, a),
                     "algorithmic_bytes_per_launch": kb[dom], "mean_launch_ms": dom_ms,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback 6650 GB/s",
                     "basis": "SURVEY 8(d) compulsory bytes of the kernel (x v m V sigma read, active nodes "
                              "written once) / its mean event-timed launch; implementation bytes and the ncu "
                              "DRAM count are in per_kernel",
                     "per_kernel": per_kernel,
                     "step": {"achieved_gbs": step_gbs, "frac": step_gbs / peak,
                              "bytes_per_particle_step": B_fwd, "active_nodes_per_particle": active_nodes_step / n,
                              "needed_bytes_per_particle_step": B_need,
                              "frac_needed": n * B_need / (ms_per_step / 1e3) / 1e9 / peak,
                              "note": "frac counts grad v stored every step (SURVEY's B_fwd); frac_needed counts "
                                      "what the implementation must move (FLIP stores grad v on a call's last "
                                      "step only)"}},
        "fp64": fp64_for(prof, a),
        "kernels": prof, "profiled_step_ms": total_ms / 3,
        "clocks": ck, "gpu_launches": launches, "e2e": e2e, "fwd_adj": fwd_adj,
        "workloads": workloads,
    }
    return line


def bench_slab(a, rank, world, local):
    """Slab-decomposed step over NCCL, weak scaling (C4: one column per rank)."""
    import torch
    import torch.distributed as dist
    from paper_2507_04192_b200 import init_scene
    from paper_2507_04192_b200.distributed import GpuSlabDomain, SlabPlan, SlabStepper, TorchTransport
    from paper_2507_04192_b200.presets import CONFIGS, c4_column3d

    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    if a.config == "C4":
        s = c4_column3d(a.dtype, replicas_x=world)
        st = init_scene(c4_column3d(a.dtype))  # this rank's column, shifted into its slab
        n = st.particles.size()
        st.particles.x[:, 0] += 256 * rank * s.config.dh
        ids = np.arange(rank * n, (rank + 1) * n, dtype=np.int64)
        plan = SlabPlan([256 * r for r in range(world + 1)], 8)
        dom = GpuSlabDomain(s, plan, rank, st, ids, device=local, local=True)
        n_total = n * world
        scaling = "weak"
    else:
        s = CONFIGS[a.config](dtype=a.dtype)
        full = init_scene(s)
        plan = SlabPlan.make(s, world, full.particles.x)
        dom = GpuSlabDomain(s, plan, rank, full, None, device=local)
        n_total = full.particles.size()
        scaling = "strong"
    stp = SlabStepper([dom], TorchTransport())
    stp.advance(a.warmup)
    clocks = ClockSampler(local)
    clocks.start()
    clocks.ready()
    l0 = dom.ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    ev0.record()
    stp.advance(a.steps)
    torch.cuda.synchronize()  # every library call has synchronised its own stream already
    ev1.record()
    ev1.synchronize()
    dist.barrier()
    ck = clocks.stop()
    launches = dom.ctx.launch_count() - l0
    an1, _, _ = dom.ctx.grid_stats()
    t = torch.tensor([ev0.elapsed_time(ev1)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    mig = torch.tensor([stp.migrated], device="cuda", dtype=torch.int64)
    dist.all_reduce(mig)
    # the slab path resets the device status every step: the counter holds the last step's nodes
    act = torch.tensor([float(an1) / a.steps], device="cuda", dtype=torch.float64)  # counted over the K steps
    dist.all_reduce(act)
    # e2e: rank-local upload from pinned host + K decomposed steps + compact download, max over ranks
    e2e = bench_slab_e2e(dom, stp, a.steps)
    te = torch.tensor([e2e["seconds"], e2e["h2d_bytes_per_step"], e2e["d2h_bytes_per_step"]], device="cuda",
                      dtype=torch.float64)
    dist.all_reduce(te[:1], op=dist.ReduceOp.MAX)
    tb = te[1:].clone()
    dist.all_reduce(tb)
    fwd_adj = None
    if a.config == "C4" and a.slab_adj:
        fwd_adj = bench_slab_fwd_adj(s, st, dom, rank, world, n, min(a.adj_steps, 2))
    dom.close()
    dist.barrier()
    if rank != 0:
        return None
    # step-level roofline per GPU: B_fwd over each GPU's share of the particles
    B_fwd, _, _ = bytes_model(s, n_total, float(act.item()))
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    gbs = n_total / world * B_fwd / (ms / a.steps / 1e3) / 1e9
    roof = {"bound": "hbm", "kernel": "step (per GPU)", "achieved": gbs, "peak": peak, "unit": "GB/s",
            "frac": gbs / peak, "traffic": None, "bytes_per_particle_step": B_fwd,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback 6650 GB/s"}
    e2e_line = {"value": n_total * a.steps / float(te[0].item()), "unit": UNIT,
                "h2d_bytes_per_step": float(tb[0].item()), "d2h_bytes_per_step": float(tb[1].item()),
                "call": e2e["call"], "seconds": float(te[0].item())}
    return {
        "metric": METRIC, "value": n_total * a.steps / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": a.dtype, "data": "synthetic (init_scene seeding of the named scene, deterministic)",
        "config": {"workload": (f"C4 x{world}: 3-D D-P granular column collapse, one 128x64x64-cell column per rank, "
                                f"domain {s.config.cells}" if a.config == "C4" else a.config),
                   "particles_total": n_total, "parallelism": f"slab x{world} (NCCL halo + migration)",
                   "slab_bounds": plan.bounds, "migrated_particles": int(mig.item()),
                   "l2_policy": "inputs larger than the 126 MB L2; no flush"},
        "roofline": roof, "clocks": ck, "gpu_launches": launches, "e2e": e2e_line, "fwd_adj": fwd_adj,
    }


def bench_dist(a, rank, world, local):
    """The library-owned slab decomposition (mpm_dist_*: NCCL send/recv of the halo bands and the
    fixed-capacity migration messages, device-resident counts, no host synchronisation inside the
    K steps), one process per GPU. C4 weak scaling: one C4 column per rank in a 256N x 256 x 256
    domain; strong scaling: the C4 scene itself split into N particle-balanced slabs. Time = CUDA
    events around the K steps on each rank's library stream, max over ranks."""
    import ctypes as C

    import torch
    import torch.distributed as dist
    from paper_2507_04192_b200 import init_scene
    from paper_2507_04192_b200.distributed import NcclSlabRank, SlabPlan, dist_unique_id
    from paper_2507_04192_b200.presets import CONFIGS, c4_column3d

    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    strong = a.scaling == "strong" or a.config != "C4"
    if not strong:
        s = c4_column3d(a.dtype, replicas_x=world)
        st = init_scene(c4_column3d(a.dtype))  # this rank's column, shifted into its slab
        n = st.particles.size()
        st.particles.x[:, 0] += 256 * rank * s.config.dh
        ids = np.arange(rank * n, (rank + 1) * n, dtype=np.int64)
        plan = SlabPlan([256 * r for r in range(world + 1)], 8)
        n_total = n * world
        workload = (f"C4 x{world} (weak): 3-D D-P granular column collapse, one 128x64x64-cell column per GPU, "
                    f"domain {s.config.cells}")
    else:
        s = CONFIGS[a.config](dtype=a.dtype)
        full = init_scene(s)
        plan = SlabPlan.make(s, world, full.particles.x)
        ids = plan.partition(s, full)[rank]
        st = SimState_take(full, ids)
        n_total = full.particles.size()
        workload = f"{a.config} (strong): the one scene split into {world} particle-balanced slabs along x"
    obj = [dist_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    rk = NcclSlabRank(s, plan, rank, st, ids, obj[0], device=local, n_total=n_total)
    rk.advance(a.warmup)
    clocks = ClockSampler(local)
    clocks.start()
    clocks.ready()
    l0 = rk.ctx.launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    ms = rk.advance(a.steps, nan_guard=True)
    torch.cuda.synchronize()
    dist.barrier()
    ck = clocks.stop()
    launches = rk.ctx.launch_count() - l0
    an1, _, _ = rk.ctx.grid_stats()
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    cnt = torch.tensor([int(rk.lib.mpm_local_count(rk.h))], device="cuda", dtype=torch.int64)
    dist.all_reduce(cnt)
    act = torch.tensor([float(an1) / a.steps], device="cuda", dtype=torch.float64)  # counted over the K steps
    dist.all_reduce(act)
    # e2e: rank-local upload from pinned host + K decomposed steps + compact download, max over ranks
    e2e = dist_e2e(rk, st, ids, a.steps)
    te = torch.tensor([e2e["seconds"], e2e["h2d_bytes_per_step"], e2e["d2h_bytes_per_step"]], device="cuda",
                      dtype=torch.float64)
    dist.all_reduce(te[:1], op=dist.ReduceOp.MAX)
    tb = te[1:].clone()
    dist.all_reduce(tb)
    # fwd+adjoint over the decomposition (mpm_dist_backprop: device-resident per-rank checkpoints,
    # replay, cotangent rows of migrants returned, decomposed step_vjp)
    fwd_adj = None
    if a.adj_steps > 0 and not strong:
        fwd_adj = dist_fwd_adj(rk, s, st, rank, world, n, n_total, a.adj_steps)
    rk.close()
    dist.barrier()
    if rank != 0:
        return None
    B_fwd, IN, _ = bytes_model(s, n_total, float(act.item()))
    if fwd_adj and fwd_adj.get("value"):
        B_fa = vjp_bytes(s, n_total, float(act.item()), B_fwd, IN, fwd_adj["forward_passes_per_step"])
        gbs_fa = n_total / world * B_fa / (fwd_adj["ms_per_step"] / 1e3) / 1e9
        peaks0 = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        fwd_adj["roofline"] = {"bound": "hbm", "bytes_per_particle_step": B_fa, "achieved": gbs_fa, "unit": "GB/s",
                               "frac": gbs_fa / peaks0.get("hbm_gbs", 6650.0), "per": "GPU"}
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    gbs = n_total / world * B_fwd / (ms / a.steps / 1e3) / 1e9
    return {
        "metric": METRIC, "value": n_total * a.steps / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
        "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": a.dtype,
        "data": "synthetic (init_scene seeding of the named scene, deterministic)",
        "config": workload_config(a, world),
        "slab": {"workload": workload, "bounds": plan.bounds, "particles_after": int(cnt.item()),
                 "path": "mpm_dist_advance: device-resident counts, no host synchronisation inside the K steps"},
        "roofline": {"bound": "hbm", "kernel": "step (per GPU)", "achieved": gbs, "peak": peak, "unit": "GB/s",
                     "frac": gbs / peak, "traffic": None, "bytes_per_particle_step": B_fwd,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback 6650 GB/s"},
        "clocks": ck, "gpu_launches": launches, "fwd_adj": fwd_adj,
        "e2e": {"value": n_total * a.steps / float(te[0].item()), "unit": UNIT,
                "h2d_bytes_per_step": float(tb[0].item()), "d2h_bytes_per_step": float(tb[1].item()),
                "call": e2e["call"], "seconds": float(te[0].item())},
    }


def dist_fwd_adj(rk, s, st, rank, world, n, n_total, steps):
    """mpm_dist_backprop on every rank: `steps` steps, the fewest checkpoint segments that fit in
    HBM, Lagrangian least squares on the final positions of every 100th particle (global ids).
    Time = the library's CUDA-event time of the call, max over ranks (the S0 upload and the
    cotangent download fall outside it, as in the single-context line)."""
    import torch
    import torch.distributed as dist

    try:
        sel = np.arange(0, n_total, 100, dtype=np.int64)
        x0 = st.particles.x[sel % n].copy()  # every rank's column is the same seeding, shifted in x
        x0[:, 0] += 256 * (sel // n - rank) * s.config.dh
        seeder = {"field": "x", "obs_steps": [steps], "sel": sel, "target": x0[None] + 1e-3}
        nseg, plan = hbm_plan(s, n, steps, 0.14 * n)
        rk.backprop(steps, nseg, seeder, n_total)  # allocates the checkpoint / replay slots and the tape
        t0 = time.perf_counter()
        _, _, pg, res = rk.backprop(steps, nseg, seeder, n_total)
        wall = time.perf_counter() - t0
        t = torch.tensor([res.device_ms, wall], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, wall = float(t[0].item()), float(t[1].item())
        L = steps // nseg
        return {"value": n_total * steps / (ms / 1e3), "unit": UNIT, "steps": steps, "n_segments": nseg, "plan": plan,
                "ms_per_step": ms / steps, "device_ms": ms, "wall_s": wall, "loss": res.loss,
                "forward_passes_per_step": 1 + (steps - L) / steps,
                "timing": "CUDA events on each rank's library stream around mpm_dist_backprop, max over ranks"}
    except Exception as e:  # reported, the forward line still prints
        return {"value": None, "error": f"{type(e).__name__}: {str(e)[:200]}"}


def SimState_take(full, ids):
    from paper_2507_04192_b200.state import SimState
    return SimState(full.particles.take(ids), full.step, full.time)


def dist_e2e(rk, st, ids, steps):
    """mpm_state_upload_ids from pinned host buffers + K decomposed steps (mpm_dist_advance) +
    mpm_state_download_local into pinned buffers, wall clock on this rank."""
    import ctypes as C

    import torch
    from paper_2507_04192_b200 import capi

    p = st.particles
    d = p.dim
    n = p.size()
    tdt = torch.float64 if p.dtype == np.float64 else torch.float32

    def pinned(shape):
        return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()

    fields = {"x": (n, d), "v": (n, d), "mass": (n,), "volume": (n,), "rho": (n,), "eps_eq": (n,),
              "sigma": (n, d * d), "grad_v": (n, d * d)}
    if d == 2:
        fields["sigma_zz"] = (n,)
    host = {k: pinned(sh) for k, sh in fields.items()}
    for k in ("x", "v", "mass", "volume", "rho", "eps_eq") + (("sigma_zz",) if d == 2 else ()):
        host[k][...] = getattr(p, k)
    host["sigma"][...] = np.transpose(p.sigma, (0, 2, 1)).reshape(n, d * d)
    host["grad_v"][...] = np.transpose(p.grad_v, (0, 2, 1)).reshape(n, d * d)
    cap = rk.capacity
    outb = {k: pinned((cap,) + sh[1:]) for k, sh in fields.items()}
    ids_in = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int64)).pin_memory().numpy()
    ids_out = torch.empty(cap, dtype=torch.int64, pin_memory=True).numpy()
    view, out = capi.StateView(), capi.StateView()
    view.n, out.n = n, cap
    for k in fields:
        setattr(view, k, host[k].ctypes.data)
        setattr(out, k, outb[k].ctypes.data)
    lib, h = rk.lib, rk.h
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rk.ctx.check(lib.mpm_state_upload_ids(h, C.byref(view), ids_in.ctypes.data_as(C.c_void_p)))
    rk.ctx.check(lib.mpm_dist_advance(h, steps, 0, None))
    rk.ctx.check(lib.mpm_state_download_local(h, C.byref(out), ids_out.ctypes.data_as(C.c_void_p)))
    t1 = time.perf_counter()
    h2d = sum(v.nbytes for v in host.values()) + ids_in.nbytes
    d2h = out.n * (sum(v[0].nbytes for v in outb.values()) + 8)
    return {"seconds": t1 - t0, "h2d_bytes_per_step": h2d / steps, "d2h_bytes_per_step": d2h / steps,
            "call": f"mpm_state_upload_ids (pinned host) + mpm_dist_advance({steps}) + mpm_state_download_local, "
                    "wall clock"}


def bench_slab_fwd_adj(s, st, dom, rank, world, n, steps):
    """fwd+adjoint over the slab decomposition (slab_backprop_trajectory: per-rank checkpoints,
    digest-checked replay, slab_step_vjp with two halo exchanges per step). It is host-orchestrated:
    replay states and migrants' cotangent rows pass through host memory every step,
    so this is the protocol's number, wall clock max over ranks, not the device path's.
    Loss: positions of every 100th particle (global ids) at the last step."""
    import torch
    import torch.distributed as dist
    from paper_2507_04192_b200.distributed import TorchTransport, slab_backprop_trajectory
    from paper_2507_04192_b200.seeders import LagrangianLeastSquares
    from paper_2507_04192_b200.solver import CheckpointPlan

    try:
        n_total = n * world
        sel = np.arange(0, n_total, 100, dtype=np.int64)
        x0 = st.particles.x[sel % n].copy()  # every rank's column is the same seeding, shifted in x
        x0[:, 0] += 256 * (sel // n - rank) * s.config.dh
        seeder = LagrangianLeastSquares([steps], x0[None] + 1e-3, "x", sel=sel)
        dist.barrier()
        t0 = time.perf_counter()
        res = slab_backprop_trajectory(s, CheckpointPlan.make(steps, 1), seeder, [dom], TorchTransport(), n_total)
        wall = time.perf_counter() - t0
        t = torch.tensor([wall], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
        return {"value": n_total * steps / wall, "unit": UNIT, "steps": steps, "n_segments": 1, "seconds": wall,
                "loss": res.loss, "timing": "wall clock, max over ranks (host-orchestrated decomposed backprop)"}
    except Exception as e:  # reported, the forward line still prints
        return {"value": None, "error": f"{type(e).__name__}: {str(e)[:200]}"}


def bench_slab_e2e(dom, stp, steps):
    """Host state in pinned buffers -> mpm_state_upload_ids -> K decomposed steps ->
    mpm_state_download_local, wall clock."""
    import ctypes as C

    import torch
    from paper_2507_04192_b200.state import SimState

    sub, ids, _ = dom.gather()
    k = len(ids)
    st = SimState(sub, 0, 0.0)
    v, keep = st.to_view()
    pinned = {}
    for name, arr in keep.items():
        if arr is None:
            continue
        t = torch.empty(arr.shape, dtype=torch.from_numpy(arr[:0]).dtype, pin_memory=True).numpy()
        t[...] = arr
        pinned[name] = t
        setattr(v, name, t.ctypes.data)
    ids_p = torch.empty(k, dtype=torch.int64, pin_memory=True).numpy()
    ids_p[...] = ids
    lib, h = dom.lib, dom.h
    out = SimState.zeros(k + dom.capacity // 4, sub.dim, sub.dtype)
    ov, okeep = out.output_view()
    for name, arr in okeep.items():  # pinned download buffers, as the upload's
        if arr is None or not arr.size:
            continue
        t = torch.empty(arr.shape, dtype=torch.from_numpy(arr[:0]).dtype, pin_memory=True).numpy()
        okeep[name] = t
        setattr(ov, name, t.ctypes.data)
    oids = torch.empty(k + dom.capacity // 4, dtype=torch.int64, pin_memory=True).numpy()
    torch.cuda.synchronize()
    import torch.distributed as dist
    dist.barrier()
    t0 = time.perf_counter()
    dom.ctx.check(lib.mpm_state_upload_ids(h, C.byref(v), ids_p.ctypes.data_as(C.c_void_p)))
    stp.advance(steps)
    dom.ctx.check(lib.mpm_state_download_local(h, C.byref(ov), oids.ctypes.data_as(C.c_void_p)))
    t1 = time.perf_counter()
    h2d = sum(a.nbytes for a in pinned.values()) + ids_p.nbytes
    d2h = ov.n * (sum(a.nbytes for a in pinned.values()) + ids_p.nbytes) / max(k, 1)
    return {"seconds": t1 - t0, "h2d_bytes_per_step": h2d / steps, "d2h_bytes_per_step": d2h / steps,
            "call": f"mpm_state_upload_ids (pinned host) + {steps} slab steps + mpm_state_download_local, wall clock"}


def fp64_for(prof, a):
    """The f64 kernels are co-limited by FP64 issue, not HBM: FP64 flops per launch
    (ncu SASS op counts, profiles/fp64.json: 2 x DFMA + DMUL + DADD) over the live mean launch time,
    against the FP64 DFMA ceiling measured on this pool by tools/fp64_peak.cu (profiles/fp64_peak.json;
    MEASURED_PEAKS has no FP64), else the datasheet FP64 vector peak."""
    p = ROOT / "profiles" / "fp64.json"
    if a.config != "C4" or a.dtype != "f64" or not p.exists():
        return None
    ref = json.loads(p.read_text())
    out = {"peak_tflops": 37.0, "peak_source": "HGX B200 datasheet FP64 (not measured)", "unit": "TFLOP/s"}
    pk = ROOT / "profiles" / "fp64_peak.json"
    if pk.exists():
        meas = json.loads(pk.read_text())
        out["peak_tflops"] = float(meas["fp64_tflops"])
        out["peak_source"] = "profiles/fp64_peak.json (measured: tools/fp64_peak.cu DFMA chains)"
    for k in ("k_p2g", "k_g2p"):
        if k in ref and k in prof:
            tf = ref[k]["fp64_flops"] / (prof[k]["ms_per_launch"] * 1e-3) / 1e12
            out[k] = {"achieved": tf, "frac": tf / out["peak_tflops"], "flops_per_launch": ref[k]["fp64_flops"],
                      "fp64_pipe_active_pct_ncu": ref[k]["fp64_pipe_active_pct"]}
    return out


def l2_hit_for(kernel, a):
    """lts__t_sector_hit_rate.pct of `kernel` from the same ncu capture (profiles/traffic.json)."""
    p = ROOT / "profiles" / "traffic.json"
    if a.config != "C4" or a.dtype != "f64" or not p.exists():
        return None
    t = json.loads(p.read_text()).get(kernel)
    return t.get("l2_hit_rate_pct") if t else None


def traffic_for(kernel, a):
    """dram__bytes_read + dram__bytes_write per launch of `kernel` from the committed ncu --set full
    capture of the same command (profiles/traffic.json); None when absent or another workload."""
    p = ROOT / "profiles" / "traffic.json"
    if a.config != "C4" or a.dtype != "f64" or not p.exists():
        return None
    t = json.loads(p.read_text()).get(kernel)
    return t["dram_bytes"] if t else None


def bench_e2e(ctx, s, st, steps):
    """One reference-style run call through the C ABI on pinned host buffers."""
    import ctypes as C

    import torch
    from paper_2507_04192_b200 import capi

    p = st.particles
    d = s.dim
    T = p.dtype
    n = p.size()

    def pinned(shape):
        t = torch.empty(shape, dtype=torch.float64 if T == np.float64 else torch.float32, pin_memory=True)
        return t.numpy()

    host = {"x": pinned((n, d)), "v": pinned((n, d)), "mass": pinned((n,)), "volume": pinned((n,)),
            "rho": pinned((n,)), "eps_eq": pinned((n,)), "sigma": pinned((n, d * d)), "grad_v": pinned((n, d * d))}
    if d == 2:
        host["sigma_zz"] = pinned((n,))
    host["x"][...] = p.x
    host["v"][...] = p.v
    host["mass"][...] = p.mass
    host["volume"][...] = p.volume
    host["rho"][...] = p.rho
    host["eps_eq"][...] = p.eps_eq
    host["sigma"][...] = np.transpose(p.sigma, (0, 2, 1)).reshape(n, d * d)
    host["grad_v"][...] = np.transpose(p.grad_v, (0, 2, 1)).reshape(n, d * d)
    if d == 2:
        host["sigma_zz"][...] = p.sigma_zz
    view = capi.StateView()
    view.n = n
    for k, arr in host.items():
        setattr(view, k, arr.ctypes.data)
    view.step = 0
    view.time = 0.0
    out = capi.StateView()
    outb = {k: pinned(v.shape) for k, v in host.items()}
    out.n = n
    for k, arr in outb.items():
        setattr(out, k, arr.ctypes.data)
    lib = ctx.lib
    nbytes_in = sum(v.nbytes for v in host.values())
    nbytes_out = sum(v.nbytes for v in outb.values())
    # warm path once
    ctx.check(lib.mpm_state_upload(ctx.h, C.byref(view)))
    ctx.check(lib.mpm_advance(ctx.h, 1, 0))
    ctx.check(lib.mpm_state_download(ctx.h, C.byref(out)))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.check(lib.mpm_state_upload(ctx.h, C.byref(view)))
    ctx.check(lib.mpm_advance(ctx.h, steps, 0))
    ctx.check(lib.mpm_state_download(ctx.h, C.byref(out)))
    t1 = time.perf_counter()
    return {"value": n * steps / (t1 - t0), "unit": UNIT, "h2d_bytes_per_step": nbytes_in / steps,
            "d2h_bytes_per_step": nbytes_out / steps,
            "call": f"mpm_state_upload (pinned host) + mpm_advance({steps}) + mpm_state_download, wall clock",
            "seconds": t1 - t0}


def bench_reference(a, rank, world):
    """--impl reference: the reference's own CPU implementation of the step (oracle/_ref: the
    reference's headers compiled unmodified against the Eigen shim), rank 0 only, on all host
    cores: P processes (one per core, capped by host memory) each run the full scene -- the
    reference is serial and independent scenes are its only concurrency -- with
    ceil(W / P) untimed and ceil(K / P) timed steps (the reference's run() timer), so the whole
    run stays within a few minutes. value = sum of the per-process rates; `config` is the GPU
    arm's (workload_config)."""
    if rank != 0:
        return None
    import oracle
    cores = os.cpu_count() or 1
    per_proc_gb = _PROC_GB["fwd"].get(a.config, 1.0) * (0.5 if a.dtype == "f32" else 1.0)
    procs = max(1, min(cores, int(_mem_available_gb() * 0.6 / per_proc_gb)))
    k_each = max(1, -(-a.steps // procs))
    res = cpu_sample(a.config, a.dtype, k_each, procs=procs, warm=max(0, -(-a.warmup // procs)))
    value = res["value"]
    n = N_PARTICLES[a.config]
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": k_each * res["cores"], "warmup": a.warmup, "ms_per_step": n / value * 1e3,
            "higher_is_better": True, "scaling": "weak" if (world == 1 or a.scaling == "weak") else "strong",
            "vs_baseline": None, "dtype": a.dtype, "data": "synthetic (init_scene seeding, the reference's own)",
            "config": workload_config(a, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": res["cores"], "kind": res["kind"],
                             "sample": res["sample"], "cpu_model": res["cpu_model"], "label": res["label"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "steps = full-scene steps executed in total over the concurrent processes; ms_per_step = one "
                    "full-scene step at the aggregate rate"}


def main():
    a = parse()
    rank, world, local = dist_env()
    if a.impl == "reference":
        line = bench_reference(a, rank, world)
        if line:
            print(json.dumps(line), flush=True)
        return
    if a.mode == "pyslab":
        line = bench_slab(a, rank, world, local)
    elif a.mode == "slab" or (a.mode == "auto" and world > 1):
        line = bench_dist(a, rank, world, local)
    else:
        line = bench_b200(a, rank, world, local)
    if line is not None:
        if not a.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_baseline(a.config, a.dtype, 1)
            except Exception as e:  # the baseline is reported, never the target
                line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
            if line.get("fwd_adj"):
                try:
                    line["fwd_adj"]["cpu_baseline"] = cpu_baseline_adj(a.config, a.dtype)
                except Exception as e:
                    line["fwd_adj"]["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
