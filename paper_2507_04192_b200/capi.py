"""ctypes mirror of include/mpm_capi.h (the C ABI of libmpm_b200.so).

The structs here are byte-compatible with the header; `load_library()` opens the in-tree
CUDA library and fails loudly when it is missing -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "_lib" / "libmpm_b200.so"

MPM_F32, MPM_F64 = 0, 1
MPM_OK = 0
MPM_ERR_USAGE = 1
MPM_ERR_VALIDATION = 2
MPM_ERR_NUMERICAL = 3
MPM_ERR_OUT_OF_DOMAIN = 4
MPM_ERR_CHECKPOINT = 5
MPM_ERR_CUDA = 6

SCHEME = {"pic": 0, "flip": 1, "blend": 2, "apic": 3, "tpic": 4}
WALL = {"slip": 0, "no_slip": 1, "fixed": 2, "fixed_wall": 2, "coulomb": 3}
MAT_FLUID, MAT_DP = 0, 1
MPM_ADV_NAN_GUARD = 1
MPM_ADV_STORE_GRID = 2
MPM_SEEDER_NONE, MPM_SEEDER_LAGRANGIAN_LS, MPM_SEEDER_EULERIAN_LS = 0, 1, 2

c_double_p = C.POINTER(C.c_double)


class SceneDesc(C.Structure):
    _fields_ = [
        ("dim", C.c_int),
        ("dtype", C.c_int),
        ("dh", C.c_double),
        ("cells", C.c_int * 3),
        ("origin", C.c_double * 3),
        ("dt", C.c_double),
        ("gravity", C.c_double * 3),
        ("scheme", C.c_int),
        ("alpha_flip", C.c_double),
        ("track_def_grad", C.c_int),
        ("material", C.c_int),
        ("rho0", C.c_double),
        ("viscosity", C.c_double),
        ("sound_speed", C.c_double),
        ("rate_form", C.c_int),
        ("K", C.c_double),
        ("nu", C.c_double),
        ("G", C.c_double),
        ("phi", C.c_double),
        ("psi", C.c_double),
        ("cohesion", C.c_double),
        ("sigma_t", C.c_double),
        ("q_phi", C.c_double),
        ("k_phi", C.c_double),
        ("q_psi", C.c_double),
        ("tau_P", C.c_double),
        ("alpha_P", C.c_double),
        ("band_layers", C.c_int),
        ("wall_kind", C.c_int * 6),
        ("n_friction", C.c_int * 6),
        ("friction", c_double_p * 6),
        ("n_obstacles", C.c_int),
        ("obstacles", c_double_p),
        ("mass_epsilon", C.c_double),
    ]


class StateView(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("x", C.c_void_p),
        ("v", C.c_void_p),
        ("mass", C.c_void_p),
        ("volume", C.c_void_p),
        ("rho", C.c_void_p),
        ("eps_eq", C.c_void_p),
        ("sigma_zz", C.c_void_p),
        ("sigma", C.c_void_p),
        ("grad_v", C.c_void_p),
        ("affine", C.c_void_p),
        ("def_grad", C.c_void_p),
        ("step", C.c_int64),
        ("time", C.c_double),
    ]


class CotView(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("x", C.c_void_p),
        ("v", C.c_void_p),
        ("rho", C.c_void_p),
        ("volume", C.c_void_p),
        ("eps_eq", C.c_void_p),
        ("sigma_zz", C.c_void_p),
        ("sigma", C.c_void_p),
        ("grad_v", C.c_void_p),
        ("affine", C.c_void_p),
    ]


class ParamGradsView(C.Structure):
    _fields_ = [
        ("sound_speed", C.c_double),
        ("viscosity", C.c_double),
        ("wall_friction", c_double_p * 6),
    ]


class GridView(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_int64),
        ("mass", C.c_void_p),
        ("momentum", C.c_void_p),
        ("v_old", C.c_void_p),
        ("v", C.c_void_p),
        ("force", C.c_void_p),
    ]


class SeederDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("field", C.c_int),
        ("n_obs", C.c_int),
        ("obs_steps", C.POINTER(C.c_int64)),
        ("n_sel", C.c_int64),
        ("sel", C.POINTER(C.c_int64)),
        ("target", C.c_void_p),
        ("n_regions", C.c_int64),
        ("centers", C.c_void_p),
        ("half", C.c_void_p),
        ("mask", C.POINTER(C.c_ubyte)),
    ]


class Region(C.Structure):
    """mpm_region: GeometryRegion + VelocityExpr (config.hpp:99-184)"""
    _fields_ = [
        ("shape", C.c_int),
        ("lo", C.c_double * 3), ("hi", C.c_double * 3),
        ("center", C.c_double * 3), ("radius", C.c_double), ("zmin", C.c_double), ("zmax", C.c_double),
        ("vel_kind", C.c_int),
        ("value", C.c_double * 3), ("alpha", C.c_double), ("h0", C.c_double), ("amplitude", C.c_double),
        ("perturbation", C.c_double), ("frequency", C.c_double),
        ("min_y", C.c_double),
    ]


class BackpropResultView(C.Structure):
    _fields_ = [
        ("loss", C.c_double),
        ("checkpoints_stored", C.c_int64),
        ("peak_replay_states", C.c_int64),
        ("device_ms", C.c_double),
    ]


def ptr(a: np.ndarray | None) -> int | None:
    """Raw data pointer of a C-contiguous numpy array (or None)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data


# Entry points exported by libmpm_b200.so (must match include/mpm_capi.h); tests check that
# every symbol declared in the header is exported.
_PROTOS = {
    "mpm_ctx_create": (C.c_int, [C.POINTER(SceneDesc), C.c_int64, C.c_int, C.POINTER(C.c_void_p)]),
    "mpm_ctx_destroy": (None, [C.c_void_p]),
    "mpm_last_error": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                 C.c_char_p, C.c_size_t]),
    "mpm_version": (C.c_int, []),
    "mpm_device_name": (C.c_int, [C.c_char_p, C.c_size_t]),
    "mpm_state_upload": (C.c_int, [C.c_void_p, C.POINTER(StateView)]),
    "mpm_state_download": (C.c_int, [C.c_void_p, C.POINTER(StateView)]),
    "mpm_state_digest": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "mpm_max_speed": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "mpm_advance": (C.c_int, [C.c_void_p, C.c_int64, C.c_uint32]),
    "mpm_advance_timed": (C.c_int, [C.c_void_p, C.c_int64, C.c_uint32, C.POINTER(C.c_double)]),
    "mpm_p2g": (C.c_int, [C.c_void_p]),
    "mpm_grid_momentum_update": (C.c_int, [C.c_void_p]),
    "mpm_grid_corrections": (C.c_int, [C.c_void_p]),
    "mpm_g2p": (C.c_int, [C.c_void_p]),
    "mpm_constitutive": (C.c_int, [C.c_void_p]),
    "mpm_grid_download": (C.c_int, [C.c_void_p, C.POINTER(GridView)]),
    "mpm_grid_upload": (C.c_int, [C.c_void_p, C.POINTER(GridView)]),
    "mpm_step_vjp": (C.c_int, [C.c_void_p, C.POINTER(StateView), C.POINTER(CotView), C.POINTER(CotView),
                               C.POINTER(ParamGradsView)]),
    "mpm_backprop": (C.c_int, [C.c_void_p, C.POINTER(StateView), C.c_int64, C.c_int, C.POINTER(SeederDesc),
                               C.POINTER(CotView), C.POINTER(ParamGradsView), C.POINTER(BackpropResultView)]),
    "mpm_slab_set": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int64]),
    "mpm_state_upload_ids": (C.c_int, [C.c_void_p, C.POINTER(StateView), C.c_void_p]),
    "mpm_state_download_local": (C.c_int, [C.c_void_p, C.POINTER(StateView), C.c_void_p]),
    "mpm_local_count": (C.c_int64, [C.c_void_p]),
    "mpm_step_p2g_local": (C.c_int, [C.c_void_p]),
    "mpm_step_grid_interior": (C.c_int, [C.c_void_p]),
    "mpm_snapshot_begin": (C.c_int, [C.c_void_p, C.c_int]),
    "mpm_snapshot_fetch": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(StateView)]),
    "mpm_init_scene": (C.c_int, [C.c_void_p, C.POINTER(Region), C.c_int, C.c_double, C.c_double, C.c_double,
                                 C.POINTER(C.c_int64)]),
    "mpm_slab_vjp_begin": (C.c_int, [C.c_void_p, C.POINTER(CotView)]),
    "mpm_slab_vjp_interior": (C.c_int, [C.c_void_p]),
    "mpm_slab_vjp_scatter": (C.c_int, [C.c_void_p]),
    "mpm_halo_cot": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int]),
    "mpm_slab_vjp_finish": (C.c_int, [C.c_void_p, C.POINTER(CotView), C.POINTER(ParamGradsView)]),
    "mpm_halo": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int]),
    "mpm_step_finish_local": (C.c_int, [C.c_void_p, C.c_uint32]),
    "mpm_step_finish_async": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p]),
    "mpm_step_commit": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int]),
    "mpm_particle_record_size": (C.c_int, [C.c_void_p]),
    "mpm_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "mpm_migrate_counts": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "mpm_migrate_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                     C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "mpm_migrate_import": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]),
    "mpm_profile_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "mpm_profile_query": (C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "mpm_profile_reset": (C.c_int, [C.c_void_p]),
    "mpm_launch_count": (C.c_int64, [C.c_void_p]),
    "mpm_grid_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "mpm_dist_unique_id": (C.c_int, [C.c_void_p]),
    "mpm_dist_attach_nccl": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int64]),
    "mpm_dist_advance": (C.c_int, [C.c_void_p, C.c_int64, C.c_uint32, C.POINTER(C.c_double)]),
    "mpm_dist_attach_local": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.POINTER(C.c_int), C.c_int64]),
    "mpm_dist_advance_local": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int64, C.c_uint32]),
    "mpm_dist_backprop": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.POINTER(SeederDesc), C.c_int64,
                                    C.POINTER(CotView), C.c_void_p, C.POINTER(ParamGradsView),
                                    C.POINTER(BackpropResultView)]),
    "mpm_dist_backprop_local": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int64, C.c_int, C.POINTER(SeederDesc),
                                          C.c_int64, C.POINTER(CotView), C.POINTER(C.c_void_p),
                                          C.POINTER(ParamGradsView), C.POINTER(BackpropResultView)]),
}
DIST_ID_BYTES = 128

_lib = None


def load_library(path: str | os.PathLike | None = None) -> C.CDLL:
    """Open libmpm_b200.so (in-tree build). Raises if it is missing: no fallback path."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"libmpm_b200.so not found at {p}; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return list(_PROTOS)
