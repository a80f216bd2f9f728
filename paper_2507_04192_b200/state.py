"""Host-side mirror of the reference's state types (state.hpp, adjoint.hpp) as numpy arrays.

Matrices are stored as [n, dim, dim] with [p, i, j] = M_p(i, j); the ABI views use the
reference's Eigen layout (column-major per particle), converted in `to_view` / `from_view`.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi


def _colmajor(m: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.transpose(m, (0, 2, 1)))


def _from_colmajor(buf: np.ndarray, n: int, d: int) -> np.ndarray:
    return np.ascontiguousarray(buf.reshape(n, d, d).transpose(0, 2, 1))


class ParticleSoA:
    """state.hpp:17-63"""

    FIELDS = ("x", "v", "mass", "volume", "rho", "eps_eq", "sigma_zz", "sigma", "grad_v", "affine", "def_grad")

    def __init__(self, n, dim, dtype, with_affine=False, with_def_grad=False):
        T = dtype
        self.dim = dim
        self.x = np.zeros((n, dim), T)
        self.v = np.zeros((n, dim), T)
        self.mass = np.zeros(n, T)
        self.volume = np.zeros(n, T)
        self.rho = np.zeros(n, T)
        self.eps_eq = np.zeros(n, T)
        self.sigma_zz = np.zeros(n if dim == 2 else 0, T)
        self.sigma = np.zeros((n, dim, dim), T)
        self.grad_v = np.zeros((n, dim, dim), T)
        self.affine = np.zeros((n, dim, dim), T) if with_affine else None
        self.def_grad = np.tile(np.eye(dim, dtype=T), (n, 1, 1)) if with_def_grad else None

    def size(self) -> int:
        return len(self.x)

    @property
    def dtype(self):
        return self.x.dtype

    def all_finite(self) -> bool:
        """state.hpp:48-62"""
        fs = [self.x, self.v, self.volume, self.rho, self.eps_eq, self.sigma_zz, self.sigma, self.grad_v]
        if self.affine is not None:
            fs.append(self.affine)
        return all(np.isfinite(a).all() for a in fs)

    def copy(self) -> "ParticleSoA":
        c = ParticleSoA.__new__(ParticleSoA)
        c.dim = self.dim
        for f in self.FIELDS:
            a = getattr(self, f)
            setattr(c, f, None if a is None else a.copy())
        return c


    def take(self, idx) -> "ParticleSoA":
        """rows idx (a rank's subset under a slab decomposition)"""
        c = ParticleSoA.__new__(ParticleSoA)
        c.dim = self.dim
        for f in self.FIELDS:
            a = getattr(self, f)
            setattr(c, f, None if a is None else (a[idx] if a.shape[0] else a.copy()))
        return c

    def put(self, idx, other: "ParticleSoA"):
        """rows idx <- other (inverse of take)"""
        for f in self.FIELDS:
            a, b = getattr(self, f), getattr(other, f)
            if a is not None and a.shape[0]:
                a[idx] = b


class SimState:
    """state.hpp:65-87"""

    def __init__(self, particles: ParticleSoA, step: int = 0, time: float = 0.0):
        self.particles = particles
        self.step = step
        self.time = time

    @staticmethod
    def zeros(n, dim, dtype, with_affine=False, with_def_grad=False) -> "SimState":
        return SimState(ParticleSoA(n, dim, dtype, with_affine, with_def_grad))

    def copy(self) -> "SimState":
        return SimState(self.particles.copy(), self.step, self.time)

    # ---- ABI views -------------------------------------------------------------------
    def to_view(self):
        """Returns (StateView, keepalive). Matrices converted to Eigen column-major."""
        p = self.particles
        n, d = p.size(), p.dim
        keep = {
            "x": np.ascontiguousarray(p.x),
            "v": np.ascontiguousarray(p.v),
            "mass": np.ascontiguousarray(p.mass),
            "volume": np.ascontiguousarray(p.volume),
            "rho": np.ascontiguousarray(p.rho),
            "eps_eq": np.ascontiguousarray(p.eps_eq),
            "sigma_zz": np.ascontiguousarray(p.sigma_zz) if d == 2 else None,
            "sigma": _colmajor(p.sigma),
            "grad_v": _colmajor(p.grad_v),
            "affine": _colmajor(p.affine) if p.affine is not None else None,
            "def_grad": _colmajor(p.def_grad) if p.def_grad is not None else None,
        }
        v = capi.StateView()
        v.n = n
        for k, a in keep.items():
            setattr(v, k, capi.ptr(a) if a is not None and a.size else None)
        v.step = int(self.step)
        v.time = float(self.time)
        return v, keep

    def output_view(self):
        """A writable view whose buffers are filled by the callee; call `sync_from(keep)` after."""
        p = self.particles
        n, d = p.size(), p.dim
        T = p.dtype
        keep = {
            "x": np.empty((n, d), T), "v": np.empty((n, d), T), "mass": np.empty(n, T),
            "volume": np.empty(n, T), "rho": np.empty(n, T), "eps_eq": np.empty(n, T),
            "sigma_zz": np.empty(n, T) if d == 2 else None,
            "sigma": np.empty(n * d * d, T), "grad_v": np.empty(n * d * d, T),
            "affine": np.empty(n * d * d, T) if p.affine is not None else None,
            "def_grad": np.empty(n * d * d, T) if p.def_grad is not None else None,
        }
        v = capi.StateView()
        v.n = n
        for k, a in keep.items():
            setattr(v, k, capi.ptr(a) if a is not None and a.size else None)
        return v, keep

    def sync_from(self, view, keep):
        p = self.particles
        n, d = p.size(), p.dim
        for k in ("x", "v", "mass", "volume", "rho", "eps_eq"):
            getattr(p, k)[...] = keep[k].reshape(getattr(p, k).shape)
        if d == 2:
            p.sigma_zz[...] = keep["sigma_zz"]
        for k in ("sigma", "grad_v", "affine", "def_grad"):
            if keep[k] is not None and getattr(p, k) is not None:
                getattr(p, k)[...] = _from_colmajor(keep[k].reshape(-1), n, d)
        self.step = int(view.step)
        self.time = float(view.time)

    def hash_inputs(self):
        return self.to_view()


class StateCotangent:
    """adjoint.hpp:10-72 (sigma/grad_v/affine cotangents are full matrices)."""

    FIELDS = ("x", "v", "rho", "volume", "eps_eq", "sigma_zz", "sigma", "grad_v", "affine")

    def __init__(self, n, dim, dtype, with_affine=False):
        T = dtype
        self.dim = dim
        self.x = np.zeros((n, dim), T)
        self.v = np.zeros((n, dim), T)
        self.rho = np.zeros(n, T)
        self.volume = np.zeros(n, T)
        self.eps_eq = np.zeros(n, T)
        self.sigma_zz = np.zeros(n if dim == 2 else 0, T)
        self.sigma = np.zeros((n, dim, dim), T)
        self.grad_v = np.zeros((n, dim, dim), T)
        self.affine = np.zeros((n, dim, dim), T) if with_affine else None

    @staticmethod
    def zeros_like(prt: ParticleSoA) -> "StateCotangent":
        return StateCotangent(prt.size(), prt.dim, prt.dtype, prt.affine is not None)

    def copy(self):
        c = StateCotangent.__new__(StateCotangent)
        c.dim = self.dim
        for f in self.FIELDS:
            a = getattr(self, f)
            setattr(c, f, None if a is None else a.copy())
        return c

    def take(self, idx) -> "StateCotangent":
        """rows idx (a rank's particles under the slab decomposition)"""
        c = StateCotangent.__new__(StateCotangent)
        c.dim = self.dim
        for f in self.FIELDS:
            a = getattr(self, f)
            setattr(c, f, None if a is None else (a[idx] if a.shape[0] else a.copy()))
        return c

    def put(self, idx, other: "StateCotangent"):
        for f in self.FIELDS:
            a, b = getattr(self, f), getattr(other, f)
            if a is not None and a.shape[0]:
                a[idx] = b

    def axpy(self, a, o: "StateCotangent"):
        for f in self.FIELDS:
            x = getattr(self, f)
            if x is not None:
                x += a * getattr(o, f)

    def dot(self, o: "StateCotangent") -> float:
        s = 0.0
        for f in ("x", "v", "rho", "volume", "sigma_zz", "sigma", "grad_v", "affine"):
            x = getattr(self, f)
            if x is not None:
                s += float((x.astype(np.float64) * getattr(o, f).astype(np.float64)).sum())
        return s

    def to_view(self):
        n, d = len(self.x), self.dim
        keep = {
            "x": np.ascontiguousarray(self.x), "v": np.ascontiguousarray(self.v),
            "rho": np.ascontiguousarray(self.rho), "volume": np.ascontiguousarray(self.volume),
            "eps_eq": np.ascontiguousarray(self.eps_eq),
            "sigma_zz": np.ascontiguousarray(self.sigma_zz) if d == 2 else None,
            "sigma": _colmajor(self.sigma), "grad_v": _colmajor(self.grad_v),
            "affine": _colmajor(self.affine) if self.affine is not None else None,
        }
        v = capi.CotView()
        v.n = n
        for k, a in keep.items():
            setattr(v, k, capi.ptr(a) if a is not None and a.size else None)
        return v, keep

    def sync_from(self, keep):
        n, d = len(self.x), self.dim
        for k in ("x", "v", "rho", "volume", "eps_eq"):
            getattr(self, k)[...] = keep[k].reshape(getattr(self, k).shape)
        if d == 2:
            self.sigma_zz[...] = keep["sigma_zz"]
        for k in ("sigma", "grad_v", "affine"):
            if keep[k] is not None and getattr(self, k) is not None:
                getattr(self, k)[...] = _from_colmajor(keep[k].reshape(-1), n, d)


class ParamGrads:
    """adjoint.hpp:77-90"""

    def __init__(self, boundary):
        self.sound_speed = 0.0
        self.viscosity = 0.0
        self.wall_friction = [np.zeros(len(w.friction), np.float64) for w in boundary.walls]
        while len(self.wall_friction) < 6:
            self.wall_friction.append(np.zeros(0, np.float64))

    @staticmethod
    def zeros_like(boundary) -> "ParamGrads":
        return ParamGrads(boundary)

    def to_view(self):
        v = capi.ParamGradsView()
        v.sound_speed = self.sound_speed
        v.viscosity = self.viscosity
        for w in range(6):
            a = self.wall_friction[w]
            v.wall_friction[w] = a.ctypes.data_as(capi.c_double_p) if len(a) else None
        return v

    def sync_from(self, v):
        self.sound_speed = float(v.sound_speed)
        self.viscosity = float(v.viscosity)

    def flat(self) -> np.ndarray:
        """(c, mu, friction of every wall) as one f64 vector"""
        return np.concatenate([[self.sound_speed, self.viscosity], *self.wall_friction]).astype(np.float64)

    def add_flat(self, vec: np.ndarray):
        self.sound_speed += float(vec[0])
        self.viscosity += float(vec[1])
        k = 2
        for a in self.wall_friction:
            a += vec[k:k + len(a)]
            k += len(a)


class Grid:
    """state.hpp:172-254 (dense, row-major node index)."""

    def __init__(self, cells, dh, origin, dtype, dim):
        self.cells = list(cells[:dim])
        self.dh = dh
        self.origin = list(origin[:dim])
        self.dim = dim
        n = self.num_nodes()
        self.mass = np.zeros(n, dtype)
        self.momentum = np.zeros((n, dim), dtype)
        self.v_old = np.zeros((n, dim), dtype)
        self.v = np.zeros((n, dim), dtype)
        self.force = np.zeros((n, dim), dtype)

    def num_nodes(self) -> int:
        n = 1
        for c in self.cells:
            n *= c + 1
        return n

    def node_index(self, idx) -> int:
        r = 0
        for a in range(self.dim):
            r = r * (self.cells[a] + 1) + idx[a]
        return r

    def to_view(self):
        v = capi.GridView()
        v.num_nodes = self.num_nodes()
        for k in ("mass", "momentum", "v_old", "v", "force"):
            setattr(v, k, capi.ptr(getattr(self, k)))
        return v
