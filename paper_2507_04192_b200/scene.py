"""Host-side mirror of the reference's scene description (scene.hpp, config.hpp, material.hpp).

Same names and meaning as the reference C++ types so parity tests read like the reference's own
tests: `Scene.config.{dh,cells,dt,gravity,scheme,origin,...}`, `Scene.material`,
`Scene.boundary.walls[w]`, `Scene.obstacles`, `Scene.geometry`, `Scene.mass_epsilon`.

`init_scene` is the reference's seeding (scene.hpp:55-116), vectorised with numpy: it is an
init-only host function (SURVEY.md §2 marks device seeding as "next"), kept here so the product
path never depends on the test oracle.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import capi
from .errors import ValidationError


def np_dtype(dtype: str):
    return np.float64 if dtype in ("f64", "float64", "double") else np.float32


@dataclass
class TransferScheme:
    """config.hpp:15-32"""
    kind: str = "flip"
    alpha_flip: float = 1.0

    def flip_fraction(self) -> float:
        return 1.0 if self.kind == "flip" else (self.alpha_flip if self.kind == "blend" else 0.0)

    def uses_affine(self) -> bool:
        return self.kind == "apic"

    def uses_velocity_gradient_transfer(self) -> bool:
        return self.kind == "tpic"


@dataclass
class FluidParams:
    """material.hpp:13-29 (positional order as the reference aggregate: rho0, viscosity, sound_speed)."""
    rho0: float = 1000.0
    viscosity: float = 0.0
    sound_speed: float = 35.0
    rate_form: bool = False

    def validate(self):
        if not self.rho0 > 0:
            raise ValidationError("fluid: rho0 must be positive")
        if not self.sound_speed > 0:
            raise ValidationError("fluid: sound_speed must be positive")
        if self.viscosity < 0:
            raise ValidationError("fluid: viscosity must be non-negative")


@dataclass
class DruckerPragerParams:
    """material.hpp:52-95; use DruckerPragerParams.make(...) for the derived constants."""
    rho0: float = 2650.0
    K: float = 7e5
    nu: float = 0.3
    G: float = 0.0
    phi: float = 0.0
    psi: float = 0.0
    cohesion: float = 0.0
    sigma_t: float = 0.0
    q_phi: float = 0.0
    k_phi: float = 0.0
    q_psi: float = 0.0
    tau_P: float = 0.0
    alpha_P: float = 0.0

    @staticmethod
    def make(rho0, K, nu, phi, psi, cohesion, sigma_t) -> "DruckerPragerParams":
        """DruckerPragerParams::make + dp_derived_params (material.hpp:37-84)."""
        s3 = math.sqrt(3.0)
        p = DruckerPragerParams(rho0=rho0, K=K, nu=nu, phi=phi, psi=psi, cohesion=cohesion, sigma_t=sigma_t)
        p.G = 3.0 * K * (1.0 - 2.0 * nu) / (2.0 * (1.0 + nu))
        p.q_phi = 6.0 * math.sin(phi) / (s3 * (3.0 + math.sin(phi)))
        p.k_phi = 6.0 * cohesion * math.cos(phi) / (s3 * (3.0 + math.sin(phi)))
        p.q_psi = 6.0 * math.sin(psi) / (s3 * (3.0 + math.sin(psi)))
        p.tau_P = p.k_phi - p.q_phi * sigma_t
        p.alpha_P = math.sqrt(1.0 + p.q_phi * p.q_phi) - p.q_phi
        p.validate()
        return p

    def validate(self):
        if not self.rho0 > 0:
            raise ValidationError("drucker_prager: rho0 must be positive")
        if not self.K > 0:
            raise ValidationError("drucker_prager: bulk modulus must be positive")
        if not (0 <= self.nu < 0.5):
            raise ValidationError("drucker_prager: poisson ratio must lie in [0, 0.5)")
        if not self.G > 0:
            raise ValidationError("drucker_prager: derived shear modulus must be positive")
        if not (0 <= self.phi < 1.5707963267948966):
            raise ValidationError("drucker_prager: friction angle must lie in [0, pi/2)")
        if not (0 <= self.psi <= self.phi):
            raise ValidationError("drucker_prager: dilation angle must lie in [0, phi]")
        if self.cohesion < 0 or self.sigma_t < 0:
            raise ValidationError("drucker_prager: cohesion and tension cutoff must be non-negative")
        if self.q_phi > 0 and self.sigma_t > self.k_phi / self.q_phi:
            raise ValidationError("drucker_prager: tension cutoff must not exceed the cone apex k_phi/q_phi")


def material_wave_speed(m) -> float:
    """material.hpp:116-125"""
    if isinstance(m, FluidParams):
        return m.sound_speed
    return math.sqrt((m.K + 4.0 * m.G / 3.0) / m.rho0)


@dataclass
class Wall:
    """config.hpp:39-43"""
    kind: str = "slip"
    friction: list = field(default_factory=list)


@dataclass
class BoundarySpec:
    """config.hpp:45-57 (wall index w = 2*axis + side)"""
    dim: int = 2
    walls: list = None
    band_layers: int = 2

    def __post_init__(self):
        if self.walls is None:
            self.walls = [Wall() for _ in range(2 * self.dim)]

    def has_coulomb(self) -> bool:
        return any(w.kind == "coulomb" for w in self.walls)


@dataclass
class Obstacle:
    """config.hpp:61-88"""
    lo: list
    hi: list


@dataclass
class VelocityExpr:
    """config.hpp:99-130 (mlp_field is not supported on this path)."""
    kind: str = "constant"  # constant | linear_in_y | parabolic_sine
    value: list = None
    alpha: float = 0.0
    h0: float = 1.0
    amplitude: float = 2.0
    perturbation: float = 0.2
    frequency: float = 4.0


@dataclass
class GeometryRegion:
    """config.hpp:136-184"""
    shape: str = "box"  # box | cylinder
    lo: list = None
    hi: list = None
    center: list = None
    radius: float = 0.0
    zmin: float = 0.0
    zmax: float = 0.0
    velocity: VelocityExpr = field(default_factory=VelocityExpr)

    def bound_lo(self, dim):
        if self.shape == "box":
            return list(self.lo)
        b = [c - self.radius for c in self.center[:dim]]
        if dim == 3:
            b[2] = self.zmin
        return b

    def bound_hi(self, dim):
        if self.shape == "box":
            return list(self.hi)
        b = [c + self.radius for c in self.center[:dim]]
        if dim == 3:
            b[2] = self.zmax
        return b

    def min_y(self):
        return self.lo[1] if self.shape == "box" else self.center[1] - self.radius


@dataclass
class SimConfig:
    """config.hpp:188-227"""
    dim: int = 2
    dh: float = 0.0
    cells: list = None
    dt: float = 0.0
    num_steps: int = 0
    snapshot_stride: int = 0
    gravity: list = None
    scheme: TransferScheme = field(default_factory=TransferScheme)
    particles_per_cell: int = None
    seed: int = 0
    track_def_grad: bool = False
    origin: list = None

    def __post_init__(self):
        d = self.dim
        self.cells = list(self.cells) if self.cells is not None else [0] * d
        self.gravity = list(self.gravity) if self.gravity is not None else [0.0] * d
        self.origin = list(self.origin) if self.origin is not None else [0.0] * d
        if self.particles_per_cell is None:
            self.particles_per_cell = 1 << d

    def domain_extent(self):
        return [c * self.dh for c in self.cells]

    def validate(self):
        if not self.dh > 0:
            raise ValidationError("config: grid spacing must be positive")
        if any(c < 5 for c in self.cells[: self.dim]):
            raise ValidationError("config: need at least 5 cells per axis")
        if not self.dt > 0:
            raise ValidationError("config: time step must be positive")
        if self.num_steps < 0:
            raise ValidationError("config: step count must be non-negative")
        if self.particles_per_cell != (1 << self.dim):
            raise ValidationError("config: particles_per_cell must be 2^dim (regular sub-cell lattice)")


def cfl_report(cfg: SimConfig, material, vmax: float) -> float:
    """config.hpp:229-234: Courant number dt*(c_eff + vmax)/dh."""
    return cfg.dt * (material_wave_speed(material) + vmax) / cfg.dh


class Scene:
    """scene.hpp:9-49. `dtype` selects T (f64 = the reference's tested instantiation)."""

    def __init__(self, dim: int = 2, dtype: str = "f64"):
        self.dim = dim
        self.dtype = dtype
        self.config = SimConfig(dim=dim)
        self.material = FluidParams()
        self.boundary = BoundarySpec(dim=dim)
        self.obstacles: list[Obstacle] = []
        self.geometry: list[GeometryRegion] = []
        self.mass_epsilon = 0.0

    @property
    def np_dtype(self):
        return np_dtype(self.dtype)

    def copy(self) -> "Scene":
        import copy
        return copy.deepcopy(self)

    def validate(self):
        cfg = self.config
        cfg.validate()
        self.material.validate()
        if not self.geometry:
            raise ValidationError("scene: no geometry regions")
        ext = cfg.domain_extent()
        margin = 2 * cfg.dh
        for g in self.geometry:
            lo, hi = g.bound_lo(self.dim), g.bound_hi(self.dim)
            for a in range(self.dim):
                if not hi[a] > lo[a]:
                    raise ValidationError(f"scene: geometry region is empty on axis {a}")
                if lo[a] < margin - 1e-12 * cfg.dh or hi[a] > ext[a] - margin + 1e-12 * cfg.dh:
                    raise ValidationError(f"scene: geometry must keep a 2-cell margin inside the grid (axis {a})")
        self.validate_dynamics()

    def validate_dynamics(self):
        ext = self.config.domain_extent()
        for ob in self.obstacles:
            for a in range(self.dim):
                if ob.lo[a] < 0 or ob.hi[a] > ext[a] or not ob.hi[a] > ob.lo[a]:
                    raise ValidationError("scene: obstacle box must be a non-empty box inside the domain")
        for w in self.boundary.walls:
            if w.kind == "coulomb":
                if not w.friction:
                    raise ValidationError("scene: coulomb wall needs at least one segment")
                if any(mu < 0 for mu in w.friction):
                    raise ValidationError("scene: friction coefficients must be non-negative")

    # ---- ABI descriptor -------------------------------------------------------------
    def to_desc(self) -> "DescHolder":
        return DescHolder(self)


class DescHolder:
    """Owns an `mpm_scene_desc` plus the arrays its pointers reference."""

    def __init__(self, s: Scene):
        d = capi.SceneDesc()
        cfg = s.config
        d.dim = s.dim
        d.dtype = capi.MPM_F64 if s.np_dtype == np.float64 else capi.MPM_F32
        d.dh = cfg.dh
        for a in range(s.dim):
            d.cells[a] = int(cfg.cells[a])
            d.origin[a] = cfg.origin[a]
            d.gravity[a] = cfg.gravity[a]
        d.dt = cfg.dt
        d.scheme = capi.SCHEME[cfg.scheme.kind]
        d.alpha_flip = cfg.scheme.alpha_flip
        d.track_def_grad = int(bool(cfg.track_def_grad))
        m = s.material
        if isinstance(m, FluidParams):
            d.material = capi.MAT_FLUID
            d.rho0, d.viscosity, d.sound_speed, d.rate_form = m.rho0, m.viscosity, m.sound_speed, int(m.rate_form)
        else:
            d.material = capi.MAT_DP
            for k in ("rho0", "K", "nu", "G", "phi", "psi", "cohesion", "sigma_t", "q_phi", "k_phi", "q_psi",
                      "tau_P", "alpha_P"):
                setattr(d, k, getattr(m, k))
        d.band_layers = s.boundary.band_layers
        self._fr = []
        for w, wall in enumerate(s.boundary.walls):
            d.wall_kind[w] = capi.WALL[wall.kind]
            arr = np.ascontiguousarray(np.asarray(wall.friction, dtype=np.float64))
            self._fr.append(arr)
            d.n_friction[w] = len(arr)
            d.friction[w] = arr.ctypes.data_as(capi.c_double_p) if len(arr) else None
        obs = []
        for ob in s.obstacles:
            obs += list(ob.lo[: s.dim]) + list(ob.hi[: s.dim])
        self._obs = np.ascontiguousarray(np.asarray(obs, dtype=np.float64))
        d.n_obstacles = len(s.obstacles)
        d.obstacles = self._obs.ctypes.data_as(capi.c_double_p) if len(obs) else None
        d.mass_epsilon = s.mass_epsilon
        self.desc = d
        self.scene = s

    @property
    def ref(self):
        return C.byref(self.desc)


# ---------------------------------------------------------------------------------------
def _region_contains(g: GeometryRegion, p: np.ndarray, dim: int, T) -> np.ndarray:
    """GeometryRegion::contains (config.hpp:146-162), vectorised over points p[n, dim]."""
    if g.shape == "box":
        ok = np.ones(len(p), dtype=bool)
        for a in range(dim):
            ok &= (p[:, a] >= T(g.lo[a])) & (p[:, a] < T(g.hi[a]))
        return ok
    ok = np.ones(len(p), dtype=bool)
    if dim == 3:
        ok &= (p[:, 2] >= T(g.zmin)) & (p[:, 2] < T(g.zmax))
    dx = p[:, 0] - T(g.center[0])
    dy = p[:, 1] - T(g.center[1])
    r = T(g.radius)
    return ok & (dx * dx + dy * dy < r * r)


def _velocity(g: GeometryRegion, y_rel: np.ndarray, dim: int, T) -> np.ndarray:
    """VelocityExpr::evaluate (config.hpp:109-129)."""
    ve = g.velocity
    out = np.zeros((len(y_rel), dim), dtype=T)
    if ve.kind == "constant":
        val = ve.value if ve.value is not None else [0.0] * dim
        out[:] = np.asarray(val[:dim], dtype=T)
    elif ve.kind == "linear_in_y":
        out[:, 0] = T(ve.alpha) * (T(ve.h0) - y_rel)
    elif ve.kind == "parabolic_sine":
        yn = y_rel / T(ve.h0)
        out[:, 0] = T(ve.amplitude) * (T(1) - yn * yn) + T(ve.perturbation) * np.sin(
            T(ve.frequency) * T(math.pi) * yn)
    else:
        raise ValidationError(f"velocity expression {ve.kind!r} is not supported")
    return out


def seeding_constants(scene: Scene):
    """(mpm_region list, mass, volume, rho0) of init_scene for the device seeding; validates the
    scene and sets scene.mass_epsilon exactly as init_scene does"""
    from . import capi

    scene.validate()
    dim, T = scene.dim, scene.np_dtype
    dh = T(scene.config.dh)
    rho0 = T(scene.material.rho0)
    mp = T(rho0 * T(T(dh) ** dim) / T(1 << dim))
    kinds = {"constant": 0, "linear_in_y": 1, "parabolic_sine": 2}
    regs = []
    for g in scene.geometry:
        r = capi.Region()
        r.shape = 0 if g.shape == "box" else 1
        for a in range(dim):
            if g.shape == "box":
                r.lo[a], r.hi[a] = g.lo[a], g.hi[a]
        if g.shape != "box":
            for a in range(2):
                r.center[a] = g.center[a]
            r.radius, r.zmin, r.zmax = g.radius, g.zmin, g.zmax
        ve = g.velocity
        if ve.kind not in kinds:
            raise ValidationError(f"velocity expression {ve.kind!r} is not supported")
        r.vel_kind = kinds[ve.kind]
        val = ve.value if ve.value is not None else [0.0] * dim
        for a in range(dim):
            r.value[a] = val[a]
        r.alpha, r.h0, r.amplitude, r.perturbation, r.frequency = ve.alpha, ve.h0, ve.amplitude, ve.perturbation, \
            ve.frequency
        r.min_y = float(T(g.min_y()))
        regs.append(r)
    scene.mass_epsilon = float(T(T(1e-12) * mp))
    return regs, float(mp), float(T(mp / rho0)), float(rho0)


def seeding_capacity(scene: Scene) -> int:
    """upper bound on init_scene's particle count: 2^d per cell of the regions' bounding box"""
    cfg, dim = scene.config, scene.dim
    n = 1 << dim
    for a in range(dim):
        lo = min(g.bound_lo(dim)[a] for g in scene.geometry)
        hi = max(g.bound_hi(dim)[a] for g in scene.geometry)
        lc = max(0, int(math.floor((lo - cfg.origin[a]) / cfg.dh)) - 1)
        hc = min(cfg.cells[a], int(math.ceil((hi - cfg.origin[a]) / cfg.dh)) + 1)
        n *= max(0, hc - lc)
    return n


def init_scene(scene: Scene):
    """init_scene (scene.hpp:55-116): 2^d sub-cell lattice at +-dh/4 in every covered cell, cells
    visited row-major (axis 0 slowest), corners in bit order; first containing region owns the
    particle. Sets scene.mass_epsilon and returns a SimState."""
    from .state import SimState

    scene.validate()
    dim, T = scene.dim, scene.np_dtype
    cfg = scene.config
    dh = T(cfg.dh)
    rho0 = T(scene.material.rho0)
    mp = T(rho0 * T(T(dh) ** dim) / T(1 << dim))
    # restrict the row-major cell visit to the union bounding box of the regions (order-preserving)
    lo_c, hi_c = [], []
    for a in range(dim):
        los = [g.bound_lo(dim)[a] for g in scene.geometry]
        his = [g.bound_hi(dim)[a] for g in scene.geometry]
        lo_c.append(max(0, int(math.floor((min(los) - cfg.origin[a]) / cfg.dh)) - 1))
        hi_c.append(min(cfg.cells[a], int(math.ceil((max(his) - cfg.origin[a]) / cfg.dh)) + 1))
    xs, owners = [], []
    corners = np.array([[((c >> a) & 1) for a in range(dim)] for c in range(1 << dim)], dtype=bool)
    quarter = T(dh / T(4))
    for i0 in range(lo_c[0], hi_c[0]):  # chunk along axis 0 (slowest)
        axes = [np.array([i0])] + [np.arange(lo_c[a], hi_c[a]) for a in range(1, dim)]
        grid = np.meshgrid(*axes, indexing="ij")
        ci = np.stack([g.reshape(-1) for g in grid], axis=1)  # row-major cells
        center = np.empty(ci.shape, dtype=T)
        for a in range(dim):
            center[:, a] = T(cfg.origin[a]) + (ci[:, a].astype(T) + T(0.5)) * dh
        p = np.repeat(center, 1 << dim, axis=0)
        cb = np.tile(corners, (len(center), 1))
        p = np.where(cb, p + quarter, p - quarter).astype(T)
        owner = np.full(len(p), -1, dtype=np.int64)
        for r, g in enumerate(scene.geometry):
            hit = (owner < 0) & _region_contains(g, p, dim, T)
            owner[hit] = r
        keep = owner >= 0
        if keep.any():
            xs.append(p[keep])
            owners.append(owner[keep])
    if not xs:
        raise ValidationError("scene: geometry produced no particles")
    x = np.ascontiguousarray(np.concatenate(xs))
    owner = np.concatenate(owners)
    n = len(x)
    st = SimState.zeros(n, dim, T, with_affine=cfg.scheme.uses_affine(), with_def_grad=cfg.track_def_grad)
    st.particles.x[:] = x
    st.particles.mass[:] = mp
    st.particles.rho[:] = rho0
    st.particles.volume[:] = T(mp / rho0)
    for r, g in enumerate(scene.geometry):
        sel = owner == r
        if sel.any():
            st.particles.v[sel] = _velocity(g, x[sel, 1] - T(g.min_y()), dim, T)
    scene.mass_epsilon = float(T(T(1e-12) * mp))
    if isinstance(scene.material, FluidParams):
        vmax = float(np.sqrt((st.particles.v.astype(np.float64) ** 2).sum(axis=1)).max())
        courant = cfl_report(cfg, scene.material, vmax)
        if courant > 1:
            raise ValidationError(f"scene: CFL violation, Courant number {courant} > 1 (reduce dt or coarsen the grid)")
    return st
