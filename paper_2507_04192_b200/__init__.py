"""B200-native MPM one-step operator Phi = G2P o U o P2G and its adjoint (arXiv 2507.04192).

Host-side mirror of the reference's C++ solver API (namespace mpm in /root/reference/proj/include)
over the C ABI of the in-tree CUDA library `_lib/libmpm_b200.so` (include/mpm_capi.h).
"""
from .errors import MPMError, NumericalError, OutOfDomainError, ValidationError, DeviceError  # noqa: F401
from .scene import (  # noqa: F401
    BoundarySpec, DruckerPragerParams, FluidParams, GeometryRegion, Obstacle, Scene, SimConfig,
    TransferScheme, VelocityExpr, Wall, cfl_report, init_scene, material_wave_speed,
)
from .state import Grid, ParamGrads, ParticleSoA, SimState, StateCotangent  # noqa: F401


def __getattr__(name):
    # the solver loads the CUDA library; import it lazily so CPU-only tooling can use the types
    if name in ("Stepper", "run", "step_vjp", "backprop_trajectory", "CheckpointPlan", "Context",
                "AdjointWorkspace", "RunResult", "max_particle_speed", "constitutive_update", "p2g",
                "grid_momentum_update", "apply_grid_corrections", "g2p"):
        from . import solver
        return getattr(solver, name)
    raise AttributeError(name)
