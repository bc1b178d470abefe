"""B200-native MLS-MPM substep core behind the reference package's Worker API."""
from .errors import (BarrierTimeoutError, ConfigError, ContractViolationError,
                     DegenerateStateError, ModeConflictError, RejectedInputError,
                     ResourceError, SimulationError, SpatialDomainError)
from .domain import Material, MaterialKind, SimParams, cfl_dt
from .options import (BoundaryBox, PipelineOptions, StepFlags, free_zone_check)
from .multiworker import SharedRuntime, efficiency, partition_particles

__all__ = [
    "BarrierTimeoutError", "ConfigError", "ContractViolationError", "DegenerateStateError",
    "ModeConflictError", "RejectedInputError", "ResourceError", "SimulationError",
    "SpatialDomainError", "Material", "MaterialKind", "SimParams", "cfl_dt", "BoundaryBox",
    "PipelineOptions", "StepFlags", "free_zone_check", "SharedRuntime", "efficiency",
    "partition_particles", "CudaWorker", "CudaCluster", "make_single_worker",
]


def __getattr__(name):
    # the CUDA-facing classes import torch; keep `import paper_2111_00699_b200` light
    if name in ("CudaWorker", "make_single_worker"):
        from . import worker
        return getattr(worker, name)
    if name == "CudaCluster":
        from .cluster import CudaCluster
        return CudaCluster
    raise AttributeError(name)
