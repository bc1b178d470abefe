"""B200-native MLS-MPM substep core behind the reference package's Worker API."""
from .errors import (BarrierTimeoutError, ConfigError, ContractViolationError,
                     DegenerateStateError, ModeConflictError, RejectedInputError,
                     ResourceError, SimulationError, SpatialDomainError)
from .domain import Material, MaterialKind, SimParams, cfl_dt
from .options import (BoundaryBox, PipelineOptions, StepFlags, free_zone_check)

__all__ = [
    "BarrierTimeoutError", "ConfigError", "ContractViolationError", "DegenerateStateError",
    "ModeConflictError", "RejectedInputError", "ResourceError", "SimulationError",
    "SpatialDomainError", "Material", "MaterialKind", "SimParams", "cfl_dt", "BoundaryBox",
    "PipelineOptions", "StepFlags", "free_zone_check",
]
