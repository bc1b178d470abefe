"""Pipeline switches and boundary description (host side of the boundary).

Same names, defaults and validation as the reference's
/root/reference/pkg/src/mpmbench/pipeline.py:50-114.  The ablation arms that exist only
to re-measure the paper's V100 ablations on a CPU (`fusion=split_*`, `sort=full_every_step`)
are accepted for API compatibility but rejected by the CUDA worker with ConfigError:
the CUDA core implements the default arms plus `transfer=split|g2p2g`,
`rebuild=amortized|every_step` and `sort=amortized|none_between`.
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError

FREE_ZONE_LO_CELLS = 3.5
FREE_ZONE_HI_CELLS = 6.5
FUSED_MARGIN_CELLS = 1.0
DEFAULT_FUSED_THRESHOLD = 100_000

N_COUNTERS = 6
C_ACCUM, C_QUARANTINE, C_DEGENERATE, C_SVD_CLAMP, C_ADDRESS_ERR, C_SUBGROUPS = range(6)

REBUILD_MODES = ("amortized", "every_step")
SORT_MODES = ("amortized", "full_every_step", "none_between")
FUSION_MODES = ("merged", "split_stress", "split_bc", "split_clear")
TRANSFER_MODES = ("split", "g2p2g")


@dataclass
class PipelineOptions:
    rebuild: str = "amortized"
    sort: str = "amortized"
    fusion: str = "merged"
    transfer: str = "split"
    deterministic: bool = False
    fused_threshold: int = DEFAULT_FUSED_THRESHOLD
    collect_conservation: bool = False

    def __post_init__(self):
        for value, allowed, name in ((self.rebuild, REBUILD_MODES, "rebuild"),
                                     (self.sort, SORT_MODES, "sort"),
                                     (self.fusion, FUSION_MODES, "fusion"),
                                     (self.transfer, TRANSFER_MODES, "transfer")):
            if value not in allowed:
                raise ConfigError(f"{name} must be one of {allowed}, got {value!r}")


@dataclass
class StepFlags:
    rebuild_needed: bool = True
    steps_since_rebuild: int = 0
    fused_mode: bool = False
    deterministic_mode: bool = False


@dataclass
class BoundaryBox:
    """Axis-aligned collision box: nodes on or outside it lose their outward normal
    velocity component (slip) or all velocity (sticky)."""
    min_corner: tuple
    max_corner: tuple
    mode: str = "slip"

    def __post_init__(self):
        if self.mode not in ("slip", "sticky"):
            raise ConfigError(f"boundary mode must be slip or sticky, got {self.mode!r}")
        for a in range(3):
            if not self.min_corner[a] < self.max_corner[a]:
                raise ConfigError("boundary box must have min < max per axis")


def free_zone_check(pos, block_origin, dx: float) -> bool:
    """True iff `pos` left the (10 dx)^3 free zone [origin-3.5dx, origin+6.5dx) of its block."""
    for a in range(3):
        lo = float(block_origin[a]) - FREE_ZONE_LO_CELLS * dx
        hi = float(block_origin[a]) + FREE_ZONE_HI_CELLS * dx
        if float(pos[a]) < lo or float(pos[a]) >= hi:
            return True
    return False
