"""Step parameters and material description (host side of the boundary).

Mirrors the reference's value types field for field
(/root/reference/pkg/src/mpmbench/domain.py:26-113, 523-532) so a scene written for the
reference constructs the CUDA worker unchanged.  Units are CGS.  Two material kinds the
reference does not have are added for the plastic rows of the scope table
(SNOW = fixed-corotated + singular-value clamp with hardening, SAND = Drucker-Prager);
they are handled by the same kernels through `Material.kind`.
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass

from .errors import RejectedInputError


class MaterialKind(enum.IntEnum):
    WEAKLY_COMPRESSIBLE_FLUID = 0
    FIXED_COROTATED = 1
    SNOW = 2          # not in the reference: Stomakhin clamp + hardening
    SAND = 3          # not in the reference: Drucker-Prager return mapping


@dataclass
class SimParams:
    dx: float
    dt: float
    gravity: tuple = (0.0, 0.0, -981.0)
    frame_dt: float = 1.0 / 48.0
    steps_per_frame: int = 36
    cfl: float = 0.5
    lane_width: int = 32
    flip_blend: float = 0.0

    def __post_init__(self):
        if not (self.dx > 0.0):
            raise RejectedInputError(f"dx must be positive, got {self.dx}")
        if not (self.dt > 0.0):
            raise RejectedInputError(f"dt must be positive, got {self.dt}")
        if self.steps_per_frame < 1:
            raise RejectedInputError(f"steps_per_frame must be >= 1, got {self.steps_per_frame}")
        if not (0.0 < self.cfl <= 1.0):
            raise RejectedInputError(f"cfl must be in (0, 1], got {self.cfl}")
        lw = self.lane_width
        if lw < 1 or lw > 64 or (lw & (lw - 1)) != 0:
            raise RejectedInputError(f"lane_width must be a power of two <= 64, got {lw}")
        if not (0.0 <= self.flip_blend <= 1.0):
            raise RejectedInputError(f"flip_blend must be in [0, 1], got {self.flip_blend}")
        self.gravity = tuple(float(g) for g in self.gravity)


@dataclass
class Material:
    kind: MaterialKind
    density: float
    bulk_modulus: float = 0.0
    gamma: float = 7.0
    mu: float = 0.0
    lam: float = 0.0
    clamp_tension: bool = False
    # plastic extensions (ignored by kinds 0/1)
    theta_c: float = 2.5e-2      # snow: critical compression
    theta_s: float = 7.5e-3      # snow: critical stretch
    hardening: float = 10.0      # snow: xi
    friction_angle: float = 30.0  # sand: degrees

    def __post_init__(self):
        self.kind = MaterialKind(int(self.kind))
        if not (self.density > 0.0):
            raise RejectedInputError(f"density must be positive, got {self.density}")
        if self.kind == MaterialKind.WEAKLY_COMPRESSIBLE_FLUID and not (self.bulk_modulus > 0.0):
            raise RejectedInputError(
                f"fluid bulk modulus must be positive, got {self.bulk_modulus}")
        if self.kind != MaterialKind.WEAKLY_COMPRESSIBLE_FLUID and (self.mu < 0.0 or self.lam < 0.0):
            raise RejectedInputError(
                f"elastic moduli must be nonnegative, got mu={self.mu} lam={self.lam}")

    def sound_speed(self) -> float:
        if self.kind == MaterialKind.WEAKLY_COMPRESSIBLE_FLUID:
            return float(math.sqrt(self.gamma * self.bulk_modulus / self.density))
        return float(math.sqrt((self.lam + 2.0 * self.mu) / self.density))

    @staticmethod
    def fluid(density, bulk_modulus, gamma=7.0, clamp_tension=False) -> "Material":
        return Material(MaterialKind.WEAKLY_COMPRESSIBLE_FLUID, density,
                        bulk_modulus=bulk_modulus, gamma=gamma, clamp_tension=clamp_tension)

    @staticmethod
    def _lame(young, poisson):
        mu = young / (2.0 * (1.0 + poisson))
        lam = young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson))
        return mu, lam

    @staticmethod
    def fixed_corotated(density, young, poisson) -> "Material":
        mu, lam = Material._lame(young, poisson)
        return Material(MaterialKind.FIXED_COROTATED, density, mu=mu, lam=lam)

    @staticmethod
    def snow(density, young, poisson, theta_c=2.5e-2, theta_s=7.5e-3, hardening=10.0) -> "Material":
        mu, lam = Material._lame(young, poisson)
        return Material(MaterialKind.SNOW, density, mu=mu, lam=lam, theta_c=theta_c,
                        theta_s=theta_s, hardening=hardening)

    @staticmethod
    def sand(density, young, poisson, friction_angle=30.0) -> "Material":
        mu, lam = Material._lame(young, poisson)
        return Material(MaterialKind.SAND, density, mu=mu, lam=lam,
                        friction_angle=friction_angle)


_SPEED_EPS = 1e-12


def cfl_dt(max_speed: float, params: SimParams, frame_remaining: float) -> float:
    """Step size with per-step travel below cfl*dx, never beyond the frame remainder."""
    if max_speed < 0.0 or not math.isfinite(max_speed):
        raise RejectedInputError(f"max_speed must be finite and >= 0, got {max_speed}")
    dt = params.cfl * params.dx / max(max_speed, _SPEED_EPS)
    return min(frame_remaining, dt)
