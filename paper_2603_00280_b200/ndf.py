"""Roughness parameter types (reference ndf.py:34-78).

Only the host-side parameter objects live here; every NDF / projected-area /
vNDF evaluation on the hot path runs in the CUDA kernels
(csrc/mf_math.cuh)."""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass

from .errors import ParameterDomainError


@dataclass(frozen=True)
class KernelParams:
    """Squared-exponential kernel: field std-dev and correlation lengths
    (ndf.py:34-48)."""

    sigma: float
    lx: float
    ly: float
    lz: float

    def __post_init__(self):
        for name in ("sigma", "lx", "ly", "lz"):
            v = getattr(self, name)
            if not (math.isfinite(v) and v > 0.0):
                raise ParameterDomainError(f"KernelParams.{name} must be finite and > 0, got {v}")


@dataclass(frozen=True)
class RoughnessTriple:
    """Per-axis slope roughness; az = 0 is the height-field limit (ndf.py:51-66)."""

    ax: float
    ay: float
    az: float = 0.0

    def __post_init__(self):
        if not (math.isfinite(self.ax) and self.ax > 0.0):
            raise ParameterDomainError(f"ax must be finite and > 0, got {self.ax}")
        if not (math.isfinite(self.ay) and self.ay > 0.0):
            raise ParameterDomainError(f"ay must be finite and > 0, got {self.ay}")
        if not (math.isfinite(self.az) and self.az >= 0.0):
            raise ParameterDomainError(f"az must be finite and >= 0, got {self.az}")


class NdfKind(enum.Enum):
    BECKMANN = "beckmann"
    GGX = "ggx"
    GENERALIZED = "generalized"


def roughness_from_kernel(kernel: KernelParams) -> RoughnessTriple:
    """alpha_i = sqrt(2) sigma / l_i (ndf.py:75-78); l_z = inf gives az = 0."""
    s = math.sqrt(2.0) * kernel.sigma
    return RoughnessTriple(s / kernel.lx, s / kernel.ly, s / kernel.lz)
