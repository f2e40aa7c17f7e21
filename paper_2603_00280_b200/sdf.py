"""Analytic SDF primitives bound to shells (reference sdf.py:18-52).

Plane and Sphere are what the device kernels trace (exact 1-Lipschitz
fields with exact level-set distances); their SDF / gradient are evaluated
on the GPU inside the walker.  `surface_distance` is the construction-time
overlap check of ShellScene (sdf.py:87-122)."""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import ParameterDomainError


@dataclass(frozen=True)
class Plane:
    """Horizontal plane z = z0, outside is above."""

    z0: float = 0.0


@dataclass(frozen=True)
class Sphere:
    center: tuple
    radius: float

    def __post_init__(self):
        if not self.radius > 0:
            raise ParameterDomainError(f"sphere radius must be > 0, got {self.radius}")
        object.__setattr__(self, "center", tuple(float(c) for c in self.center))


def surface_distance(a, b):
    """Distance between the zero level sets of two primitives (exact for the
    plane / sphere pairs, sdf.py:101-116)."""
    if isinstance(a, Plane) and isinstance(b, Plane):
        return abs(a.z0 - b.z0)
    if isinstance(a, Sphere) and isinstance(b, Plane):
        a, b = b, a
    if isinstance(a, Plane) and isinstance(b, Sphere):
        return max(0.0, abs(b.center[2] - a.z0) - b.radius)
    gap = math.dist(a.center, b.center)
    return max(0.0, gap - a.radius - b.radius)
