"""Analytic SDF primitives bound to shells (reference sdf.py:18-84).

Plane, Sphere and Box are what the device kernels trace (exact 1-Lipschitz
fields; exact level-set distances for planes and spheres, the Lipschitz
bound plus the recede test for boxes, transport.py:70-108); their SDF /
gradient are evaluated on the GPU inside the walker.  `surface_distance` is
the construction-time overlap check of ShellScene (sdf.py:87-122).

Every function here dispatches on the class NAME, so the reference's own
Plane / Sphere / Box objects work as well as these (the drop-in rule)."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

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


@dataclass(frozen=True)
class Box:
    """Axis-aligned box (sdf.py:55-84): exact signed distance, convex exterior."""

    center: tuple
    half_extents: tuple

    def __post_init__(self):
        if any(not h > 0 for h in self.half_extents):
            raise ParameterDomainError("box half extents must be > 0")
        object.__setattr__(self, "center", tuple(float(c) for c in self.center))
        object.__setattr__(self, "half_extents", tuple(float(h) for h in self.half_extents))


def shape_name(sdf) -> str:
    return type(sdf).__name__


def box_sdf(box, p):
    """Signed distance to a box (host helper for the overlap check)."""
    q = np.abs(np.asarray(p, dtype=np.float64) - np.asarray(box.center)) - \
        np.asarray(box.half_extents)
    return float(np.linalg.norm(np.maximum(q, 0.0)) + min(float(np.max(q)), 0.0))


def _box_box(a, b):
    ca, cb = np.asarray(a.center), np.asarray(b.center)
    ha, hb = np.asarray(a.half_extents), np.asarray(b.half_extents)
    sep = np.maximum(np.abs(ca - cb) - (ha + hb), 0.0)
    if np.any(sep > 0.0):
        return float(np.linalg.norm(sep))           # disjoint volumes
    inside_ab = np.all(np.abs(cb - ca) + hb <= ha)
    inside_ba = np.all(np.abs(ca - cb) + ha <= hb)
    if not (inside_ab or inside_ba):
        return 0.0                                  # the surfaces cross
    # nested: the nearest points are on facing (parallel) faces
    return float(np.min(np.minimum(np.abs((ca + ha) - (cb + hb)), np.abs((ca - ha) - (cb - hb)))))


def surface_distance(a, b):
    """Distance between the zero level sets of two primitives (exact for
    every pair of plane / sphere / axis-aligned box)."""
    na, nb = shape_name(a), shape_name(b)
    if na > nb:
        a, b, na, nb = b, a, nb, na
    if na == "Plane" and nb == "Plane":
        return abs(a.z0 - b.z0)
    if na == "Plane" and nb == "Sphere":
        return max(0.0, abs(b.center[2] - a.z0) - b.radius)
    if na == "Box" and nb == "Plane":
        lo, hi = a.center[2] - a.half_extents[2], a.center[2] + a.half_extents[2]
        return 0.0 if lo <= b.z0 <= hi else min(abs(b.z0 - lo), abs(b.z0 - hi))
    if na == "Sphere" and nb == "Sphere":
        return max(0.0, math.dist(a.center, b.center) - a.radius - b.radius)
    if na == "Box" and nb == "Sphere":
        return max(0.0, abs(box_sdf(a, b.center)) - b.radius)
    if na == "Box" and nb == "Box":
        return _box_box(a, b)
    raise ParameterDomainError(f"no surface distance for {na} / {nb}")
