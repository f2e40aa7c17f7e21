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

    # host evaluation of the field for callers (sdf.py:25-33); the walkers
    # evaluate it on the device
    def sdf(self, p):
        return np.asarray(p, dtype=np.float64)[..., 2] - self.z0

    def gradient(self, p):
        g = np.zeros(np.shape(p))
        g[..., 2] = 1.0
        return g


@dataclass(frozen=True)
class Sphere:
    center: tuple
    radius: float

    def __post_init__(self):
        if not self.radius > 0:
            raise ParameterDomainError(f"sphere radius must be > 0, got {self.radius}")
        object.__setattr__(self, "center", tuple(float(c) for c in self.center))

    def sdf(self, p):
        """|p - c| - r (sdf.py:45-47)."""
        return np.linalg.norm(np.asarray(p, dtype=np.float64) - self.center, axis=-1) - self.radius

    def gradient(self, p):
        """Outward unit radial direction (the +z axis at the centre)."""
        d = np.asarray(p, dtype=np.float64) - self.center
        r = np.linalg.norm(d, axis=-1, keepdims=True)
        return np.where(r > 0.0, d / np.where(r > 0.0, r, 1.0), np.array([0.0, 0.0, 1.0]))


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

    def sdf(self, p):
        """Exact signed distance (sdf.py:66-72): the length of the positive
        part of q = |p - c| - h plus the (non-positive) largest component."""
        q = np.abs(np.asarray(p, dtype=np.float64) - self.center) - np.asarray(self.half_extents)
        return np.linalg.norm(np.maximum(q, 0.0), axis=-1) + np.minimum(q.max(axis=-1), 0.0)

    def gradient(self, p):
        """Gradient a.e. (sdf.py:74-84): outside, along the positive part of
        q with the octant's signs; inside, the normal of the nearest face."""
        d = np.asarray(p, dtype=np.float64) - self.center
        q = np.abs(d) - np.asarray(self.half_extents)
        sgn = np.where(d >= 0.0, 1.0, -1.0)
        pos = np.maximum(q, 0.0)
        n = np.linalg.norm(pos, axis=-1, keepdims=True)
        inside = np.eye(3)[np.argmax(q, axis=-1)] * sgn
        return np.where(n > 0.0, sgn * pos / np.where(n > 0.0, n, 1.0), inside)


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
