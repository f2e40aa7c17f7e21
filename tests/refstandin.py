"""Reference-shaped stand-ins for the drop-in tests.

The GPU box has no /root/reference, so the tests that check that scenes
built from the reference package's own classes render unchanged use these
look-alikes: frozen dataclasses with the reference's CLASS NAMES and field
names (scene.py:19-129, sdf.py:18-84, medium.py:35-67, ndf.py:34-72) and
none of this package's types.  Where the reference itself is importable
(the build container), tests/test_api_cpu.py also runs the real classes."""

from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np


class NdfKind(enum.Enum):
    BECKMANN = "beckmann"
    GGX = "ggx"
    GENERALIZED = "generalized"


@dataclass(frozen=True)
class RoughnessTriple:
    ax: float
    ay: float
    az: float = 0.0


@dataclass(frozen=True)
class MacrofacetMedium:
    kind: NdfKind
    a3: RoughnessTriple
    sigma: float
    fresnel_eta: tuple = (0.2, 0.92, 1.1)
    fresnel_k: tuple = (3.9, 2.45, 2.14)
    mix_ratio: float = 0.5
    fresnel_one: bool = False


@dataclass(frozen=True)
class Plane:
    z0: float = 0.0


@dataclass(frozen=True)
class Sphere:
    center: tuple
    radius: float


@dataclass(frozen=True)
class Box:
    center: tuple
    half_extents: tuple


@dataclass(frozen=True)
class Camera:
    position: tuple
    look_at: tuple
    fov_deg: float
    width: int
    height: int


@dataclass(frozen=True)
class Environment:
    radiance: tuple = (1.0, 1.0, 1.0)
    latlong: Optional[np.ndarray] = None


@dataclass(frozen=True)
class DirectionalLight:
    direction: tuple
    radiance: tuple

    def __post_init__(self):
        # the reference normalises the travel direction (scene.py:91-94)
        d = np.asarray(self.direction, dtype=np.float64)
        object.__setattr__(self, "direction", tuple(float(x) for x in d / np.linalg.norm(d)))


@dataclass(frozen=True)
class ShellPrimitive:
    sdf: object
    medium: MacrofacetMedium


@dataclass(frozen=True)
class ShellScene:
    primitives: tuple
    camera: Camera
    environment: Environment = field(default_factory=Environment)
    sun: Optional[DirectionalLight] = None
