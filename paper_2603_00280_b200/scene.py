"""Renderable world: shells, camera and lights (reference scene.py:19-129).

Extensions the BASELINE configs need (not in the reference, recorded in
DESIGN.md): an orthographic camera (`Camera(..., ortho=True,
film_height=...)`), a point light (`PointLight`, NEE weight I / r^2) and a
constant grey albedo on the medium.  Scenes are immutable; `to_c_scene`
flattens one into the C-ABI struct uploaded by value with every launch."""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .errors import ConfigError, UnsupportedGeometryError
from .medium import MacrofacetMedium, to_c_medium
from .sdf import Plane, Sphere, surface_distance


@dataclass(frozen=True)
class Camera:
    """Pinhole camera (scene.py:19-51); `ortho=True` gives parallel rays
    along look_at - position through a film `film_height` world units tall
    centred on `position`."""

    position: tuple
    look_at: tuple
    fov_deg: float
    width: int
    height: int
    ortho: bool = False
    film_height: float = 1.0


@dataclass(frozen=True)
class Environment:
    """Constant environment radiance (scene.py:54-84).  Lat-long maps are
    not supported on the device path."""

    radiance: tuple = (1.0, 1.0, 1.0)
    latlong: Optional[np.ndarray] = None


@dataclass(frozen=True)
class DirectionalLight:
    """Delta light; `direction` is the travel direction, `radiance` acts as
    irradiance (scene.py:87-96)."""

    direction: tuple
    radiance: tuple

    def __post_init__(self):
        d = np.asarray(self.direction, dtype=np.float64)
        d = d / np.linalg.norm(d)
        object.__setattr__(self, "direction", tuple(float(x) for x in d))
        object.__setattr__(self, "radiance", tuple(float(x) for x in self.radiance))


@dataclass(frozen=True)
class PointLight:
    """Isotropic point light of radiant intensity `intensity` (W/sr per
    channel); NEE contributes I / r^2 (BASELINE config 3 extension)."""

    position: tuple
    intensity: tuple

    def __post_init__(self):
        inten = self.intensity
        if np.isscalar(inten):
            inten = (inten, inten, inten)
        object.__setattr__(self, "position", tuple(float(x) for x in self.position))
        object.__setattr__(self, "intensity", tuple(float(x) for x in inten))


@dataclass(frozen=True)
class ShellPrimitive:
    sdf: object  # Plane | Sphere
    medium: MacrofacetMedium


@dataclass(frozen=True)
class ShellScene:
    """Primitives with bound media, camera and lights; shells of distinct
    primitives must not overlap (scene.py:104-129)."""

    primitives: tuple
    camera: Camera
    environment: Environment = field(default_factory=Environment)
    sun: Optional[DirectionalLight] = None
    point: Optional[PointLight] = None

    def __post_init__(self):
        object.__setattr__(self, "primitives", tuple(self.primitives))
        prims = self.primitives
        from .grid import GridSDF

        if any(isinstance(p.sdf, GridSDF) for p in prims):
            if len(prims) != 1:
                raise ConfigError("a grid field must be the scene's only primitive")
            return
        for i in range(len(prims)):
            for j in range(i + 1, len(prims)):
                gap = surface_distance(prims[i].sdf, prims[j].sdf)
                need = prims[i].medium.shell_half_width + prims[j].medium.shell_half_width
                if gap <= need:
                    raise ConfigError(
                        f"shells of primitives {i} and {j} overlap: surface gap "
                        f"{gap:.6g} <= combined half-widths {need:.6g}")


def to_c_scene(scene: ShellScene) -> _lib.MfScene:
    if len(scene.primitives) > _lib.MF_MAX_PRIMS:
        raise UnsupportedGeometryError(f"at most {_lib.MF_MAX_PRIMS} primitives")
    if scene.environment.latlong is not None:
        raise UnsupportedGeometryError("lat-long environments are not supported on the device")
    c = _lib.MfScene()
    c.n_prims = len(scene.primitives)
    c.n_media = len(scene.primitives)
    from .grid import GridSDF, fill_scene_grid

    for j, pr in enumerate(scene.primitives):
        cp = c.prims[j]
        if isinstance(pr.sdf, GridSDF):
            fill_scene_grid(c, j, pr.sdf, pr.medium)
            continue
        if isinstance(pr.sdf, Plane):
            cp.shape = _lib.SHAPE_PLANE
            cp.z0 = float(pr.sdf.z0)
        elif isinstance(pr.sdf, Sphere):
            cp.shape = _lib.SHAPE_SPHERE
            cp.center[:] = pr.sdf.center
            cp.radius = float(pr.sdf.radius)
        else:
            raise UnsupportedGeometryError(
                f"{type(pr.sdf).__name__} shells are not supported on the device")
        cp.medium = j
        c.media[j] = to_c_medium(pr.medium)
    cam = scene.camera
    c.camera.ortho = 1 if cam.ortho else 0
    c.camera.width, c.camera.height = int(cam.width), int(cam.height)
    c.camera.position[:] = tuple(float(v) for v in cam.position)
    c.camera.look_at[:] = tuple(float(v) for v in cam.look_at)
    c.camera.fov_deg = float(cam.fov_deg)
    c.camera.film_height = float(cam.film_height)
    c.env[:] = tuple(float(v) for v in scene.environment.radiance)
    if scene.sun is not None:
        c.has_sun = 1
        c.sun_dir[:] = scene.sun.direction
        c.sun_radiance[:] = scene.sun.radiance
    if scene.point is not None:
        c.has_point = 1
        c.point_pos[:] = scene.point.position
        c.point_intensity[:] = scene.point.intensity
    return c
