"""Renderable world: shells, camera and lights (reference scene.py:19-129).

Extensions the BASELINE configs need (not in the reference, recorded in
DESIGN.md): an orthographic camera (`Camera(..., ortho=True,
film_height=...)`), a point light (`PointLight`, NEE weight I / r^2) and a
constant grey albedo on the medium.  Scenes are immutable; `to_c_scene`
flattens one into the C-ABI struct uploaded by value with every launch.

Drop-in rule: `to_c_scene` reads scenes by attribute and dispatches shapes
on their class NAME, so a scene built from the reference package's own
classes (macrofacet.ShellScene / ShellPrimitive / Plane / Sphere / Box /
MacrofacetMedium / Camera / Environment / DirectionalLight) renders on the
device unchanged; the BASELINE extensions are read with getattr defaults."""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .errors import ConfigError, UnsupportedGeometryError
from .medium import MacrofacetMedium, to_c_medium
from .sdf import shape_name, surface_distance


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
    """Environment light (scene.py:54-84): constant radiance, or a
    latitude-longitude map (H, W, 3), theta down the rows, evaluated
    bilinearly on the device when a path escapes."""

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

        if any(type(p.sdf) is GridSDF for p in prims):
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


# device copies of lat-long maps, keyed by (device, id(array)); the entry
# holds the array so the id cannot be reused while it is cached
_ENV_MAPS: dict = {}


def _env_map(img):
    """Upload (once per device) a lat-long map as float32 (H, W, 3)."""
    torch = _lib.require_cuda()
    dev = torch.cuda.current_device()
    key = (dev, id(img))
    hit = _ENV_MAPS.get(key)
    if hit is not None and hit[0] is img:
        return hit[1]
    a = np.ascontiguousarray(np.asarray(img, dtype=np.float32))
    if a.ndim != 3 or a.shape[2] != 3 or a.shape[0] < 1 or a.shape[1] < 1:
        raise UnsupportedGeometryError("lat-long environment must be an (H, W, 3) array")
    if len(_ENV_MAPS) > 64:
        _ENV_MAPS.clear()
    t = torch.from_numpy(a).to(torch.device("cuda", dev))
    _ENV_MAPS[key] = (img, t)
    return t


def _vec3(v, name):
    v = tuple(float(x) for x in np.broadcast_to(np.asarray(v, dtype=np.float64), (3,)))
    if not all(np.isfinite(v)):
        raise ConfigError(f"{name} must be finite")
    return v


def to_c_scene(scene) -> _lib.MfScene:
    """Flatten a scene (this package's or the reference's) into the C ABI."""
    prims = tuple(scene.primitives)
    if len(prims) > _lib.MF_MAX_PRIMS:
        raise UnsupportedGeometryError(f"at most {_lib.MF_MAX_PRIMS} primitives")
    c = _lib.MfScene()
    c.n_prims = len(prims)
    c.n_media = len(prims)
    from .grid import GridSDF, fill_scene_grid

    for j, pr in enumerate(prims):
        cp = c.prims[j]
        if type(pr.sdf) is GridSDF:
            fill_scene_grid(c, j, pr.sdf, pr.medium)
            continue
        name = shape_name(pr.sdf)
        if name == "Plane":
            cp.shape = _lib.SHAPE_PLANE
            cp.z0 = float(pr.sdf.z0)
        elif name == "Sphere":
            cp.shape = _lib.SHAPE_SPHERE
            cp.center[:] = _vec3(pr.sdf.center, "sphere center")
            cp.radius = float(pr.sdf.radius)
        elif name == "Box":
            cp.shape = _lib.SHAPE_BOX
            cp.center[:] = _vec3(pr.sdf.center, "box center")
            cp.half_extents[:] = _vec3(pr.sdf.half_extents, "box half extents")
        else:
            raise UnsupportedGeometryError(
                f"unknown SDF primitive {type(pr.sdf).__module__}.{name} (the device traces "
                "Plane, Sphere, Box and GridSDF)")
        cp.medium = j
        c.media[j] = to_c_medium(pr.medium)
    cam = scene.camera
    c.camera.ortho = 1 if getattr(cam, "ortho", False) else 0
    c.camera.width, c.camera.height = int(cam.width), int(cam.height)
    c.camera.position[:] = _vec3(cam.position, "camera position")
    c.camera.look_at[:] = _vec3(cam.look_at, "camera look_at")
    c.camera.fov_deg = float(cam.fov_deg)
    c.camera.film_height = float(getattr(cam, "film_height", 1.0))
    env = scene.environment
    c.env[:] = _vec3(env.radiance, "environment radiance")
    latlong = getattr(env, "latlong", None)
    if latlong is not None:
        t = _env_map(latlong)
        c.d_env_map = t.data_ptr()
        c.env_height, c.env_width = int(t.shape[0]), int(t.shape[1])
    sun = getattr(scene, "sun", None)
    if sun is not None:
        c.has_sun = 1
        c.sun_dir[:] = _vec3(sun.direction, "sun direction")
        c.sun_radiance[:] = _vec3(sun.radiance, "sun radiance")
    point = getattr(scene, "point", None)
    if point is not None:
        c.has_point = 1
        c.point_pos[:] = _vec3(point.position, "point light position")
        c.point_intensity[:] = _vec3(point.intensity, "point light intensity")
    return c


def shell_intersect(origin, direction, scene, t_max=1e6):
    """Ordered disjoint ray intervals inside the primitives' 3-sigma shells
    and whether the ray reaches below a shell (scene.py:132-200): sphere
    tracing of min_k |f_k| - w_k with the 1-Lipschitz step, every boundary
    bisected 60 times, the march ended once the ray is outside every shell
    and receding from every (convex-exterior) primitive.  Host float64
    geometry query on the callers' SDF objects; the device walkers use
    their own exact level-set distances.  Returns ([(t_in, t_out, k)],
    deep)."""
    from .errors import NumericFailureError

    o = np.asarray(origin, dtype=np.float64)
    d = np.asarray(direction, dtype=np.float64)
    prims = scene.primitives
    if not prims:
        return [], False
    w = np.array([pr.medium.shell_half_width for pr in prims])

    def fields(t):
        p = o + t * d
        return np.array([float(pr.sdf.sdf(p)) for pr in prims])

    def gap(t):                         # signed distance to the nearest shell, its index
        f = fields(t)
        g = np.abs(f) - w
        k = int(np.argmin(g))
        return f, float(g[k]), k

    def crossing(lo, hi, k):            # the boundary of shell k on [lo, hi]
        pr, wk = prims[k], w[k]
        g = lambda t: abs(float(pr.sdf.sdf(o + t * d))) - wk  # noqa: E731
        out_lo = g(lo) > 0.0
        for _ in range(60):
            mid = 0.5 * (lo + hi)
            if (g(mid) > 0.0) == out_lo:
                lo = mid
            else:
                hi = mid
        return 0.5 * (lo + hi)

    eps = 1e-7 * max(1.0, float(np.linalg.norm(o)))
    f, g, k = gap(0.0)
    deep = bool(np.any(f < -w))
    cur = k if g <= 0.0 else None        # the shell the ray is in, if any
    spans = [[0.0, None, cur]] if cur is not None else []
    t_prev, t = 0.0, max(abs(g), eps)
    for _ in range(1_000_000):
        if t >= t_max:
            break
        f, g, k = gap(t)
        deep = deep or bool(np.any(f < -w))
        if cur is None and g <= 0.0:
            spans.append([crossing(t_prev, t, k), None, k])
            cur = k
        elif cur is not None and g > 0.0:
            spans[-1][1] = crossing(t_prev, t, cur)
            cur = None
        if cur is None and g > 0.0:
            p = o + t * d
            if all(float(np.dot(pr.sdf.gradient(p), d)) >= 0.0 for pr in prims):
                break                    # receding from every convex exterior
        t_prev, t = t, t + max(abs(g), eps)
    else:
        raise NumericFailureError("shell_intersect exceeded its iteration cap")
    if spans and spans[-1][1] is None:
        spans[-1][1] = min(t, t_max)
    return [tuple(s) for s in spans], deep
