"""The BASELINE.json workloads as scenes, with the conventions the
reference leaves open fixed here (recorded in DESIGN.md section 2):

config 1  coefficient queries: N = 2^20 from numpy default_rng(0), order
          p ~ U[-1,1]^3, wo = normalize(N(0,I)), wi likewise, u ~ U[0,1)^2,
          all cast to float32; plane field f = p_z; GENERALIZED,
          sigma = 0.05, alpha = sqrt(2)*0.05/0.1 on all axes, R = 0.5, F == 1.
config 2  plane z=0, sigma 0.05, l = 0.05 (alpha = sqrt 2, generalized),
          albedo 0.8, orthographic camera travelling (cos45, 0, -sin45),
          to-light (cos30, 0, sin30) with unit irradiance, black
          environment, 256^2 x 64 spp, depth 16, seed 1.
config 3  unit sphere, sigma 0.1, l = 0.05 (alpha = 2.828), albedo 0.9,
          pinhole 40 deg at (0,-4,0) looking at the origin, 512^2 x 256 spp,
          depth 32, point light I = 10 at (3,3,3), environment 0.1, seed 2.
config 4  3x3 planar panels sigma in {0.01, 0.05, 0.2} x l_z in {0.02, 0.1,
          inf (BECKMANN)}, l_xy = 0.05, otherwise config 2's scene at
          1024^2 x 1024 spp, depth 64.
"""

from __future__ import annotations

import math

import numpy as np

from .medium import MacrofacetMedium
from .ndf import KernelParams, NdfKind, RoughnessTriple, roughness_from_kernel
from .scene import Camera, DirectionalLight, Environment, PointLight, ShellPrimitive, ShellScene
from .sdf import Plane, Sphere

SQRT2 = math.sqrt(2.0)


def config1_medium():
    a = SQRT2 * 0.05 / 0.1
    return MacrofacetMedium(kind=NdfKind.GENERALIZED, a3=RoughnessTriple(a, a, a), sigma=0.05,
                            mix_ratio=0.5, fresnel_one=True)


def config1_inputs(n=1 << 20, seed=0):
    """(p, wo, wi, u) float32 arrays of shapes (n,3), (n,3), (n,3), (n,2)."""
    rs = np.random.default_rng(seed)
    p = rs.uniform(-1.0, 1.0, (n, 3))
    wo = rs.normal(size=(n, 3))
    wo /= np.linalg.norm(wo, axis=-1, keepdims=True)
    wi = rs.normal(size=(n, 3))
    wi /= np.linalg.norm(wi, axis=-1, keepdims=True)
    u = rs.uniform(0.0, 1.0, (n, 2))
    return tuple(a.astype(np.float32) for a in (p, wo, wi, u))


def planar_medium(sigma, l_xy, l_z, albedo):
    if math.isinf(l_z):
        a = SQRT2 * sigma / l_xy
        return MacrofacetMedium(kind=NdfKind.BECKMANN, a3=RoughnessTriple(a, a, 0.0),
                                sigma=sigma, albedo=albedo)
    a3 = roughness_from_kernel(KernelParams(sigma, l_xy, l_xy, l_z))
    return MacrofacetMedium(kind=NdfKind.GENERALIZED, a3=a3, sigma=sigma, albedo=albedo)


CAM_TRAVEL_C2 = (math.cos(math.radians(45.0)), 0.0, -math.sin(math.radians(45.0)))
TO_LIGHT_C2 = (math.cos(math.radians(30.0)), 0.0, math.sin(math.radians(30.0)))


def planar_scene(medium, width, height, elevation_deg=45.0, light_elev_deg=30.0,
                 film_height=1.0):
    e = math.radians(elevation_deg)
    travel = (math.cos(e), 0.0, -math.sin(e))
    # film centre 5 units back along the view axis: every ray starts well
    # above the thickest shell of the sweep (3 sigma <= 0.6)
    pos = (-5.0 * travel[0], 0.0, -5.0 * travel[2])
    cam = Camera(position=pos, look_at=(0.0, 0.0, 0.0), fov_deg=40.0, width=width,
                 height=height, ortho=True, film_height=film_height)
    le = math.radians(light_elev_deg)
    to_light = (math.cos(le), 0.0, math.sin(le))
    sun = DirectionalLight(direction=tuple(-v for v in to_light), radiance=(1.0, 1.0, 1.0))
    return ShellScene(primitives=(ShellPrimitive(Plane(0.0), medium),), camera=cam,
                      environment=Environment(radiance=(0.0, 0.0, 0.0)), sun=sun)


def config2_scene(width=256, height=256):
    return planar_scene(planar_medium(0.05, 0.05, 0.05, 0.8), width, height)


CONFIG2 = dict(spp=64, max_bounces=16, seed=1)


def config3_scene(width=512, height=512):
    a = SQRT2 * 0.1 / 0.05
    med = MacrofacetMedium(kind=NdfKind.GENERALIZED, a3=RoughnessTriple(a, a, a), sigma=0.1,
                           albedo=0.9)
    cam = Camera(position=(0.0, -4.0, 0.0), look_at=(0.0, 0.0, 0.0), fov_deg=40.0, width=width,
                 height=height)
    return ShellScene(primitives=(ShellPrimitive(Sphere((0.0, 0.0, 0.0), 1.0), med),), camera=cam,
                      environment=Environment(radiance=(0.1, 0.1, 0.1)),
                      point=PointLight(position=(3.0, 3.0, 3.0), intensity=10.0))


CONFIG3 = dict(spp=256, max_bounces=32, seed=2)

CONFIG4_SIGMAS = (0.01, 0.05, 0.2)
CONFIG4_LZ = (0.02, 0.1, math.inf)


def config4_scene(sigma, l_z, width=1024, height=1024):
    return planar_scene(planar_medium(sigma, 0.05, l_z, 0.8), width, height)


CONFIG4 = dict(spp=1024, max_bounces=64, seed=3)


def config5_scene(width=2048, height=2048, n_sdf=256, n_sigma=128, seed=4):
    """Heterogeneous GP field (config 5): union of 16 spheres + torus as a
    trilinear SDF grid, value-noise sigma grid, l_xy = 0.03, l_z = 0.08,
    albedo 0.85.  Camera and lights are not given by BASELINE.json; recorded
    convention: pinhole 40 deg at (0, -4, 1.2) looking at the origin,
    directional light travelling (-1, 1, -2)/|.| with irradiance 2, and a
    constant environment 0.2."""
    from .grid import GridMedium, config5_fields

    sdf, sigma = config5_fields(seed=seed, n_sdf=n_sdf, n_sigma=n_sigma)
    med = GridMedium(sigma=sigma, l_xy=0.03, l_z=0.08, albedo=0.85)
    cam = Camera(position=(0.0, -4.0, 1.2), look_at=(0.0, 0.0, 0.0), fov_deg=40.0, width=width,
                 height=height)
    return ShellScene(primitives=(ShellPrimitive(sdf, med),), camera=cam,
                      environment=Environment(radiance=(0.2, 0.2, 0.2)),
                      sun=DirectionalLight(direction=(-1.0, 1.0, -2.0), radiance=(2.0, 2.0, 2.0)))


CONFIG5 = dict(spp=4096, max_bounces=64, seed=4)
