"""Heterogeneous GP fields (BASELINE config 5; not in the reference).

`GridSDF` is a trilinearly interpolated signed-distance grid (the GP mean)
and `GridMedium` the per-voxel field std-dev grid with anisotropic kernel
lengths (alpha = sqrt2 sigma(p) / l).  They form one `ShellPrimitive`; the
device path (csrc/mf_grid.cuh) tracks rays through a majorant grid built
on the GPU by `mf_grid_majorant`.  Grids are float32 numpy arrays indexed
[ix, iy, iz], vertex-centred over `bounds`; they are uploaded once per
device and cached on the object.

`config5_fields` builds the BASELINE config-5 inputs: a seeded union of 16
spheres (radii U[0.1, 0.3], centres U[-0.7, 0.7]^3) and a torus (R = 0.6,
r = 0.15, axis z) as a 256^3 SDF, and 128^3 smooth value noise in
[0.01, 0.2] as sigma.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ParameterDomainError
from .medium import DEFAULT_ETA, DEFAULT_K


@dataclass(eq=False)
class GridSDF:
    values: np.ndarray                       # (n, n, n) float32 signed distance
    bounds: tuple = ((-1.6, -1.6, -1.6), (1.6, 1.6, 1.6))
    _dev: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        v = np.ascontiguousarray(self.values, dtype=np.float32)
        if v.ndim != 3 or len(set(v.shape)) != 1 or v.shape[0] < 2:
            raise ParameterDomainError("GridSDF.values must be a cubic (n, n, n) array, n >= 2")
        self.values = v


@dataclass(eq=False)
class GridMedium:
    """Per-voxel field std-dev `sigma` with kernel lengths l_xy, l_z; the
    remaining fields mirror MacrofacetMedium (medium.py:35-67)."""

    sigma: np.ndarray                        # (m, m, m) float32, > 0
    l_xy: float
    l_z: float
    albedo: tuple | None = None
    mix_ratio: float = 0.5
    fresnel_one: bool = False
    fresnel_eta: tuple = DEFAULT_ETA
    fresnel_k: tuple = DEFAULT_K
    majorant_res: int = 64

    def __post_init__(self):
        s = np.ascontiguousarray(self.sigma, dtype=np.float32)
        if s.ndim != 3 or len(set(s.shape)) != 1 or s.shape[0] < 2:
            raise ParameterDomainError("GridMedium.sigma must be a cubic (m, m, m) array, m >= 2")
        if not np.all(s > 0):
            raise ParameterDomainError("GridMedium.sigma must be > 0 everywhere")
        self.sigma = s
        if not (self.l_xy > 0 and self.l_z > 0):
            raise ParameterDomainError("kernel lengths must be > 0")
        if self.albedo is not None and np.isscalar(self.albedo):
            self.albedo = (float(self.albedo),) * 3

    @property
    def shell_half_width(self):
        return 3.0 * float(self.sigma.max())


def _device_tensors(sdf: GridSDF, med: GridMedium):
    """Upload (once per device) and build the majorant grid."""
    torch = _lib.require_cuda()
    dev = torch.cuda.current_device()
    key = (dev, id(med))
    if key in sdf._dev:
        return sdf._dev[key]
    lib = _lib.load()
    d = torch.device("cuda", dev)
    t_sdf = torch.from_numpy(sdf.values).to(d)
    t_sig = torch.from_numpy(med.sigma).to(d)
    n_maj = int(med.majorant_res)
    t_maj = torch.empty(n_maj ** 3, dtype=torch.float32, device=d)
    g = grid_struct(sdf, med, t_sdf, t_sig, t_maj)
    _lib.check(lib.mf_grid_majorant(ctypes.byref(g), ctypes.c_void_p(t_maj.data_ptr()),
                                    _lib.stream_handle(torch, d)))
    sdf._dev[key] = (t_sdf, t_sig, t_maj)
    return sdf._dev[key]


def grid_struct(sdf, med, t_sdf, t_sig, t_maj):
    g = _lib.MfGridField()
    g.d_sdf = t_sdf.data_ptr()
    g.d_sigma = t_sig.data_ptr()
    g.d_majorant = t_maj.data_ptr()
    g.n_sdf = sdf.values.shape[0]
    g.n_sigma = med.sigma.shape[0]
    g.n_maj = int(med.majorant_res)
    g.bmin[:] = tuple(float(v) for v in sdf.bounds[0])
    g.bmax[:] = tuple(float(v) for v in sdf.bounds[1])
    g.l_xy = float(med.l_xy)
    g.l_z = float(med.l_z)
    return g


def fill_scene_grid(c_scene, prim_index, sdf: GridSDF, med: GridMedium):
    """Set the C scene's grid field for primitive `prim_index` (device upload)."""
    t_sdf, t_sig, t_maj = _device_tensors(sdf, med)
    c_scene.has_grid = 1
    c_scene.grid = grid_struct(sdf, med, t_sdf, t_sig, t_maj)
    cp = c_scene.prims[prim_index]
    cp.shape = _lib.SHAPE_GRID
    cp.medium = prim_index
    cm = c_scene.media[prim_index]
    cm.kind = _lib.KIND["generalized"]
    cm.ax = cm.ay = cm.az = 1.0          # placeholders: alpha comes from sigma(p)
    cm.sigma = 1.0
    cm.mix_ratio = float(med.mix_ratio)
    if med.albedo is not None:
        cm.fresnel = _lib.FRESNEL_ALBEDO
        cm.albedo[:] = tuple(med.albedo)
    elif med.fresnel_one:
        cm.fresnel = _lib.FRESNEL_ONE
    else:
        cm.fresnel = _lib.FRESNEL_CONDUCTOR
    cm.eta[:] = tuple(med.fresnel_eta)
    cm.k[:] = tuple(med.fresnel_k)


# ---------------------------------------------------------------------------
# BASELINE config-5 fields


def _lattice(n, bounds):
    x = np.linspace(bounds[0][0], bounds[1][0], n, dtype=np.float64)
    y = np.linspace(bounds[0][1], bounds[1][1], n, dtype=np.float64)
    z = np.linspace(bounds[0][2], bounds[1][2], n, dtype=np.float64)
    return np.meshgrid(x, y, z, indexing="ij")


def union_sdf(n, bounds, spheres, torus):
    """min over exact sphere SDFs and the torus SDF (ring in the xy plane)."""
    X, Y, Z = _lattice(n, bounds)
    f = np.full(X.shape, np.inf)
    for c, r in spheres:
        f = np.minimum(f, np.sqrt((X - c[0]) ** 2 + (Y - c[1]) ** 2 + (Z - c[2]) ** 2) - r)
    if torus is not None:
        R, r = torus
        q = np.sqrt(X ** 2 + Y ** 2) - R
        f = np.minimum(f, np.sqrt(q ** 2 + Z ** 2) - r)
    return f.astype(np.float32)


def value_noise(n, seed, lo=0.01, hi=0.2, cells=6):
    """Smooth value noise: random lattice values on a (cells+1)^3 grid,
    smoothstep-interpolated to n^3, rescaled to [lo, hi]."""
    rs = np.random.default_rng(seed)
    lat = rs.uniform(0.0, 1.0, (cells + 1,) * 3)
    t = np.linspace(0.0, cells, n)
    i = np.minimum(t.astype(int), cells - 1)
    f = t - i
    s = f * f * (3.0 - 2.0 * f)
    out = np.zeros((n, n, n))
    for dx in (0, 1):
        wx = s if dx else 1.0 - s
        for dy in (0, 1):
            wy = s if dy else 1.0 - s
            for dz in (0, 1):
                wz = s if dz else 1.0 - s
                vals = lat[np.ix_(i + dx, i + dy, i + dz)]
                out += vals * wx[:, None, None] * wy[None, :, None] * wz[None, None, :]
    out = (out - out.min()) / max(out.max() - out.min(), 1e-12)
    return (lo + (hi - lo) * out).astype(np.float32)


def config5_fields(seed=4, n_sdf=256, n_sigma=128, bounds=((-1.6,) * 3, (1.6,) * 3)):
    rs = np.random.default_rng(seed)
    radii = rs.uniform(0.1, 0.3, 16)
    centres = rs.uniform(-0.7, 0.7, (16, 3))
    spheres = list(zip(centres, radii))
    sdf = union_sdf(n_sdf, bounds, spheres, (0.6, 0.15))
    sigma = value_noise(n_sigma, seed + 1)
    return GridSDF(sdf, bounds), sigma
