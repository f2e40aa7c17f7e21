"""Oracle for heterogeneous grid fields (BASELINE config 5), float64 numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference has no grid fields: the field representation
-- a trilinear SDF grid for the mean, a trilinear per-voxel sigma grid,
roughness alpha = sqrt2 sigma / l -- is this repository's convention and has
no reference to pin it to ("parity unpinned" for the representation).  What
this module pins is everything evaluated ON that field: the density rho(f)
(medium.py:70-88), the projected area sigma(w) (ndf.py:156-164) and the
extinction rho sigma(w) (medium.py:91-95) are the reference's coefficient
functions (oracle/microfacet.py, checked against the reference's golden
values), applied point by point along a ray, and the transmittance is plain
quadrature of exp(-int sigma_t ds) -- no tracking, no majorants, no DDA.
It checks the device's grid walker (trilinear fetches, gradient frames,
region rules, majorant grid, delta / ratio tracking) on config 5's own
fields.  Region rule of shadow / ratio walks: |f| <= 3 sigma(p)
(transport.py:161-166 with sigma = sigma(p)).
"""

from __future__ import annotations

import math

import numpy as np

from . import microfacet as om


def trilinear(values, bounds, p, grad=False):
    """Trilinear interpolant of a vertex-centred n^3 grid over `bounds` at
    points p (..., 3); with grad=True also the gradient of the interpolant
    (world units).  Coordinates are clamped to the grid as on the device."""
    v = np.asarray(values, dtype=np.float64)
    n = v.shape[0]
    lo = np.asarray(bounds[0], dtype=np.float64)
    hi = np.asarray(bounds[1], dtype=np.float64)
    inv_h = (n - 1) / (hi - lo)
    g = np.clip((np.asarray(p, dtype=np.float64) - lo) * inv_h, 0.0, n - 1.0)
    i = np.clip(g.astype(np.int64), 0, n - 2)
    t = g - i
    ix, iy, iz = i[..., 0], i[..., 1], i[..., 2]
    tx, ty, tz = t[..., 0], t[..., 1], t[..., 2]
    c = {(a, b, k): v[ix + a, iy + b, iz + k] for a in (0, 1) for b in (0, 1) for k in (0, 1)}
    c00 = c[0, 0, 0] + tz * (c[0, 0, 1] - c[0, 0, 0])
    c01 = c[0, 1, 0] + tz * (c[0, 1, 1] - c[0, 1, 0])
    c10 = c[1, 0, 0] + tz * (c[1, 0, 1] - c[1, 0, 0])
    c11 = c[1, 1, 0] + tz * (c[1, 1, 1] - c[1, 1, 0])
    c0 = c00 + ty * (c01 - c00)
    c1 = c10 + ty * (c11 - c10)
    val = c0 + tx * (c1 - c0)
    if not grad:
        return val
    gx = c1 - c0
    gy = (1.0 - tx) * (c01 - c00) + tx * (c11 - c10)
    d00, d01 = c[0, 0, 1] - c[0, 0, 0], c[0, 1, 1] - c[0, 1, 0]
    d10, d11 = c[1, 0, 1] - c[1, 0, 0], c[1, 1, 1] - c[1, 1, 0]
    d0 = d00 + ty * (d01 - d00)
    d1 = d10 + ty * (d11 - d10)
    gz = d0 + tx * (d1 - d0)
    return val, np.stack([gx * inv_h[0], gy * inv_h[1], gz * inv_h[2]], axis=-1)


def extinction(sdf, sigma, bounds, l_xy, l_z, p, d, lo_mult=-3.0):
    """sigma_t(p, d) on the grid field: rho(f; sigma(p)) sigma(w) with w the
    direction d in the frame about the SDF gradient and alpha = sqrt2
    sigma(p) / l (isotropic in xy, so only <n, d> enters); 0 outside
    [lo_mult sigma, 3 sigma]."""
    f, g = trilinear(sdf, bounds, p, grad=True)
    s = np.maximum(trilinear(sigma, bounds, p), 1e-6)
    gn = np.linalg.norm(g, axis=-1)
    dd = np.asarray(d, dtype=np.float64)
    c = np.where(gn > 0.0, np.einsum("...k,k->...", g, dd) / np.where(gn > 0.0, gn, 1.0), dd[2])
    c = np.clip(c, -1.0, 1.0)
    w = np.stack([np.sqrt(np.maximum(1.0 - c * c, 0.0)), np.zeros_like(c), c], axis=-1)
    ax = math.sqrt(2.0) * s / l_xy
    az = math.sqrt(2.0) * s / l_z
    area = om.projected_area_erf(w, ax, ax, az)
    rho = om.density(f, s)
    inside = (f >= lo_mult * s) & (f <= 3.0 * s)
    return np.where(inside, rho * area, 0.0)


def box_span(bounds, o, d):
    """Parametric entry / exit of the ray o + t d through the grid bounds
    (entry clamped to 0); None on a miss."""
    lo = np.asarray(bounds[0], dtype=np.float64)
    hi = np.asarray(bounds[1], dtype=np.float64)
    o = np.asarray(o, dtype=np.float64)
    d = np.asarray(d, dtype=np.float64)
    t0, t1 = 0.0, math.inf
    for a in range(3):
        if d[a] == 0.0:
            if o[a] < lo[a] or o[a] > hi[a]:
                return None
            continue
        u, v = (lo[a] - o[a]) / d[a], (hi[a] - o[a]) / d[a]
        t0, t1 = max(t0, min(u, v)), min(t1, max(u, v))
    return (t0, t1) if t0 <= t1 else None


def transmittance(sdf, sigma, bounds, l_xy, l_z, o, d, step=2e-5, lo_mult=-3.0):
    """exp(-int sigma_t ds) along the ray through the grid by the composite
    trapezoid rule with the given step (the integrand jumps at the region
    edges: the error is O(jump x step) per crossing)."""
    span = box_span(bounds, o, d)
    if span is None:
        return 1.0
    t0, t1 = span
    n = max(int(math.ceil((t1 - t0) / step)), 2)
    tau = 0.0
    chunk = 1 << 18
    ts_all = np.linspace(t0, t1, n + 1)
    o = np.asarray(o, dtype=np.float64)
    dd = np.asarray(d, dtype=np.float64)
    for k in range(0, n + 1, chunk):
        ts = ts_all[k:k + chunk + 1]   # one overlapping node joins the chunks
        st = extinction(sdf, sigma, bounds, l_xy, l_z, o[None] + ts[:, None] * dd[None], dd,
                        lo_mult)
        tau += float(np.trapezoid(st, ts))
    return math.exp(-tau)


class _LocalMedium:
    """The medium at one point of the field, duck-typed for oracle.microfacet."""

    kind = "generalized"
    mix_ratio = 0.5
    fresnel_one = False
    fresnel_eta = (1.0, 1.0, 1.0)
    fresnel_k = (0.0, 0.0, 0.0)

    def __init__(self, s, l_xy, l_z, albedo, mix_ratio):
        class A:
            ax = ay = math.sqrt(2.0) * s / l_xy
            az = math.sqrt(2.0) * s / l_z

        self.a3 = A
        self.sigma = s
        self.albedo = albedo
        self.mix_ratio = mix_ratio


def _frame(n):
    n = n / np.linalg.norm(n)
    a = np.array([1.0, 0.0, 0.0]) if abs(n[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
    t = np.cross(a, n)
    t /= np.linalg.norm(t)
    return t, np.cross(n, t), n


def single_scatter_radiance(sdf, sigma, bounds, l_xy, l_z, albedo, o, d, sun_to, sun_radiance,
                            env_radiance, mix_ratio=0.5, step=2.5e-4, stride=8, sun_step=5e-4):
    """Depth-1 radiance along the ray o + t d through the grid field (the
    renderer's estimator at max_bounces = 1, render.py:32-108, as an
    integral): T6(total) env + int T6(t) sigma_t(t) phase(t) Tr_sun(t) dt
    sun_radiance, with T6 the transmittance over the collision-walk region
    [-6 sigma, 3 sigma], the phase function of the local medium in the frame
    about the SDF gradient (medium.py:158-178) and Tr_sun the shadow
    transmittance over |f| <= 3 sigma.  Channel-0 value (grey albedo)."""
    span = box_span(bounds, o, d)
    o = np.asarray(o, dtype=np.float64)
    dd = np.asarray(d, dtype=np.float64)
    sl = np.asarray(sun_to, dtype=np.float64)
    if span is None:
        return float(env_radiance)
    t0, t1 = span
    n = max(int(math.ceil((t1 - t0) / step)), 2)
    ts = np.linspace(t0, t1, n + 1)
    pts = o[None] + ts[:, None] * dd[None]
    st = extinction(sdf, sigma, bounds, l_xy, l_z, pts, dd, lo_mult=-6.0)
    tau = np.concatenate([[0.0], np.cumsum(0.5 * (st[1:] + st[:-1]) * np.diff(ts))])
    t6 = np.exp(-tau)
    wgt = t6 * st
    idx = np.arange(0, n + 1, stride)
    keep = wgt[idx] > 1e-7 * max(wgt.max(), 1e-300)
    vals = np.zeros(len(idx))
    for j in np.nonzero(keep)[0]:
        i = idx[j]
        p = pts[i]
        f, g = trilinear(sdf, bounds, p[None], grad=True)
        s = max(float(trilinear(sigma, bounds, p[None])[0]), 1e-6)
        gn = np.linalg.norm(g[0])
        t, b, nn = _frame(g[0] if gn > 0.0 else np.array([0.0, 0.0, 1.0]))
        wo_l = np.array([dd @ t, dd @ b, dd @ nn])
        wi_l = np.array([sl @ t, sl @ b, sl @ nn])
        m = _LocalMedium(s, l_xy, l_z, albedo, mix_ratio)
        try:
            ph = float(om.phase_eval_local(wo_l[None], wi_l[None], m)[0, 0])
        except om.OracleDomainError:
            ph = 0.0
        if ph <= 0.0:
            continue
        tr = transmittance(sdf, sigma, bounds, l_xy, l_z, p, sl, step=sun_step, lo_mult=-3.0)
        vals[j] = wgt[i] * ph * tr
    return float(t6[-1] * env_radiance + np.trapezoid(vals, ts[idx]) * sun_radiance)
