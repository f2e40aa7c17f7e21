"""The brute-force Gaussian-random-field oracle on the GPU (reference gp.py,
SURVEY.md 8(f) rank 4).

The macrofacet medium replaces explicit GP realisations; this module keeps
the reference's realisation machinery -- the competitor the paper compares
against and the ground truth of the `oracle` CLI experiments and the
`multiplicativity` validation suite -- and runs it B200-side in float64:

* white noise: RandomStream.normal drawn on the device, bit for bit
  (`mf_gp_noise`, SplitMix64 + Box-Muller, rng.py:46-97);
* filtering: one batched cuFFT forward / inverse transform of every
  realisation of a call (torch.fft, float64) times the square root of the
  wrapped kernel's DFT (gp.py:68-77, built on the host as the reference
  does);
* field_at / gradient_at / first_hit / the ensemble's specular bounce loop:
  `mf_gp_eval`, `mf_gp_first_hit`, `mf_gp_reflect_paths` (csrc/mf_gp.cuh),
  one thread per ray over all realisations of a call, in the reference's
  float64 operation order.

The experiments (empirical_transmittance, empirical_vndf,
multiplicativity_probe, ensemble_radiance) draw from the same streams as
the reference (rng.derive(i) per realisation), so their results match it
to float64 rounding (tests/test_gpu_gp.py against tests/golden/gp_ref.npz).
The reference's desk-scale limits (<= 64 x 64 pixels, <= 4096
realisations, grid validity) are kept as errors for drop-in behaviour.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from functools import lru_cache
from typing import Optional

import numpy as np

from . import _lib
from .errors import ConfigError, ParameterDomainError
from .ndf import KernelParams
from .rng import derive_bases, stream_base

_BATCH = 256          # realisations per device batch


@dataclass(frozen=True)
class GridSpec:
    """Cubic periodic grid: n cells per axis, world spacing per cell, centred
    on the origin (gp.py:26-41)."""

    n: int
    spacing: float

    @property
    def extent(self):
        return self.n * self.spacing

    @property
    def origin(self):
        return -0.5 * self.extent


def default_grid(kernel: KernelParams, factor=8.5):
    """Smallest valid grid: extent >= 8 max(l), spacing <= min(l) / 4
    (gp.py:44-52)."""
    lmax = max(kernel.lx, kernel.ly, kernel.lz)
    lmin = min(kernel.lx, kernel.ly, kernel.lz)
    spacing = lmin / 4.0
    n = int(np.ceil(factor * lmax / spacing))
    n += n % 2
    return GridSpec(n=n, spacing=spacing)


def _validate_grid(kernel: KernelParams, spec: GridSpec):
    lmax = max(kernel.lx, kernel.ly, kernel.lz)
    lmin = min(kernel.lx, kernel.ly, kernel.lz)
    if spec.extent < 8.0 * lmax:
        raise ConfigError(f"grid extent {spec.extent:.4g} < 8 * max correlation {8*lmax:.4g}")
    if spec.spacing > lmin / 4.0 + 1e-12:
        raise ConfigError(f"grid spacing {spec.spacing:.4g} > min correlation / 4 = {lmin/4:.4g}")


@lru_cache(maxsize=8)
def _filter_sqrt_host(kernel: KernelParams, spec: GridSpec):
    # square roots of the DFT eigenvalues of the wrapped squared-exponential
    # covariance (gp.py:68-77), on the host in numpy as the reference
    n, h = spec.n, spec.spacing
    lag = np.minimum(np.arange(n), n - np.arange(n)) * h
    ex = np.exp(-0.5 * (lag / kernel.lx) ** 2)
    ey = np.exp(-0.5 * (lag / kernel.ly) ** 2)
    ez = np.exp(-0.5 * (lag / kernel.lz) ** 2)
    cov = kernel.sigma**2 * ex[:, None, None] * ey[None, :, None] * ez[None, None, :]
    return np.sqrt(np.maximum(np.fft.fftn(cov).real, 0.0))


_FILTERS = {}


def _filter_sqrt(kernel, spec, torch, dev):
    key = (kernel, spec, dev)
    f = _FILTERS.get(key)
    if f is None:
        if len(_FILTERS) > 8:
            _FILTERS.clear()
        f = _FILTERS[key] = torch.from_numpy(_filter_sqrt_host(kernel, spec)).to(dev)
    return f


def _dev():
    torch = _lib.require_cuda()
    return torch, torch.device("cuda", torch.cuda.current_device())


def _base_of(rng):
    """SplitMix64 base state of a RandomStream-like object (ours or the
    reference's: seed / stream / counter fields)."""
    return np.uint64(stream_base(int(rng.seed), int(rng.stream)))


@dataclass
class GpBatch:
    """Realisations of one call on the device: grid (B, n, n, n) float64."""

    grid: object
    spec: GridSpec
    kernel: KernelParams
    mean: str
    bound: object = None     # (B,) max |value| per realisation (march early exit)

    def c_grid(self):
        g = _lib.MfGpGrid()
        g.d_grid = self.grid.data_ptr()
        g.n = self.spec.n
        g.spacing = self.spec.spacing
        g.origin = self.spec.origin
        g.planar = 1 if self.mean == "planar" else 0
        g.d_bound = self.bound.data_ptr() if self.bound is not None else None
        return g


def _realize(kernel, mean, spec, bases, counter0=0):
    """Realisations of the streams with SplitMix64 base states `bases`
    (noise counters from counter0): white noise on the device, one batched
    FFT filtering (gp.py:131-141)."""
    if mean not in ("planar", "zero"):
        raise ParameterDomainError(f"mean must be 'planar' or 'zero', got {mean!r}")
    torch, dev = _dev()
    lib = _lib.load()
    n = spec.n
    b = torch.from_numpy(np.ascontiguousarray(bases, dtype=np.uint64).view(np.int64)).to(dev)
    white = torch.empty((len(bases), n, n, n), dtype=torch.float64, device=dev)
    _lib.check(lib.mf_gp_noise(ctypes.c_void_p(b.data_ptr()), len(bases), int(counter0), n ** 3,
                               ctypes.c_void_p(white.data_ptr()), _lib.stream_handle(torch, dev)))
    spec_f = torch.fft.fftn(white, dim=(1, 2, 3)) * _filter_sqrt(kernel, spec, torch, dev)
    grid = torch.fft.ifftn(spec_f, dim=(1, 2, 3)).real.contiguous()
    bound = grid.abs().amax(dim=(1, 2, 3)).contiguous()
    return GpBatch(grid=grid, spec=spec, kernel=kernel, mean=mean, bound=bound)


def _noise_draws(n_cells):
    """Counters RandomStream.normal(n) consumes (two per pair)."""
    return 2 * ((n_cells + 1) // 2)


@dataclass
class GpRealization:
    """One sampled field on a periodic grid; the planar mean is analytic
    (gp.py:80-127).  The grid lives on the device (float64)."""

    batch: GpBatch
    index: int = 0

    @property
    def spec(self):
        return self.batch.spec

    @property
    def kernel(self):
        return self.batch.kernel

    @property
    def mean(self):
        return self.batch.mean

    @property
    def grid(self):
        """The stationary field values, (n, n, n) float64 (host copy)."""
        return self.batch.grid[self.index].cpu().numpy()

    def _eval(self, p, want_f, want_g):
        torch, dev = _dev()
        lib = _lib.load()
        p = np.asarray(p, dtype=np.float64)
        shape = p.shape[:-1]
        pts = p.reshape(-1, 3)
        m = pts.shape[0]
        P = torch.from_numpy(np.ascontiguousarray(pts.T)).to(dev)
        real = torch.full((m,), self.index, dtype=torch.int32, device=dev)
        f = torch.empty(m, dtype=torch.float64, device=dev) if want_f else None
        g = torch.empty((3, m), dtype=torch.float64, device=dev) if want_g else None
        cg = self.batch.c_grid()
        _lib.check(lib.mf_gp_eval(ctypes.byref(cg), ctypes.c_void_p(P.data_ptr()),
                                  ctypes.c_void_p(real.data_ptr()), m,
                                  ctypes.c_void_p(f.data_ptr()) if f is not None else None,
                                  ctypes.c_void_p(g.data_ptr()) if g is not None else None,
                                  _lib.stream_handle(torch, dev)))
        if want_f:
            return f.cpu().numpy().reshape(shape)
        return g.cpu().numpy().T.reshape(shape + (3,))

    def field_at(self, p):
        """Trilinear periodic interpolation plus the mean."""
        return self._eval(p, True, False)

    def gradient_at(self, p):
        """Central differences of the interpolant (step = one cell)."""
        return self._eval(p, False, True)


def realize_gp(kernel: KernelParams, mean, spec: Optional[GridSpec], rng):
    """Draw one stationary field realisation (gp.py:131-141); rng is a
    RandomStream (ours or the reference's), advanced by the noise draws."""
    if mean not in ("planar", "zero"):
        raise ParameterDomainError(f"mean must be 'planar' or 'zero', got {mean!r}")
    if spec is None:
        spec = default_grid(kernel)
    _validate_grid(kernel, spec)
    batch = _realize(kernel, mean, spec, [_base_of(rng)], int(rng.counter))
    rng.counter = int(rng.counter) + _noise_draws(spec.n ** 3)
    return GpRealization(batch, 0)


@dataclass
class FirstHit:
    """First zero crossings for a batch of rays (arrays over rays)."""

    hit: np.ndarray
    position: np.ndarray
    normal: np.ndarray
    travel: np.ndarray


def _first_hit_dev(batch, o, d, real, t_max, tmax_real=None):
    """first_hit of device rays o, d (SoA [3][m] float64 tensors) in the
    realisations real (int32 tensor); returns device tensors."""
    torch, dev = _dev()
    lib = _lib.load()
    m = o.shape[1]
    k = batch.kernel
    step = min(k.lx, k.ly, k.lz) / 8.0
    hit = torch.empty(m, dtype=torch.uint8, device=dev)
    pos = torch.empty((3, m), dtype=torch.float64, device=dev)
    nrm = torch.empty((3, m), dtype=torch.float64, device=dev)
    trv = torch.empty(m, dtype=torch.float64, device=dev)
    cg = batch.c_grid()
    _lib.check(lib.mf_gp_first_hit(
        ctypes.byref(cg), ctypes.c_void_p(o.data_ptr()), ctypes.c_void_p(d.data_ptr()),
        ctypes.c_void_p(real.data_ptr()), m, step,
        ctypes.c_void_p(tmax_real.data_ptr()) if tmax_real is not None else None, float(t_max),
        ctypes.c_void_p(hit.data_ptr()), ctypes.c_void_p(pos.data_ptr()),
        ctypes.c_void_p(nrm.data_ptr()), ctypes.c_void_p(trv.data_ptr()),
        _lib.stream_handle(torch, dev)))
    return hit, pos, nrm, trv


def first_hit(real: GpRealization, origins, directions, t_max):
    """Fixed-step march (min(l)/8) to the first sign change of the
    interpolated field, refined by 30 bisections; the normal is the
    normalised central-difference gradient at the crossing (gp.py:148-197)."""
    torch, dev = _dev()
    o = np.atleast_2d(np.asarray(origins, dtype=np.float64))
    d = np.atleast_2d(np.asarray(directions, dtype=np.float64))
    o, d = np.broadcast_arrays(o, d)
    m = o.shape[0]
    O = torch.from_numpy(np.ascontiguousarray(o.T)).to(dev)
    D = torch.from_numpy(np.ascontiguousarray(d.T)).to(dev)
    R = torch.full((m,), real.index, dtype=torch.int32, device=dev)
    hit, pos, nrm, trv = _first_hit_dev(real.batch, O, D, R, t_max)
    return FirstHit(hit=hit.cpu().numpy().astype(bool), position=pos.cpu().numpy().T.copy(),
                    normal=nrm.cpu().numpy().T.copy(), travel=trv.cpu().numpy())


def _batches(m):
    for a in range(0, m, _BATCH):
        yield a, min(m, a + _BATCH)


def empirical_transmittance(kernel, z0, theta, phi, t_grid, m_realizations, rng, spec=None):
    """Fraction of realisations whose first crossing exceeds each t, rays
    from the fixed point (0, 0, z0); realisations whose start lies inside
    the solid are skipped (gp.py:200-237).  Returns rows (t, Tr, SE)."""
    if m_realizations < 64:
        raise ParameterDomainError("need at least 64 realizations")
    if spec is None:
        spec = default_grid(kernel)
    _validate_grid(kernel, spec)
    torch, dev = _dev()
    d = np.array([np.sin(theta) * np.cos(phi), np.sin(theta) * np.sin(phi), np.cos(theta)])
    o = np.array([0.0, 0.0, z0])
    t_grid = np.asarray(t_grid, dtype=np.float64)
    t_max = float(t_grid.max())
    bases = derive_bases(int(rng.seed), int(rng.stream), np.arange(m_realizations))
    crossings = []
    for a, b in _batches(m_realizations):
        batch = _realize(kernel, "planar", spec, bases[a:b])
        B = b - a
        O = torch.from_numpy(np.ascontiguousarray(np.tile(o, (B, 1)).T)).to(dev)
        D = torch.from_numpy(np.ascontiguousarray(np.tile(d, (B, 1)).T)).to(dev)
        R = torch.arange(B, dtype=torch.int32, device=dev)
        f0 = _eval_batch(batch, O, R)
        _, _, _, trv = _first_hit_dev(batch, O, D, R, t_max)
        keep = f0 > 0.0
        crossings.extend(trv.cpu().numpy()[keep].tolist())
    crossings = np.asarray(crossings)
    kept = len(crossings)
    rows = []
    for t in t_grid:
        p = float(np.mean(crossings > t))
        se = float(np.sqrt(max(p * (1.0 - p), 1e-12) / kept))
        rows.append((float(t), p, se))
    return rows


def _eval_batch(batch, P, R):
    torch, dev = _dev()
    lib = _lib.load()
    m = P.shape[1]
    f = torch.empty(m, dtype=torch.float64, device=dev)
    cg = batch.c_grid()
    _lib.check(lib.mf_gp_eval(ctypes.byref(cg), ctypes.c_void_p(P.data_ptr()),
                              ctypes.c_void_p(R.data_ptr()), m, ctypes.c_void_p(f.data_ptr()),
                              None, _lib.stream_handle(torch, dev)))
    return f.cpu().numpy()


def _uniforms(bases, counter0, n):
    """RandomStream.uniform(n) of every stream in `bases` from counter0, on
    the device: (len(bases), n) float64 host array."""
    torch, dev = _dev()
    lib = _lib.load()
    b = torch.from_numpy(np.ascontiguousarray(bases, dtype=np.uint64).view(np.int64)).to(dev)
    out = torch.empty((len(bases), n), dtype=torch.float64, device=dev)
    _lib.check(lib.mf_gp_uniform(ctypes.c_void_p(b.data_ptr()), len(bases), int(counter0), n,
                                 ctypes.c_void_p(out.data_ptr()), _lib.stream_handle(torch, dev)))
    return out.cpu().numpy()


def empirical_vndf(kernel, wo, n_theta, n_phi, m_realizations, rng, rays_per_realization=256,
                   spec=None, z_start=None):
    """Histogram density of first-hit normals for parallel rays along wo
    (gp.py:240-281).  Returns (hist (n_theta, n_phi), (theta edges, phi
    edges)); bins integrate to 1."""
    wo = np.asarray(wo, dtype=np.float64)
    wo = wo / np.linalg.norm(wo, axis=-1, keepdims=True)
    if spec is None:
        spec = default_grid(kernel)
    _validate_grid(kernel, spec)
    torch, dev = _dev()
    sigma = kernel.sigma
    if z_start is None:
        z_start = 5.0 * sigma
    counts = np.zeros((n_theta, n_phi))
    t_max = (z_start + 4.0 * sigma) / max(1e-9, -wo[2]) if wo[2] < 0 else spec.extent
    nr = rays_per_realization
    bases = derive_bases(int(rng.seed), int(rng.stream), np.arange(m_realizations))
    skip = _noise_draws(spec.n ** 3)   # the stream draws the noise first, then the offsets
    for a, b in _batches(m_realizations):
        B = b - a
        batch = _realize(kernel, "planar", spec, bases[a:b])
        lat = _uniforms(bases[a:b], skip, 2 * nr).reshape(B, nr, 2) * spec.extent
        o = np.stack([lat[..., 0], lat[..., 1], np.full((B, nr), z_start)], axis=-1).reshape(-1, 3)
        O = torch.from_numpy(np.ascontiguousarray(o.T)).to(dev)
        D = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(wo, o.shape).T)).to(dev)
        R = torch.arange(B, dtype=torch.int32, device=dev).repeat_interleave(nr)
        hit, _, nrm, _ = _first_hit_dev(batch, O, D, R, t_max)
        hit = hit.cpu().numpy().astype(bool).reshape(B, nr)
        nm_all = nrm.cpu().numpy().T.reshape(B, nr, 3)
        for j in range(B):   # the reference's per-realisation histogram sums
            nm = nm_all[j][hit[j]]
            th = np.arccos(np.clip(nm[:, 2], -1.0, 1.0))
            ph = np.mod(np.arctan2(nm[:, 1], nm[:, 0]), 2.0 * np.pi)
            h, _, _ = np.histogram2d(th, ph, bins=[n_theta, n_phi],
                                     range=[[0.0, np.pi], [0.0, 2.0 * np.pi]])
            counts += h
    te = np.linspace(0.0, np.pi, n_theta + 1)
    pe = np.linspace(0.0, 2.0 * np.pi, n_phi + 1)
    solid = np.outer(np.cos(te[:-1]) - np.cos(te[1:]), np.diff(pe))
    total = counts.sum()
    dens = counts / (max(total, 1.0) * solid)
    return dens, (te, pe)


def multiplicativity_probe(kernel, origin, direction, split_t, t_end, m_realizations, rng,
                           spec=None, n_boot=1000):
    """Transmittance multiplicativity on shared realisations: Tr over (0,
    t_end], (0, split_t], (split_t, t_end] and the gap |Tr_xy - Tr_xz
    Tr_zy| with a bootstrap SE (gp.py:284-331)."""
    if m_realizations < 256:
        raise ParameterDomainError("need at least 256 realizations")
    if spec is None:
        spec = default_grid(kernel)
    _validate_grid(kernel, spec)
    torch, dev = _dev()
    o = np.asarray(origin, dtype=np.float64)
    d = np.asarray(direction, dtype=np.float64)
    d = d / np.linalg.norm(d, axis=-1, keepdims=True)
    o2 = o + split_t * d
    bases = derive_bases(int(rng.seed), int(rng.stream), np.arange(m_realizations))
    clear_a, clear_b, valid_a, valid_b = [], [], [], []
    for a, b in _batches(m_realizations):
        B = b - a
        batch = _realize(kernel, "planar", spec, bases[a:b])
        R = torch.arange(B, dtype=torch.int32, device=dev)
        Oa = torch.from_numpy(np.ascontiguousarray(np.tile(o, (B, 1)).T)).to(dev)
        Ob = torch.from_numpy(np.ascontiguousarray(np.tile(o2, (B, 1)).T)).to(dev)
        D = torch.from_numpy(np.ascontiguousarray(np.tile(d, (B, 1)).T)).to(dev)
        valid_a.extend((_eval_batch(batch, Oa, R) > 0.0).tolist())
        valid_b.extend((_eval_batch(batch, Ob, R) > 0.0).tolist())
        ha = _first_hit_dev(batch, Oa, D, R, split_t)[0].cpu().numpy()
        hb = _first_hit_dev(batch, Ob, D, R, t_end - split_t)[0].cpu().numpy()
        clear_a.extend((ha == 0).tolist())
        clear_b.extend((hb == 0).tolist())
    clear_a, clear_b = np.asarray(clear_a), np.asarray(clear_b)
    valid_a, valid_b = np.asarray(valid_a), np.asarray(valid_b)

    def stats(a, b, va, vb):
        xz = np.sum(a & va) / max(np.sum(va), 1)
        zy = np.sum(b & vb) / max(np.sum(vb), 1)
        xy = np.sum(a & b & va) / max(np.sum(va), 1)
        return xy, xz, zy

    tr_xy, tr_xz, tr_zy = stats(clear_a, clear_b, valid_a, valid_b)
    gap = abs(tr_xy - tr_xz * tr_zy)
    boot = rng.derive(0xB007)
    idx = (boot.uniform((n_boot, m_realizations)) * m_realizations).astype(np.int64)
    gaps = np.empty(n_boot)
    for k in range(n_boot):
        xy, xz, zy = stats(clear_a[idx[k]], clear_b[idx[k]], valid_a[idx[k]], valid_b[idx[k]])
        gaps[k] = abs(xy - xz * zy)
    se = float(np.std(gaps, ddof=1))
    return float(tr_xy), float(tr_xz), float(tr_zy), gap, se


def camera_rays(camera, px, py, jitter_x, jitter_y):
    """Pinhole rays through pixel (px, py) + jitter (scene.py:30-51), float64."""
    pos = np.asarray(camera.position, dtype=np.float64)
    fwd = np.asarray(camera.look_at, dtype=np.float64) - pos
    fwd = fwd / np.linalg.norm(fwd, axis=-1, keepdims=True)
    up = np.array([0.0, 0.0, 1.0])
    if abs(fwd @ up) > 0.999:
        up = np.array([0.0, 1.0, 0.0])
    right = np.cross(fwd, up)
    right = right / np.linalg.norm(right, axis=-1, keepdims=True)
    true_up = np.cross(right, fwd)
    half_h = np.tan(0.5 * np.deg2rad(camera.fov_deg))
    half_w = half_h * camera.width / camera.height
    ndc_x = ((px + jitter_x) / camera.width) * 2.0 - 1.0
    ndc_y = 1.0 - ((py + jitter_y) / camera.height) * 2.0
    d = fwd + ndc_x[..., None] * half_w * right + ndc_y[..., None] * half_h * true_up
    d = d / np.linalg.norm(d, axis=-1, keepdims=True)
    return np.broadcast_to(pos, d.shape), d


def ensemble_radiance(kernel, camera, spp, m_realizations, rng, env_radiance=1.0, fresnel=None,
                      max_bounces=64, spec=None, work=None):
    """Ensemble-averaged radiance of a planar statistical surface patch:
    per sample round one fresh realisation shared by all pixels; paths
    reflect specularly off first-hit normals until they escape upward and
    gather the constant environment (gp.py:334-398).  All rounds run in one
    batch on the device.  `work` (a dict, optional) receives the number of
    interpolant evaluations and paths."""
    w, h = camera.width, camera.height
    if w * h > 64 * 64:
        raise ConfigError("ensemble radiance is desk-scale only (<= 64x64 pixels)")
    if m_realizations > 4096:
        raise ConfigError("realization cap is 4096")
    if spec is None:
        spec = default_grid(kernel)
    _validate_grid(kernel, spec)
    torch, dev = _dev()
    lib = _lib.load()
    n_rounds = max(int(spp), 1)
    # round s: r = rng.derive(s); the realisation from r.derive(1); the
    # jitter from r's own first 2 h w uniforms
    rounds = np.arange(n_rounds)
    r_bases = derive_bases(int(rng.seed), int(rng.stream), rounds)
    r_streams = _child_streams(int(rng.stream), rounds)
    real_bases = np.array([derive_bases(int(rng.seed), int(s), [1])[0] for s in r_streams],
                          dtype=np.uint64)
    # the camera basis exactly as Camera.rays computes it (scene.py:30-51)
    pos = np.asarray(camera.position, dtype=np.float64)
    fwd = np.asarray(camera.look_at, dtype=np.float64) - pos
    fwd = fwd / np.linalg.norm(fwd, axis=-1, keepdims=True)
    up = np.array([0.0, 0.0, 1.0])
    if abs(fwd @ up) > 0.999:
        up = np.array([0.0, 1.0, 0.0])
    right = np.cross(fwd, up)
    right = right / np.linalg.norm(right, axis=-1, keepdims=True)
    true_up = np.cross(right, fwd)
    half_h = float(np.tan(0.5 * np.deg2rad(camera.fov_deg)))
    half_w = half_h * camera.width / camera.height
    vec = lambda a: (ctypes.c_double * 3)(*[float(x) for x in a])  # noqa: E731
    eps = spec.spacing * 0.25
    step = min(kernel.lx, kernel.ly, kernel.lz) / 8.0
    eta_k = None
    if fresnel is not None:
        eta_k = (vec(np.asarray(fresnel[0])), vec(np.asarray(fresnel[1])))
    s = _lib.stream_handle(torch, dev)
    img = torch.zeros((h, w, 3), dtype=torch.float64, device=dev)
    for a, b in _batches(n_rounds):
        B = b - a
        m = B * h * w
        batch = _realize(kernel, "planar", spec, real_bases[a:b])
        rb = torch.from_numpy(np.ascontiguousarray(r_bases[a:b]).view(np.int64)).to(dev)
        O = torch.empty((3, m), dtype=torch.float64, device=dev)
        D = torch.empty((3, m), dtype=torch.float64, device=dev)
        _lib.check(lib.mf_gp_camera_rays(vec(pos), vec(fwd), vec(right), vec(true_up), half_w,
                                         half_h, w, h, ctypes.c_void_p(rb.data_ptr()), B,
                                         ctypes.c_void_p(O.data_ptr()),
                                         ctypes.c_void_p(D.data_ptr()), s))
        T = torch.ones((3, m), dtype=torch.float64, device=dev)
        L = torch.zeros((3, m), dtype=torch.float64, device=dev)
        R = torch.arange(B, dtype=torch.int32, device=dev).repeat_interleave(h * w)
        ev = torch.zeros(1, dtype=torch.int64, device=dev) if work is not None else None
        cg = batch.c_grid()
        _lib.check(lib.mf_gp_reflect_paths(
            ctypes.byref(cg), ctypes.c_void_p(O.data_ptr()), ctypes.c_void_p(D.data_ptr()),
            ctypes.c_void_p(T.data_ptr()), ctypes.c_void_p(L.data_ptr()),
            ctypes.c_void_p(R.data_ptr()), m, B, float(kernel.sigma), float(env_radiance),
            float(eps), float(step), int(max_bounces),
            eta_k[0] if eta_k else None, eta_k[1] if eta_k else None,
            ctypes.c_void_p(ev.data_ptr()) if ev is not None else None, s))
        if work is not None:
            work["evals"] = work.get("evals", 0) + int(ev.item())
            work["paths"] = work.get("paths", 0) + m
        # the reference's round-by-round sum, continued across batches
        _lib.check(lib.mf_gp_round_sum(ctypes.c_void_p(L.data_ptr()), w, h, B, 1 if a else 0,
                                       ctypes.c_void_p(img.data_ptr()), s))
    return img.cpu().numpy() / n_rounds



def _child_streams(stream, indices):
    """Stream ids of RandomStream(seed, stream).derive(i) (rng.py:99-107)."""
    from .rng import _M1, _PHI, _U, _mix

    with np.errstate(over="ignore"):
        return _mix(np.asarray(stream, dtype=np.uint64) * _PHI
                    ^ np.asarray(indices, dtype=np.uint64) * _M1 + _U(1))
