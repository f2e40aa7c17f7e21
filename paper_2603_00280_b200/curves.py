"""Closed-form curves of the microflake statistics, evaluated on the GPU
(C ABI `mf_curve`, `curve_kernel`).

Reference-named functions (same arguments and meaning, float64 numpy in
and out, fp32 device arithmetic):

    generalized_lambda(theta, phi, a3)            ndf.py:138-144
    generalized_lambda_dir(w, a3)                 ndf.py:120-135
    projected_area(theta, phi, a3)                ndf.py:174-177
    projected_area_dir(wo, kind, a3)              ndf.py:180-186
    generalized_ndf(theta_m, phi_m, a3)           ndf.py:227-229
    generalized_ndf_dir(wm, a3)                   ndf.py:209-224
    ndf_dir(wm, kind, a3)                         ndf.py:85-103 / 209-224 by kind
    vndf_eval(wm, wo, kind, a3)                   ndf.py:299-315 (one wo per call)
    planar_transmittance(h0, h1, theta, phi, medium)   medium.py:98-124

The erf-family functions take the roughness triple as given (az = 0 is the
Beckmann height-field limit), as the reference does.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import GrazingSingularityError, ParameterDomainError, UnsupportedGeometryError
from .medium import MacrofacetMedium, to_c_medium
from .ndf import NdfKind, RoughnessTriple


def _sph_dir(theta, phi):
    theta = np.asarray(theta, dtype=np.float64)
    phi = np.asarray(phi, dtype=np.float64)
    st = np.sin(theta)
    return np.stack(np.broadcast_arrays(st * np.cos(phi), st * np.sin(phi), np.cos(theta)),
                    axis=-1)


def _erf_medium(a3: RoughnessTriple):
    kind = NdfKind.GENERALIZED if a3.az > 0.0 else NdfKind.BECKMANN
    return MacrofacetMedium(kind=kind, a3=a3, sigma=1.0, fresnel_one=True)


def curve_device(medium: MacrofacetMedium, kind, x, y=None, z=None, wo=(0.0, 0.0, 1.0), z0=0.0,
                 out=None, stream=None):
    """mf_curve on device float32 tensors (x, y, z: direction components,
    or x = end field values h1 for "transmittance", from h0 = z0); returns
    the output tensor."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    if kind not in _lib.CURVE:
        raise ParameterDomainError(f"unknown curve kind {kind!r}")
    n = x.numel()
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=x.device)
    prm = (ctypes.c_double * 4)(*(float(v) for v in wo), float(z0))
    cm = to_c_medium(medium)
    ptr = (lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None)
    s = stream if stream is not None else _lib.stream_handle(torch, x.device)
    _lib.check(lib.mf_curve(ctypes.byref(cm), _lib.CURVE[kind], ptr(x), ptr(y), ptr(z), n, prm,
                            ptr(out), s))
    return out


def _curve_host(medium, kind, w=None, t=None, wo=(0.0, 0.0, 1.0), z0=0.0):
    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())

    def col(a):
        return torch.from_numpy(np.ascontiguousarray(np.reshape(a, -1), dtype=np.float32)).to(dev)

    if t is not None:
        t = np.asarray(t, dtype=np.float64)
        r = curve_device(medium, kind, col(t), wo=wo, z0=z0)
        return r.cpu().numpy().astype(np.float64).reshape(t.shape)[()]
    w = np.asarray(w, dtype=np.float64)
    shape = w.shape[:-1]
    r = curve_device(medium, kind, col(w[..., 0]), col(w[..., 1]), col(w[..., 2]), wo=wo)
    return r.cpu().numpy().astype(np.float64).reshape(shape)[()]


def generalized_lambda_dir(w, a3: RoughnessTriple):
    """Smith Lambda(w) = sigma(w) / cos(theta); GrazingSingularityError at
    grazing directions, as the reference (ndf.py:120-135)."""
    w = np.asarray(w, dtype=np.float64)
    if np.any(np.abs(w[..., 2]) < 1e-9 * np.linalg.norm(w, axis=-1)):
        raise GrazingSingularityError("Lambda diverges at grazing directions; use projected_area")
    return _curve_host(_erf_medium(a3), "lambda", w=w)


def generalized_lambda(theta, phi, a3: RoughnessTriple):
    return generalized_lambda_dir(_sph_dir(theta, phi), a3)


def projected_area_dir(wo, kind: NdfKind, a3: RoughnessTriple):
    if kind is NdfKind.GENERALIZED:
        med = MacrofacetMedium(kind=kind, a3=a3, sigma=1.0, fresnel_one=True)
    else:
        med = MacrofacetMedium(kind=kind, a3=RoughnessTriple(a3.ax, a3.ay, 0.0), sigma=1.0,
                               fresnel_one=True)
    return _curve_host(med, "projected-area", w=wo)


def projected_area(theta, phi, a3: RoughnessTriple):
    return _curve_host(_erf_medium(a3), "projected-area", w=_sph_dir(theta, phi))


def generalized_ndf_dir(wm, a3: RoughnessTriple):
    if a3.az <= 0.0:
        raise ParameterDomainError("generalized NDF requires az > 0")
    return _curve_host(_erf_medium(a3), "ndf", w=wm)


def generalized_ndf(theta_m, phi_m, a3: RoughnessTriple):
    return generalized_ndf_dir(_sph_dir(theta_m, phi_m), a3)


def ndf_dir(wm, kind: NdfKind, a3: RoughnessTriple):
    """D(wm) dispatched on kind (the reference's _ndf_dispatch)."""
    a = a3 if kind is NdfKind.GENERALIZED else RoughnessTriple(a3.ax, a3.ay, 0.0)
    return _curve_host(MacrofacetMedium(kind=kind, a3=a, sigma=1.0, fresnel_one=True), "ndf",
                       w=wm)


def vndf_eval(wm, wo, kind: NdfKind, a3: RoughnessTriple):
    """<-wo, wm>+ D(wm) / sigma(wo) for one propagation direction wo;
    DegenerateVisibilityError when sigma(wo) < 1e-12 (ndf.py:312-313)."""
    wo = np.asarray(wo, dtype=np.float64)
    if wo.ndim != 1:
        raise ParameterDomainError("vndf_eval on the device takes one wo per call")
    a = a3 if kind is NdfKind.GENERALIZED else RoughnessTriple(a3.ax, a3.ay, 0.0)
    med = MacrofacetMedium(kind=kind, a3=a, sigma=1.0, fresnel_one=True)
    return _curve_host(med, "vndf", w=wm, wo=tuple(wo))


def planar_transmittance(h0, h1, theta, phi, medium: MacrofacetMedium):
    """exp(-Lambda (log Phi(h1/s) - log Phi(h0/s))) (medium.py:98-124), for
    scalar h0 / theta / phi and scalar or array h1."""
    theta = float(theta)
    c = np.cos(theta)
    if abs(c) < 1e-12:
        raise UnsupportedGeometryError("planar transmittance is undefined at cos(theta) = 0")
    if medium.kind is NdfKind.GGX:
        raise UnsupportedGeometryError("closed-form transmittance covers the erf-family lambda only")
    wo = tuple(_sph_dir(theta, float(phi)))
    return _curve_host(medium, "transmittance", t=h1, wo=wo, z0=float(h0))


# ---------------------------------------------------------------------------
# the reference's remaining public helpers of the path, on the device

def _scalar_curve(medium, kind, x):
    x = np.asarray(x, dtype=np.float64)
    return _curve_host(medium, kind, t=x)


def density(f, sigma):
    """Microflake density rho(f) = phi(f/s) / (s Phi(f/s)) (medium.py:70-88),
    fp32 on the device (erfcx form: no underflow deep below the surface)."""
    sigma = float(sigma)
    if not sigma > 0.0:
        raise ParameterDomainError(f"sigma must be > 0, got {sigma}")
    med = MacrofacetMedium(kind=NdfKind.GENERALIZED, a3=RoughnessTriple(1.0, 1.0, 1.0),
                           sigma=sigma, fresnel_one=True)
    return _scalar_curve(med, "density", f)


def fresnel_conductor(cos_i, eta, k):
    """Unpolarised conductor reflectance (medium.py:127-147); eta / k scalars
    or per-channel arrays broadcast against cos_i (device, fp32)."""
    cos_i = np.asarray(cos_i, dtype=np.float64)
    eta = np.asarray(eta, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    c, e, kk = np.broadcast_arrays(cos_i, eta, k)
    out = np.empty(c.shape)
    pairs = {}
    for idx in np.ndindex(c.shape) if c.shape else [()]:
        pairs.setdefault((float(e[idx]), float(kk[idx])), []).append(idx)
    for (ev, kv), idxs in pairs.items():
        med = MacrofacetMedium(kind=NdfKind.GENERALIZED, a3=RoughnessTriple(1.0, 1.0, 1.0),
                               sigma=1.0, fresnel_eta=(ev, ev, ev), fresnel_k=(kv, kv, kv))
        vals = np.atleast_1d(_scalar_curve(med, "fresnel", np.array([c[i] for i in idxs])))
        for i, v in zip(idxs, vals):
            out[i] = v
    return out[()]


def beckmann_ndf(wm, ax, ay):
    """Height-field Beckmann D(wm) (ndf.py:85-94), device."""
    return ndf_dir(wm, NdfKind.BECKMANN, RoughnessTriple(float(ax), float(ay), 0.0))


def ggx_ndf(wm, ax, ay):
    """GGX D(wm) (ndf.py:97-103), device."""
    return ndf_dir(wm, NdfKind.GGX, RoughnessTriple(float(ax), float(ay), 0.0))


def gdf_pdf(g, a3: RoughnessTriple):
    """Gradient density conditioned on a zero crossing: Gaussian with mean
    (0, 0, 1) and variances alpha_i^2 / 2 (ndf.py:232-239), device."""
    if a3.az <= 0.0:
        raise ParameterDomainError("gdf_pdf requires az > 0")
    med = MacrofacetMedium(kind=NdfKind.GENERALIZED, a3=a3, sigma=1.0, fresnel_one=True)
    return _curve_host(med, "gdf", w=g)


def sample_gdf(a3: RoughnessTriple, rng, n: int):
    """n gradients from the conditioned gradient distribution (ndf.py:242-246):
    the stream's normals scaled by alpha / sqrt2 about (0, 0, 1)."""
    z = rng.normal((n, 3))
    return z * (np.array([a3.ax, a3.ay, a3.az]) / np.sqrt(2.0)) + np.array([0.0, 0.0, 1.0])


def vndf_sample(wo, kind: NdfKind, a3: RoughnessTriple, mix_ratio, rng, n=None):
    """Visible normals for propagation direction wo and their exact mixture
    pdf (ndf.py:383-427): the device's phase sampler (query_kernel) returns
    the normal it drew and its density.  Three uniforms per sample are
    taken from rng as the reference does; the device's two-uniform
    convention uses the first and the third."""
    from .core import Frame
    from .errors import DegenerateVisibilityError
    from .medium import _host_query

    if not (0.0 <= mix_ratio <= 1.0):
        raise ParameterDomainError(f"mix_ratio must lie in [0, 1], got {mix_ratio}")
    wo = np.asarray(wo, dtype=np.float64)
    if np.any(np.asarray(projected_area_dir(wo, kind, a3)) <= 0.0):
        raise DegenerateVisibilityError("projected area is zero toward wo")
    shape = wo.shape[:-1] if n is None else (n,)
    u = rng.uniform(shape + (3,))
    if n is not None and wo.ndim == 1:
        wo = np.broadcast_to(wo, (n, 3))
    a = a3 if kind is NdfKind.GENERALIZED else RoughnessTriple(a3.ax, a3.ay, 0.0)
    med = MacrofacetMedium(kind=kind, a3=a, sigma=1.0, fresnel_one=True, mix_ratio=mix_ratio)
    ident = Frame(tangent=np.array([1.0, 0.0, 0.0]), bitangent=np.array([0.0, 1.0, 0.0]),
                  normal=np.array([0.0, 0.0, 1.0]))
    r, _ = _host_query(med, wo, None, None, ident, np.stack([u[..., 0], u[..., 2]], axis=-1),
                       ("wmx", "wmy", "wmz", "pdf_m", "flags"))
    if np.any(r["flags"] & 1):
        raise DegenerateVisibilityError("projected area is zero toward wo")
    wm = np.stack([r["wmx"], r["wmy"], r["wmz"]], axis=-1).astype(np.float64)
    pdf = r["pdf_m"].astype(np.float64)
    return wm, pdf[()]


def ndf_from_gdf_quadrature(theta_m, phi_m, a3: RoughnessTriple, rel_tol=1e-8):
    """The generalized NDF at (theta_m, phi_m) by radial quadrature of the
    gradient distribution, t^3 gdf(t wm) over t > 0 (ndf.py:254-293): the
    independent check of generalized_ndf.  32-node Gauss-Legendre pieces on
    the device in float64 (mf_gdf_radial), the piece count doubled until
    the relative change drops below rel_tol."""
    from .errors import NumericFailureError

    if a3.az <= 0.0:
        raise ParameterDomainError("quadrature requires az > 0")
    wm = np.asarray(_sph_dir(theta_m, phi_m), dtype=np.float64)
    if wm.ndim != 1:
        raise ParameterDomainError("quadrature evaluates one direction at a time")
    torch = _lib.require_cuda()
    lib = _lib.load()
    a = float((wm[0] / a3.ax) ** 2 + (wm[1] / a3.ay) ** 2 + (wm[2] / a3.az) ** 2)
    b = float(wm[2] / a3.az ** 2)
    c = float(1.0 / a3.az ** 2)
    t_peak = max(b / a, 0.0)
    t_max = t_peak + np.sqrt(44.0 / a)            # the Gaussian factor below ~1e-14 of its peak
    shift = b * b / a - c if b > 0.0 else -c      # the exponent's peak, factored out
    x, w = np.polynomial.legendre.leggauss(32)
    xs, ws = (ctypes.c_double * 32)(*x), (ctypes.c_double * 32)(*w)
    dev = torch.device("cuda", torch.cuda.current_device())
    prev = None
    for n_sub in (1, 2, 4, 8, 16, 32, 64, 128):
        tot = ctypes.c_double()
        _lib.check(lib.mf_gdf_radial(a, b, c, shift, float(t_max), n_sub, xs, ws,
                                     ctypes.byref(tot), _lib.stream_handle(torch, dev)))
        total = tot.value
        if prev is not None and abs(total - prev) <= rel_tol * abs(total):
            return total * np.exp(shift) / (np.pi ** 1.5 * a3.ax * a3.ay * a3.az)
        prev = total
    raise NumericFailureError(f"radial NDF quadrature did not converge (theta={theta_m}, "
                              f"phi={phi_m}, alpha=({a3.ax},{a3.ay},{a3.az}), last={prev})")
