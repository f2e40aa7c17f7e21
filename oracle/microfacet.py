"""Oracle microfacet / medium physics (reference L1 + L2), float64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Media are duck-typed: anything with `.kind` (enum with `.value` or str),
`.a3` (`.ax/.ay/.az`), `.sigma`, `.mix_ratio`, `.fresnel_one`,
`.fresnel_eta`, `.fresnel_k` works -- the reference's MacrofacetMedium and
this repo's mirror alike.  The repo's optional `.albedo` (grey F == albedo,
SURVEY.md 8(a) "Albedo") is honoured when present.
"""

from __future__ import annotations

import numpy as np
from scipy import special as sps

from .numerics import PI_POW_1_5, SQRT_PI, TWO_PI, erfc, frame_about, gauss_cdf, gauss_pdf
from .numerics import log_gauss_cdf, to_world, unit, vdot


class OracleDomainError(ValueError):
    """Mirror of the reference's ParameterDomain / DegenerateVisibility raises."""


def kind_of(medium):
    k = medium.kind
    return getattr(k, "value", k)


def rough(medium):
    """(ax, ay, az) with az forced to 0 for height-field kinds (medium.py:58-61)."""
    a3 = medium.a3
    az = a3.az if kind_of(medium) == "generalized" else 0.0
    return float(a3.ax), float(a3.ay), float(az)


# ---------------------------------------------------------------------------
# height-field NDFs (ndf.py:85-103)


def beckmann_d(wm, ax, ay):
    wm = np.asarray(wm, dtype=np.float64)
    z = wm[..., 2]
    upper = z > 0.0
    z2 = np.where(upper, z * z, 1.0)
    e = (wm[..., 0] / ax) ** 2 + (wm[..., 1] / ay) ** 2
    return np.where(upper, np.exp(-e / z2) / (np.pi * ax * ay * z2 * z2), 0.0)


def ggx_d(wm, ax, ay):
    wm = np.asarray(wm, dtype=np.float64)
    z = wm[..., 2]
    upper = z > 0.0
    t = (wm[..., 0] / ax) ** 2 + (wm[..., 1] / ay) ** 2 + np.where(upper, z * z, 1.0)
    return np.where(upper, 1.0 / (np.pi * ax * ay * t * t), 0.0)


# ---------------------------------------------------------------------------
# projected area sigma(w) = Lambda(w) cos(theta) (ndf.py:110-194)


def projected_area_erf(w, ax, ay, az):
    """Stable re-association, ndf.py:156-164."""
    w = np.asarray(w, dtype=np.float64)
    s = np.sqrt((ax * w[..., 0]) ** 2 + (ay * w[..., 1]) ** 2 + (az * w[..., 2]) ** 2)
    z = w[..., 2]
    ok = s > 0.0
    a = np.where(ok, z / np.where(ok, s, 1.0), np.where(z >= 0.0, np.inf, -np.inf))
    ea = np.where(np.isfinite(a), np.exp(-a * a), 0.0)
    return np.maximum(s * ea / (2.0 * SQRT_PI) - 0.5 * z * erfc(a), 0.0)


def projected_area_ggx(w, ax, ay):
    """ndf.py:167-171."""
    w = np.asarray(w, dtype=np.float64)
    z = w[..., 2]
    return 0.5 * (np.sqrt(z * z + (ax * w[..., 0]) ** 2 + (ay * w[..., 1]) ** 2) - z)


def projected_area(w, kind, ax, ay, az):
    """ndf.py:180-186 (kind dispatch; Beckmann forces az = 0)."""
    if kind == "ggx":
        return projected_area_ggx(w, ax, ay)
    return projected_area_erf(w, ax, ay, az if kind == "generalized" else 0.0)


def projected_area_bound(kind, ax, ay, az):
    """Direction-free majorant factor, ndf.py:189-194."""
    if kind == "ggx":
        return 0.5 * (max(1.0, ax, ay) + 1.0)
    zz = az if kind == "generalized" else 0.0
    return float(np.sqrt(ax * ax + ay * ay + zz * zz) / (2.0 * SQRT_PI) + 1.0)


def smith_lambda(w, ax, ay, az):
    """ndf.py:120-135 (raises at |a| < 1e-9)."""
    w = np.asarray(w, dtype=np.float64)
    s = np.sqrt((ax * w[..., 0]) ** 2 + (ay * w[..., 1]) ** 2 + (az * w[..., 2]) ** 2)
    z = w[..., 2]
    with np.errstate(divide="ignore", invalid="ignore"):
        a = np.where(s > 0.0, z / np.where(s > 0.0, s, 1.0), np.inf * np.sign(z))
    if np.any(np.abs(a) < 1e-9):
        raise OracleDomainError("Lambda singular at grazing")
    return np.exp(-a * a) / (2.0 * a * SQRT_PI) - 0.5 * erfc(a)


# ---------------------------------------------------------------------------
# generalized full-sphere NDF, Eq. 24 (ndf.py:201-224)


def generalized_d(wm, ax, ay, az):
    if az <= 0.0:
        raise OracleDomainError("generalized NDF requires az > 0")
    wm = np.asarray(wm, dtype=np.float64)
    qa = (wm[..., 0] / ax) ** 2 + (wm[..., 1] / ay) ** 2 + (wm[..., 2] / az) ** 2
    qb = wm[..., 2] / (az * az)
    qc = 1.0 / (az * az)
    r = qb * qb / qa
    t1 = np.exp(-qc) * (r + 1.0) / (2.0 * qa * qa)
    t2 = (np.exp(r - qc) * (qb * SQRT_PI / (2.0 * qa ** 2.5)) * (r + 1.5)
          * erfc(-qb / np.sqrt(qa)))
    return np.maximum((t1 + t2) / (PI_POW_1_5 * ax * ay * az), 0.0)


def ndf(wm, kind, ax, ay, az):
    """ndf.py:299-304."""
    if kind == "beckmann":
        return beckmann_d(wm, ax, ay)
    if kind == "ggx":
        return ggx_d(wm, ax, ay)
    return generalized_d(wm, ax, ay, az)


def vndf(wm, wo, kind, ax, ay, az):
    """<-wo, wm>+ D(wm) / sigma(wo), raising when sigma < 1e-12 (ndf.py:307-315)."""
    wm = np.asarray(wm, dtype=np.float64)
    wo = np.asarray(wo, dtype=np.float64)
    sig = projected_area(wo, kind, ax, ay, az)
    if np.any(np.asarray(sig) < 1e-12):
        raise OracleDomainError("projected area numerically zero toward wo")
    return np.maximum(-vdot(wo, wm), 0.0) * ndf(wm, kind, ax, ay, az) / sig


# ---------------------------------------------------------------------------
# Beckmann visible-normal sampling (ndf.py:318-406)


def visible_slopes_unit(ct, st, u1, u2):
    """Unit-roughness Beckmann visible slopes, 64 fixed safeguarded Newton /
    bisection iterations on the slope-x CDF (ndf.py:318-355)."""
    ct = np.asarray(ct, dtype=np.float64)
    st = np.asarray(st, dtype=np.float64)
    u1 = np.asarray(u1, dtype=np.float64)
    u2 = np.asarray(u2, dtype=np.float64)
    vertical = st < 1e-7
    nu = ct / np.where(vertical, 1.0, st)

    def cdf(x):
        return ct * (SQRT_PI / 2.0) * erfc(-x) + 0.5 * st * np.exp(-x * x)

    goal = u1 * cdf(nu)
    lo = np.minimum(nu, 0.0) - 9.0
    hi = np.array(np.broadcast_to(nu, lo.shape), dtype=np.float64)
    x = 0.5 * (lo + hi)
    for _ in range(64):
        g = cdf(x) - goal
        dg = (ct - x * st) * np.exp(-x * x)
        pos = g > 0.0
        hi = np.where(pos, x, hi)
        lo = np.where(pos, lo, x)
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            xn = x - g / dg
        ok = np.isfinite(xn) & (xn > lo) & (xn < hi)
        nxt = np.where(ok, xn, 0.5 * (lo + hi))
        x = np.where((hi - lo) <= 1e-14 * (1.0 + np.abs(hi)), x, nxt)
    rad = np.sqrt(-np.log1p(-u1))
    sx = np.where(vertical, rad * np.cos(TWO_PI * u2), x)
    sy = np.where(vertical, rad * np.sin(TWO_PI * u2), sps.erfinv(2.0 * u2 - 1.0))
    return sx, sy


def beckmann_visible_normal(v, ax, ay, u1, u2):
    """Stretch / sample / unstretch (ndf.py:358-372)."""
    v = np.asarray(v, dtype=np.float64)
    vs = unit(np.stack([ax * v[..., 0], ay * v[..., 1], v[..., 2]], axis=-1))
    ct = np.clip(vs[..., 2], -1.0, 1.0)
    st = np.hypot(vs[..., 0], vs[..., 1])
    x, y = visible_slopes_unit(ct, st, u1, u2)
    has_az = st > 0.0
    den = np.where(has_az, st, 1.0)
    cp = np.where(has_az, vs[..., 0] / den, 1.0)
    sp = np.where(has_az, vs[..., 1] / den, 0.0)
    sx = ax * (cp * x - sp * y)
    sy = ay * (sp * x + cp * y)
    return unit(np.stack([-sx, -sy, np.ones_like(sx)], axis=-1))


def hemisphere_about(axis, u1, u2):
    """Uniform hemisphere about `axis` (ndf.py:375-380)."""
    z = np.asarray(u1, dtype=np.float64)
    r = np.sqrt(np.maximum(1.0 - z * z, 0.0))
    phi = TWO_PI * np.asarray(u2, dtype=np.float64)
    loc = np.stack(np.broadcast_arrays(r * np.cos(phi), r * np.sin(phi), z), axis=-1)
    return to_world(frame_about(axis), loc)


def mixture_pdf(wm, wo, ax, ay, mix):
    """Exact mixture density of a visible normal (ndf.py:397-405)."""
    v = -np.asarray(wo, dtype=np.float64)
    sig_b = projected_area_erf(wo, ax, ay, 0.0)
    guided = np.asarray(sig_b) > 1e-12
    vm = vdot(v, wm)
    cv = np.maximum(vm, 0.0)
    p_b = np.where(guided, cv * beckmann_d(wm, ax, ay) / np.where(guided, sig_b, 1.0), 0.0)
    p_u = np.where(vm > 0.0, 1.0 / TWO_PI, 0.0)
    r = np.where(guided, mix, 0.0)
    return r * p_b + (1.0 - r) * p_u


def sample_visible_normal(wo, ax, ay, mix, u):
    """Mixture sampler from pre-drawn uniforms u[...,0:3] (ndf.py:383-406)."""
    wo = np.asarray(wo, dtype=np.float64)
    v = -wo
    sig_b = projected_area_erf(wo, ax, ay, 0.0)
    guided = np.asarray(sig_b) > 1e-12
    pick_b = (u[..., 0] < mix) & guided
    wm = np.where(pick_b[..., None],
                  beckmann_visible_normal(v, ax, ay, u[..., 1], u[..., 2]),
                  hemisphere_about(v, u[..., 1], u[..., 2]))
    return wm, mixture_pdf(wm, wo, ax, ay, mix)


# ---------------------------------------------------------------------------
# medium (medium.py:70-207)


def density(f, sigma):
    """phi/Phi of N(0, sigma^2), inverse-Mills series below u=-36 (medium.py:70-88)."""
    u = np.asarray(f, dtype=np.float64) / sigma
    clipped = np.maximum(u, -36.0)
    exact = gauss_pdf(clipped, 1.0) / gauss_cdf(clipped, 1.0)
    with np.errstate(divide="ignore"):
        w = 1.0 / np.where(u < -36.0, u * u, np.inf)
    series = -u / (1.0 - w * (1.0 - w * (3.0 - w * (15.0 - 105.0 * w))))
    return np.where(u < -36.0, series, exact) / sigma


def extinction_local(wo_local, f, medium):
    """rho(f) sigma(wo) with wo already in the local frame (medium.py:91-95)."""
    k = kind_of(medium)
    ax, ay, az = rough(medium)
    return density(f, medium.sigma) * projected_area(wo_local, k, ax, ay, az)


def planar_transmittance(h0, h1, cos_t, w_local, medium):
    """(Phi(h1)/Phi(h0))^(-Lambda) on a flat shell (medium.py:98-124).

    Takes the local travel direction instead of (theta, phi)."""
    k = kind_of(medium)
    if np.any(np.abs(cos_t) < 1e-12):
        raise OracleDomainError("planar transmittance undefined at cos(theta)=0")
    if k == "ggx":
        raise OracleDomainError("closed form covers erf-family Lambda only")
    ax, ay, az = rough(medium)
    lam = projected_area_erf(w_local, ax, ay, az) / cos_t
    var = medium.sigma ** 2
    return np.exp(-lam * (log_gauss_cdf(h1, var) - log_gauss_cdf(h0, var)))


def fresnel_conductor(cos_i, eta, k):
    """Unpolarised conductor Fresnel (medium.py:127-147)."""
    c = np.clip(np.asarray(cos_i, dtype=np.float64), 0.0, 1.0)
    eta = np.asarray(eta, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    c2 = c * c
    s2 = 1.0 - c2
    t0 = eta * eta - k * k - s2
    ab = np.sqrt(np.maximum(t0 * t0 + 4.0 * eta * eta * k * k, 0.0))
    t1 = ab + c2
    a = np.sqrt(np.maximum(0.5 * (ab + t0), 0.0))
    t2 = 2.0 * a * c
    den = t1 + t2
    rs = np.where(den > 0.0, (t1 - t2) / np.where(den > 0.0, den, 1.0), 0.0)
    t3 = c2 * ab + s2 * s2
    t4 = t2 * s2
    rp = rs * (t3 - t4) / np.where(t3 + t4 > 0.0, t3 + t4, 1.0)
    return 0.5 * (rs + rp)


def fresnel_rgb(medium, cos_i):
    """medium.py:150-155, plus the repo's grey-albedo extension."""
    alb = getattr(medium, "albedo", None)
    if alb is not None:
        return np.broadcast_to(np.asarray(alb, dtype=np.float64),
                               np.shape(cos_i) + (3,)).copy()
    if medium.fresnel_one:
        return np.ones(np.shape(cos_i) + (3,))
    return fresnel_conductor(np.asarray(cos_i)[..., None],
                             np.asarray(medium.fresnel_eta), np.asarray(medium.fresnel_k))


def _half(wo_local, wi_local):
    v = -np.asarray(wo_local, dtype=np.float64)
    h = v + np.asarray(wi_local, dtype=np.float64)
    hn = np.linalg.norm(h, axis=-1)
    ok = hn > 1e-12
    h = np.where(ok[..., None], h, np.array([0.0, 0.0, 1.0])) / np.where(ok[..., None],
                                                                        hn[..., None], 1.0)
    return v, h, ok


def phase_eval_local(wo_local, wi_local, medium):
    """F(|v.h|) D_v(h) / (4 |v.h|) per channel (medium.py:158-178)."""
    k = kind_of(medium)
    ax, ay, az = rough(medium)
    v, h, ok = _half(wo_local, wi_local)
    vh = np.abs(vdot(v, h))
    dv = vndf(h, wo_local, k, ax, ay, az)
    val = np.where(ok & (vh > 1e-12), dv / np.where(vh > 0, 4.0 * vh, 1.0), 0.0)
    return val[..., None] * fresnel_rgb(medium, vh)


def phase_pdf_local(wo_local, wi_local, medium):
    """Density of _phase_sample_u's output direction; restated from
    ndf.py:397-405 (mixture pdf of the half vector) and medium.py:186-189
    (half-vector Jacobian 1/(4 v.h)).  Not exported by the reference."""
    ax, ay, _ = rough(medium)
    v, h, ok = _half(wo_local, wi_local)
    vh = vdot(v, h)
    pm = mixture_pdf(h, wo_local, ax, ay, medium.mix_ratio)
    good = ok & (vh > 1e-12)
    return np.where(good, pm / np.where(good, 4.0 * vh, 1.0), 0.0)


def phase_sample_local(wo_local, medium, u):
    """Scattered direction, pdf and per-channel weight from u[...,0:3]
    (medium.py:181-193)."""
    k = kind_of(medium)
    ax, ay, az = rough(medium)
    wo_local = np.asarray(wo_local, dtype=np.float64)
    v = -wo_local
    wm, pm = sample_visible_normal(wo_local, ax, ay, medium.mix_ratio, u)
    vm = vdot(v, wm)
    wi = 2.0 * vm[..., None] * wm - v
    ok = vm > 1e-12
    pdf = np.where(ok, pm / np.where(ok, 4.0 * vm, 1.0), 0.0)
    dv = vndf(wm, wo_local, k, ax, ay, az)
    ratio = np.where(pdf > 0.0, dv / np.where(pm > 0.0, pm, 1.0), 0.0)
    return wi, pdf, ratio[..., None] * fresnel_rgb(medium, np.abs(vm))


def split_two_uniforms(u1, u2, mix):
    """Config-1 convention: two uniforms per query feed the
    reference's three-uniform sampler as (u1, u1', u2) where u1' re-uses the
    branch variable rescaled to [0, 1) inside the chosen branch."""
    u1 = np.asarray(u1, dtype=np.float64)
    take = u1 < mix
    with np.errstate(divide="ignore", invalid="ignore"):
        re = np.where(take, u1 / mix, (u1 - mix) / (1.0 - mix))
    return np.stack([u1, re, np.asarray(u2, dtype=np.float64)], axis=-1)
