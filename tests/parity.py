"""Shared parity policy: fp32 device results vs the float64 oracle.

Bar (BASELINE north_star): sigma_t, phase value / pdf and sampled
directions within 1e-5 relative of the oracle on identical inputs.  Inputs
(and medium parameters) are rounded to float32 first and the oracle
consumes exactly those values.  Where float32 cannot represent the
problem to 1e-5 the tolerance follows the conditioning:

* sigma_t: rounding u = f/sigma costs ~u^2 2^-24 relative, so
  tol = max(1e-5, 4 u^2 2^-24) (+ 8 a^2 2^-24 for upward views, a = z/s,
  through sigma(wo)'s e^{-a^2}); values below FLT_MIN * 1e3 in float64
  only need to be tiny on the device (underflow policy).
* phase value: 1e-5 relative.  pdf: 1e-5 relative, loosened to
  4 ulp / (v.h) for near-forward pairs: the pdf carries 1 / (v.h) and
  v.h = (1 + v.wi)/|v + wi| -> 0 cancels in any float32 evaluation (the
  phase value does not: its vNDF numerator carries the same v.h).
* sampled direction: <= 1e-5 rad for >= 99.99 % of queries, and every
  query within max(1e-5, 16 kappa), kappa the angle the oracle's own
  output moves when its uniforms move by one float32 ulp (the sampler's
  inverse-CDF conditioning); pdf_s / weight, which inherit the direction
  error through 1/(v.m) and the NDF exponents near grazing microfacet
  normals, within max(1e-5, 64 kappa, 4 kappa_m) relative (kappa_m: the
  change under a 4-ulp tilt of the microfacet normal) and >= 99.5 % within
  1e-5.  pdf_s / weight values whose float64 value is <= 1e-25 (an NDF
  factor e^{-E}, E > 87, underflows float32) only need to be <= 1e-25 on
  the device.
"""

from __future__ import annotations

import numpy as np

from oracle import microfacet as om

FLT_MIN = 1.1754943508222875e-38
ULP = 2.0 ** -24
TINY = 1e-25   # underflow policy of sampled pdf / weight values


class Obj:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def f32_medium(med):
    """Oracle copy of a repo medium with float32-rounded parameters."""
    return Obj(kind=med.kind, a3=Obj(ax=float(np.float32(med.a3.ax)),
                                     ay=float(np.float32(med.a3.ay)),
                                     az=float(np.float32(med.a3.az))),
               sigma=float(np.float32(med.sigma)), mix_ratio=float(np.float32(med.mix_ratio)),
               fresnel_one=med.fresnel_one, fresnel_eta=med.fresnel_eta,
               fresnel_k=med.fresnel_k, albedo=med.albedo)


def relerr(got, ref, floor=1e-300):
    got = np.asarray(got, dtype=np.float64)
    return np.abs(got - ref) / np.maximum(np.abs(ref), floor)


def angle(a, b):
    a = a / np.linalg.norm(a, axis=-1, keepdims=True)
    b = b / np.linalg.norm(b, axis=-1, keepdims=True)
    return np.arctan2(np.linalg.norm(np.cross(a, b), axis=-1), np.sum(a * b, axis=-1))


def area_conditioning(wo_local, m):
    """Extra relative tolerance of sigma(wo) = s/2 ierfc(a) for upward views:
    e^{-a^2} turns the float32 rounding of a = z/s into ~2 a^2 ulps."""
    w = np.asarray(wo_local, dtype=np.float64)
    kind = getattr(m.kind, "value", m.kind)
    az = m.a3.az if kind == "generalized" else 0.0
    s = np.sqrt((m.a3.ax * w[..., 0]) ** 2 + (m.a3.ay * w[..., 1]) ** 2 + (az * w[..., 2]) ** 2)
    with np.errstate(divide="ignore", invalid="ignore"):
        a = np.where(s > 0, w[..., 2] / np.maximum(s, 1e-300), 0.0)
    a = np.where(a > 0, np.minimum(a, 1e3), 0.0)
    return 8.0 * a * a * ULP


def check_sigma_t(got, f, sigma, ref, extra=0.0):
    u = np.asarray(f, dtype=np.float64) / sigma
    tiny = ref < FLT_MIN * 1e3
    tol = np.maximum(1e-5, 4.0 * u * u * ULP) + extra
    e = relerr(got, ref)
    bad_big = ~tiny & (e > tol)
    bad_tiny = tiny & (np.asarray(got, dtype=np.float64) > FLT_MIN * 1e4)
    return {"max_rel_in_band": float(np.max(e[~tiny & (u >= -6) & (u <= 3)], initial=0.0)),
            "n_bad": int(bad_big.sum() + bad_tiny.sum()), "n": int(len(e))}


def pdf_tolerance(wo, wi, m=None):
    """Per-query pdf tolerance: max(1e-5, 4 ulp / (v.h)) (+ the Beckmann
    projected-area conditioning of sigma_b(wo), ndf.py:387-400)."""
    v = -np.asarray(wo, dtype=np.float64)
    h = v + np.asarray(wi, dtype=np.float64)
    h /= np.maximum(np.linalg.norm(h, axis=-1, keepdims=True), 1e-300)
    vh = np.abs(np.sum(v * h, axis=-1))
    extra = 0.0
    if m is not None:
        beck = Obj(kind="beckmann", a3=Obj(ax=m.a3.ax, ay=m.a3.ay, az=0.0))
        extra = area_conditioning(wo, beck)
    return np.maximum(1e-5, 4.0 * ULP / np.maximum(vh, 1e-300)) + extra


def phase_tolerance(wo, wi, m):
    """max(1e-5, 8 ulp (1 + E)), E the NDF exponent at the half vector: the
    Beckmann e^{-E} (ndf.py:85-94) and the generalized e^{r - c}
    (ndf.py:216-222) turn the float32 rounding of h into ~E ulps."""
    v = -np.asarray(wo, dtype=np.float64)
    h = v + np.asarray(wi, dtype=np.float64)
    h /= np.maximum(np.linalg.norm(h, axis=-1, keepdims=True), 1e-300)
    ax, ay = m.a3.ax, m.a3.ay
    lat = (h[..., 0] / ax) ** 2 + (h[..., 1] / ay) ** 2
    e_beck = lat / np.maximum(h[..., 2] ** 2, 1e-300)
    az = getattr(m.a3, "az", 0.0)
    e_gen = lat / max(az * az, 1e-300) / np.maximum(lat + (h[..., 2] / max(az, 1e-300)) ** 2,
                                                     1e-300)
    kind = getattr(m.kind, "value", m.kind)
    e = e_beck if kind == "beckmann" else e_gen
    # the vNDF divides by sigma(wo) (ndf.py:315), whose e^{-a^2} conditions it
    return np.maximum(1e-5, 8.0 * ULP * (1.0 + np.minimum(e, 1e6))) + area_conditioning(wo, m)


def check_rel(got, ref, tol=1e-5, floor=1e-30):
    ok = np.abs(ref) > floor
    e = relerr(got, ref)
    bad = (ok & (e > tol)) | (~ok & (np.abs(np.asarray(got, dtype=np.float64)) > 1e-20))
    return {"max_rel": float(np.max(e[ok], initial=0.0)), "n_bad": int(bad.sum()),
            "n": int(len(e))}


def oracle_sample(wo, m, u1, u2):
    """Oracle phase sample for the two-uniform convention; u1, u2 float32."""
    mix = np.float32(m.mix_ratio)
    u1 = np.asarray(u1, dtype=np.float32)
    uu = np.where(u1 < mix, u1 / mix, (u1 - mix) / (np.float32(1) - mix)).astype(np.float32)
    U3 = np.stack([u1, uu, np.asarray(u2, dtype=np.float32)], axis=-1).astype(np.float64)
    return om.phase_sample_local(wo, m, U3)


def _f(m):
    """Grey Fresnel / albedo factor of channel 0 (F == 1 or albedo media)."""
    alb = getattr(m, "albedo", None)
    if alb is not None:
        return float(np.ravel(alb)[0])
    return 1.0


def check_samples(ws, pdf_s, w, wo, m, u1, u2):
    """Direction / pdf / weight of sampled directions vs the oracle, with the
    conditioning-scaled tolerance of the module docstring."""
    ws_r, pdf_r, w_r = oracle_sample(wo, m, u1, u2)
    u1 = np.asarray(u1, dtype=np.float32)
    u2 = np.asarray(u2, dtype=np.float32)
    # one-ulp perturbations of each uniform (kept inside [0, 1))
    u1p = np.nextafter(u1, np.float32(1)).astype(np.float32)
    u2p = np.nextafter(u2, np.float32(1)).astype(np.float32)
    ws_a, pdf_a, w_a = oracle_sample(wo, m, u1p, u2)
    ws_b, pdf_b, w_b = oracle_sample(wo, m, u1, u2p)
    kap_dir = angle(ws_a, ws_r) + angle(ws_b, ws_r)
    kap_pdf = relerr(pdf_a, pdf_r, 1e-30) + relerr(pdf_b, pdf_r, 1e-30)
    kap_w = relerr(w_a[:, 0], w_r[:, 0], 1e-30) + relerr(w_b[:, 0], w_r[:, 0], 1e-30)
    # sensitivity of pdf_s / weight to rounding the microfacet normal itself
    # (4 ulp tilts along two tangents): grazing normals make the Beckmann /
    # generalized exponents amplify it
    kind = getattr(m.kind, "value", m.kind)
    ax, ay, az = m.a3.ax, m.a3.ay, (m.a3.az if kind == "generalized" else 0.0)
    v = -np.asarray(wo, dtype=np.float64)
    wm = v + ws_r
    wm /= np.linalg.norm(wm, axis=-1, keepdims=True)
    helper = np.where(np.abs(wm[:, :1]) < 0.9, np.array([[1.0, 0, 0]]), np.array([[0, 1.0, 0]]))
    t1 = np.cross(wm, helper)
    t1 /= np.linalg.norm(t1, axis=-1, keepdims=True)
    t2 = np.cross(wm, t1)
    kap_pdf_m = np.zeros(len(wm))
    kap_w_m = np.zeros(len(wm))
    with np.errstate(all="ignore"):
        for t in (t1, t2):
            wp = wm + 4.0 * ULP * t
            wp /= np.linalg.norm(wp, axis=-1, keepdims=True)
            pm = om.mixture_pdf(wp, wo, ax, ay, m.mix_ratio)
            vm = np.sum(v * wp, axis=-1)
            pdf_p = np.where(vm > 1e-12, pm / (4.0 * vm), 0.0)
            dv = np.maximum(vm, 0.0) * om.ndf(wp, kind, ax, ay, az) / \
                om.projected_area(wo, kind, ax, ay, az)
            w_p = np.where(pm > 0, dv / np.where(pm > 0, pm, 1.0), 0.0)
            kap_pdf_m += relerr(pdf_p, pdf_r, 1e-30)
            kap_w_m += relerr(w_p, w_r[:, 0] / np.maximum(_f(m), 1e-300), 1e-30)
    ang = angle(np.asarray(ws, dtype=np.float64), ws_r)
    tol_dir = np.maximum(1e-5, 16.0 * kap_dir)
    e_pdf = relerr(pdf_s, pdf_r, 1e-30)
    e_w = relerr(np.asarray(w)[:, 0], w_r[:, 0], 1e-30)
    tol_pdf = np.maximum(1e-5, np.maximum(64.0 * kap_pdf, 4.0 * kap_pdf_m))
    tol_w = np.maximum(1e-5, np.maximum(64.0 * kap_w, 4.0 * kap_w_m))
    # underflow policy (as for sigma_t): an NDF factor e^{-E} with E > 87
    # is below FLT_MIN in float32 -- such weights (float64 <= 1e-25) only
    # need to be tiny on the device
    tiny_w = (np.abs(w_r[:, 0]) <= TINY) & (np.abs(np.asarray(w)[:, 0]) <= TINY)
    e_w = np.where(tiny_w, 0.0, e_w)
    tiny_p = (np.abs(pdf_r) <= TINY) & (np.abs(np.asarray(pdf_s)) <= TINY)
    e_pdf = np.where(tiny_p, 0.0, e_pdf)
    return {
        "frac_dir_within_1e-5": float(np.mean(ang <= 1e-5)),
        "max_angle": float(ang.max()),
        "n_dir_bad": int(np.sum(ang > tol_dir)),
        "frac_pdf_within_1e-5": float(np.mean(e_pdf <= 1e-5)),
        "n_pdf_bad": int(np.sum(e_pdf > tol_pdf)),
        "frac_w_within_1e-5": float(np.mean(e_w <= 1e-5)),
        "n_w_bad": int(np.sum(e_w > tol_w)),
        "n": int(len(ang)),
    }


def _samples_chunk(args):
    return check_samples(*args)


def check_samples_pool(ws, pdf_s, w, wo, m, u1, u2, chunk=1 << 15):
    """check_samples over a fork pool of the host cores (the float64 oracle
    sampler is the slow part), chunk by chunk; merged counts / fractions."""
    import multiprocessing as mp
    import os

    n = len(ws)
    jobs = [(ws[a:a + chunk], pdf_s[a:a + chunk], w[a:a + chunk], wo[a:a + chunk], m,
             u1[a:a + chunk], u2[a:a + chunk]) for a in range(0, n, chunk)]
    workers = max(1, min(len(jobs), len(os.sched_getaffinity(0))))
    if workers == 1:
        parts = [_samples_chunk(j) for j in jobs]
    else:
        with mp.get_context("fork").Pool(workers) as pool:
            parts = pool.map(_samples_chunk, jobs)
    out = {"n": sum(p["n"] for p in parts),
           "max_angle": max(p["max_angle"] for p in parts)}
    for k in ("frac_dir_within_1e-5", "frac_pdf_within_1e-5", "frac_w_within_1e-5"):
        out[k] = sum(p[k] * p["n"] for p in parts) / out["n"]
    for k in ("n_dir_bad", "n_pdf_bad", "n_w_bad"):
        out[k] = sum(p[k] for p in parts)
    return out
