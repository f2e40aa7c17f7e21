"""Fit the fp32 polynomial approximations used by csrc/mf_math.cuh.

Every special function the device needs is reduced to a smooth function
on [0, inf) mapped to t = (x - K) / (x + K) in [-1, 1) and approximated by
a polynomial in t (Lawson-reweighted least squares ~ minimax relative
error).  Ground truth is float64: scipy.special.erfcx / erfcinv, and for the
cancelling combinations the Laplace continued fraction rearranged so that
nothing cancels (see _cf_levels); tests/test_math_host.py re-checks the
resulting fp32 code against mpmath at 30 digits.  The script prints a
C header fragment; its output is pasted into mf_math.cuh (the numbers in
the header are this script's output, nothing else).

    python tools/fit_approx.py > /tmp/coeffs.h
"""

from __future__ import annotations

import sys

import numpy as np
from scipy import special as sps

SQPI = np.sqrt(np.pi)
CF_TERMS = 400


def _cf_levels(x):
    """Bottom-up Laplace continued fraction of sqrt(pi) erfcx(x) = 1/(x + c1),
    c_k = (k/2) / (x + c_{k+1}); returns (c1, c2, c3).  Stable (no
    cancellation) and accurate for x >= 1.5 with CF_TERMS levels."""
    c = np.zeros_like(x)
    keep = {}
    for k in range(CF_TERMS, 0, -1):
        c = (0.5 * k) / (x + c)
        if k <= 3:
            keep[k] = c
    return keep[1], keep[2], keep[3]


def f_erfcx(x):
    return sps.erfcx(x)


def f_ierfcx(x):
    """e^{x^2} * int_x^inf erfc = 1/sqrt(pi) - x erfcx(x)."""
    x = np.asarray(x, dtype=np.float64)
    direct = 1.0 / SQPI - x * sps.erfcx(x)
    c1, _, _ = _cf_levels(np.maximum(x, 1.5))
    cf = c1 / ((x + c1) * SQPI)
    return np.where(x < 1.5, direct, cf)


def f_bterm(x):
    """(1 + x^2) - sqrt(pi) x (x^2 + 3/2) erfcx(x), the cancelling bracket of
    Eq. 24 for downward normals; equals c3 / (2 (x+c1)(x+c2)(x+c3))."""
    x = np.asarray(x, dtype=np.float64)
    direct = (1.0 + x * x) - SQPI * x * (x * x + 1.5) * sps.erfcx(x)
    c1, c2, c3 = _cf_levels(np.maximum(x, 1.5))
    cf = 0.5 * c3 / ((x + c1) * (x + c2) * (x + c3))
    return np.where(x < 1.5, direct, cf)


def fit(func, scale, K, deg, n=3000, iters=30):
    """Fit P(t) ~ scale(x) * func(x), x = K (1+t)/(1-t)."""
    # Chebyshev-distributed nodes in t, clipped away from t=1 (x=inf)
    k = np.arange(n)
    t = np.cos(np.pi * (k + 0.5) / n)
    t = np.clip(t, -1.0, 1.0 - 1e-9)
    x = K * (1 + t) / (1 - t)
    y = scale(x) * func(x)
    V = np.vander(t, deg + 1, increasing=True)
    w = np.ones(n)
    for _ in range(iters):
        A = V * (w / np.abs(y))[:, None]
        b = w * np.sign(y)
        c, *_ = np.linalg.lstsq(A, b, rcond=None)
        err = np.abs(V @ c - y) / np.abs(y)
        w = w * np.sqrt(err / err.max() + 1e-3)
        w /= w.mean()
    return c, err.max()


def horner32(c, t):
    t = np.float32(t)
    acc = np.float32(c[-1])
    for ci in c[-2::-1]:
        acc = np.float32(acc * t + np.float32(ci))
    return acc


def check32(func, scale, K, c, xs):
    x32 = np.asarray(xs, dtype=np.float32)
    t = ((x32 - np.float32(K)) / (x32 + np.float32(K))).astype(np.float32)
    acc = np.full_like(t, np.float32(c[-1]))
    for ci in c[-2::-1]:
        acc = (acc * t + np.float32(ci)).astype(np.float32)
    x64 = x32.astype(np.float64)
    got = acc.astype(np.float64) / scale(x64)
    ref = func(x64)
    return float(np.max(np.abs(got - ref) / np.abs(ref)))


def fit_erfinv(lo_w, hi_w, deg, transform, inverse, n=2000, iters=30):
    """erfinv(x)/x as a polynomial in s = transform(w), w = -log((1-x)(1+x))."""
    s_lo, s_hi = transform(lo_w), transform(hi_w)
    k = np.arange(n)
    s = s_lo + (s_hi - s_lo) * 0.5 * (1 - np.cos(np.pi * (k + 0.5) / n))
    w = inverse(s)
    # (1-x)(1+x) = e^{-w}; 1 - x = e^{-w} / (1 + sqrt(1 - e^{-w})) without cancellation
    e = np.exp(-w)
    x = np.sqrt(-np.expm1(-w))
    y = sps.erfcinv(e / (1.0 + x)) / x
    V = np.vander(s, deg + 1, increasing=True)
    wt = np.ones(n)
    for _ in range(iters):
        A = V * (wt / np.abs(y))[:, None]
        c, *_ = np.linalg.lstsq(A, wt * np.sign(y), rcond=None)
        err = np.abs(V @ c - y) / np.abs(y)
        wt = wt * np.sqrt(err / err.max() + 1e-3)
        wt /= wt.mean()
    return c, err.max()


def _lit(v):
    return repr(float(np.float32(v))) + "f"


def emit(name, c, comment):
    """A Horner-form inline function (explicit constants work in both
    host and device code without device-side constant arrays)."""
    print(f"// {comment}")
    print(f"MF_HD float {name}(float t) {{")
    print(f"  float p = {_lit(c[-1])};")
    for ci in c[-2::-1]:
        print(f"  p = fmaf(p, t, {_lit(ci)});")
    print("  return p;")
    print("}")


def main():
    out = {}
    xs_check = np.concatenate([np.linspace(0, 4, 400), np.geomspace(4, 1e6, 400)])

    # scales are powers of (x + K) so that a single reciprocal r = 1/(x+2)
    # gives both t = 1 - 4r and the scale: f(x) = P(t) * r^k
    K = 2.0
    c, e = fit(f_erfcx, lambda x: x + 2.0, K, 13)
    e32 = check32(f_erfcx, lambda x: x + 2.0, K, c, xs_check)
    print(f"// erfcx: K={K} fit max rel {e:.2e}, fp32 Horner max rel {e32:.2e}", file=sys.stderr)
    out["MF_ERFCX_P"] = (c, K)

    K = 2.0
    c, e = fit(f_ierfcx, lambda x: (x + 2.0) ** 2, K, 14)
    e32 = check32(f_ierfcx, lambda x: (x + 2.0) ** 2, K, c, xs_check)
    print(f"// ierfcx: K={K} fit max rel {e:.2e}, fp32 Horner max rel {e32:.2e}", file=sys.stderr)
    out["MF_IERFCX_P"] = (c, K)

    K = 2.0
    c, e = fit(f_bterm, lambda x: (x + 2.0) ** 4, K, 16)
    e32 = check32(f_bterm, lambda x: (x + 2.0) ** 4, K, c, xs_check)
    print(f"// bterm: K={K} fit max rel {e:.2e}, fp32 Horner max rel {e32:.2e}", file=sys.stderr)
    out["MF_BTERM_P"] = (c, K)

    # erfinv(x) / x, central: s = w - 2.5 on w in [0, 5]; tail: s = sqrt(w) - 3, w in [5, 90]
    c1, e1 = fit_erfinv(1e-12, 5.0, 9, lambda w: w - 2.5, lambda s: s + 2.5)
    c2, e2 = fit_erfinv(5.0, 90.0, 13, lambda w: np.sqrt(w) - 3.0, lambda s: (s + 3.0) ** 2)
    print(f"// erfinv central max rel {e1:.2e}, tail max rel {e2:.2e}", file=sys.stderr)

    print("// ---- generated by tools/fit_approx.py; do not edit by hand ----")
    notes = {
        "MF_ERFCX_P": "(x+2) erfcx(x) as a polynomial in t = (x-2)/(x+2), x >= 0",
        "MF_IERFCX_P": "(x+2)^2 e^{x^2} ierfc(x) in t = (x-2)/(x+2), x >= 0",
        "MF_BTERM_P": "(x+2)^4 [(1+x^2) - sqrt(pi) x (x^2+3/2) erfcx(x)] in t, x >= 0",
    }
    fn = {"MF_ERFCX_P": "poly_erfcx", "MF_IERFCX_P": "poly_ierfcx", "MF_BTERM_P": "poly_bterm"}
    for name, (c, K) in out.items():
        emit(fn[name], c, notes[name])
    emit("poly_erfinv_central", c1, "erfinv(x)/x in s = w - 2.5, w = -log((1-x)(1+x)) <= 5")
    emit("poly_erfinv_tail", c2, "erfinv(x)/x in s = sqrt(w) - 3, 5 < w <= 90")


if __name__ == "__main__":
    main()
