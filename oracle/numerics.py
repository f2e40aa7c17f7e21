"""Oracle numerics: special functions, frames and the SplitMix64 streams.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  float64 throughout,
restating the reference's L0 layer:

* erfc with the Laplace continued-fraction tail   -- core.py:36-68
* Gaussian pdf / cdf / log-cdf                     -- core.py:71-98
* Duff branchless frame, to_local / to_world       -- core.py:132-169
* SplitMix64 counter streams                       -- rng.py:24-58
* per-ray counter batch (BatchRng)                 -- transport.py:52-67

The third-party arithmetic the reference calls is scipy.special
(erf, erfc, erfinv, log_ndtr; pinned only as scipy>=1.10 in
pyproject.toml:10-13; validated here with scipy 1.18.1).
"""

from __future__ import annotations

import numpy as np
from scipy import special as sps

SQRT_PI = 1.7724538509055160273
TWO_PI = 6.283185307179586
PI_POW_1_5 = np.pi ** 1.5

# ---------------------------------------------------------------------------
# erfc with a relatively accurate upper tail (core.py:36-68)

_CF_START = 8.0      # core.py:25
_CF_TERMS = 48       # core.py:26


def _exp_minus_square(x):
    """e^{-x^2}, compensating the rounding of x*x (Veltkamp split, core.py:36-44)."""
    sq = x * x
    split = x * 134217729.0
    hi = split - (split - x)
    lo = x - hi
    resid = (hi * hi - sq) + 2.0 * hi * lo + lo * lo
    return np.exp(-sq) * (1.0 - resid)


def _laplace_tail(x):
    """Laplace continued fraction of erfc, evaluated bottom-up (core.py:47-52)."""
    acc = np.zeros_like(x)
    for k in range(_CF_TERMS, 0, -1):
        acc = (0.5 * k) / (x + acc)
    return _exp_minus_square(x) / (SQRT_PI * (x + acc))


def erfc(x):
    """core.py:55-68: scipy below x=8, continued fraction above (clamped at 30)."""
    x = np.asarray(x, dtype=np.float64)
    res = sps.erfc(x)
    big = x > _CF_START
    if np.any(big):
        xs = np.minimum(np.where(big, x, _CF_START), 30.0)
        res = np.where(big, _laplace_tail(xs), res)
    return res[()]


def gauss_pdf(x, var):
    """Centered Gaussian density (core.py:71-78 with mu=0)."""
    x = np.asarray(x, dtype=np.float64)
    return np.exp(-(x * x) / (2.0 * var)) / np.sqrt(TWO_PI * var)


def gauss_cdf(x, var):
    """Centered Gaussian cdf through erfc (core.py:81-89 with mu=0)."""
    x = np.asarray(x, dtype=np.float64)
    return 0.5 * erfc(-x / np.sqrt(2.0 * var))


def log_gauss_cdf(x, var):
    """log cdf via scipy log_ndtr (core.py:92-98 with mu=0)."""
    return sps.log_ndtr(np.asarray(x, dtype=np.float64) / np.sqrt(var))


# ---------------------------------------------------------------------------
# vectors and frames (core.py:101-174)


def vdot(a, b):
    return np.sum(np.asarray(a) * np.asarray(b), axis=-1)


def unit(v):
    v = np.asarray(v, dtype=np.float64)
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def frame_about(n):
    """Duff et al. branchless basis (core.py:156-169); returns (t, b, n)."""
    n = np.asarray(n, dtype=np.float64)
    nx, ny, nz = n[..., 0], n[..., 1], n[..., 2]
    sgn = np.copysign(1.0, nz)
    a = -1.0 / (sgn + nz)
    b = nx * ny * a
    t = np.stack([1.0 + sgn * nx * nx * a, sgn * b, -sgn * nx], axis=-1)
    bt = np.stack([b, sgn + ny * ny * a, -ny], axis=-1)
    return t, bt, n


def to_local(frame, w):
    """core.py:140-145."""
    t, b, n = frame
    w = np.asarray(w, dtype=np.float64)
    return np.stack([vdot(w, t), vdot(w, b), vdot(w, n)], axis=-1)


def to_world(frame, w):
    """core.py:147-153."""
    t, b, n = frame
    w = np.asarray(w, dtype=np.float64)
    return w[..., 0:1] * t + w[..., 1:2] * b + w[..., 2:3] * n


# ---------------------------------------------------------------------------
# SplitMix64 counter streams (rng.py:24-58)

_U = np.uint64
_PHI = _U(0x9E3779B97F4A7C15)
_M1 = _U(0xBF58476D1CE4E5B9)
_M2 = _U(0x94D049BB133111EB)


def _finalize(z):
    z = (z ^ (z >> _U(30))) * _M1
    z = (z ^ (z >> _U(27))) * _M2
    return z ^ (z >> _U(31))


def stream_base(seed, stream):
    """rng.py:31-36."""
    with np.errstate(over="ignore"):
        s = np.asarray(seed, dtype=np.uint64)
        k = np.asarray(stream, dtype=np.uint64)
        return _finalize(_finalize(s * _PHI + _U(1)) ^ (k * _M2 + _U(1)))


def uniform_at(base, counter):
    """53-bit uniform of the counter-th draw (rng.py:39-48)."""
    with np.errstate(over="ignore"):
        raw = _finalize(np.asarray(base, dtype=np.uint64)
                        + np.asarray(counter, dtype=np.uint64) * _PHI)
    return (raw >> _U(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def child_bases(seed, stream, indices):
    """rng.py:51-58 (RandomStream.derive, vectorised)."""
    with np.errstate(over="ignore"):
        kid = _finalize(np.asarray(stream, dtype=np.uint64) * _PHI
                        ^ np.asarray(indices, dtype=np.uint64) * _M1 + _U(1))
    return stream_base(seed, kid)


class RayStreams:
    """Per-ray counters that only advance for rays that draw (transport.py:52-67)."""

    def __init__(self, base, counter):
        self.base = np.asarray(base, dtype=np.uint64)
        self.counter = np.array(counter, dtype=np.uint64)

    def draw(self, mask=None):
        u = uniform_at(self.base, self.counter)
        step = _U(1) if mask is None else np.asarray(mask, dtype=np.uint64)
        self.counter = self.counter + step
        return u

    def subset(self, idx):
        return RayStreams(self.base[idx], self.counter[idx])

    def merge(self, idx, sub):
        self.counter[idx] = sub.counter
