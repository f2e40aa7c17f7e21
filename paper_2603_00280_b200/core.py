"""Host-side frame helpers kept for API compatibility (reference core.py:101-174).

These build the `local_frame` arguments callers pass to extinction /
phase_eval / phase_sample; the frame arithmetic of the hot path itself runs
on the device (csrc/mf_math.cuh frame_about / to_local / to_world)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


TWO_PI = 2.0 * np.pi


def _special(which, x):
    """float64 erf / erfc / exp(-x) of an array on the device
    (mf_special_f64)."""
    import ctypes

    from . import _lib

    torch = _lib.require_cuda()
    lib = _lib.load()
    x = np.asarray(x, dtype=np.float64)
    dev = torch.device("cuda", torch.cuda.current_device())
    t = torch.from_numpy(np.ascontiguousarray(x.reshape(-1))).to(dev)
    out = torch.empty_like(t)
    _lib.check(lib.mf_special_f64(which, ctypes.c_void_p(t.data_ptr()), t.numel(),
                                  ctypes.c_void_p(out.data_ptr()), _lib.stream_handle(torch, dev)))
    return out.cpu().numpy().reshape(x.shape)[()]


def erf(x):
    """Error function, float64, exactly odd (core.py:29-33), on the device."""
    return _special(0, x)


def erfc(x):
    """Complementary error function, float64 (core.py:55-68), on the device
    (CUDA's erfc keeps relative accuracy through the tail)."""
    return _special(1, x)


def gauss_pdf(x, mu, var):
    """Gaussian density with mean mu and variance var > 0 (core.py:71-78)."""
    from .errors import ParameterDomainError

    var = np.asarray(var, dtype=np.float64)
    if np.any(var <= 0.0):
        raise ParameterDomainError(f"gauss_pdf requires var > 0, got {var}")
    z = (np.asarray(x, dtype=np.float64) - mu) ** 2 / (2.0 * var)
    return (np.asarray(_special(2, z)) / np.sqrt(TWO_PI * var))[()]


def gauss_cdf(x, mu, var):
    """Gaussian CDF through erfc, relative accuracy in the lower tail
    (core.py:81-89)."""
    from .errors import ParameterDomainError

    var = np.asarray(var, dtype=np.float64)
    if np.any(var <= 0.0):
        raise ParameterDomainError(f"gauss_cdf requires var > 0, got {var}")
    z = (np.asarray(mu, dtype=np.float64) - np.asarray(x, dtype=np.float64)) / np.sqrt(2.0 * var)
    return (0.5 * np.asarray(erfc(z)))[()]


def spherical_to_direction(theta, phi):
    """(theta, phi) -> unit direction (..., 3) (core.py:111-119)."""
    theta = np.asarray(theta, dtype=np.float64)
    phi = np.asarray(phi, dtype=np.float64)
    st = np.sin(theta)
    return np.stack(np.broadcast_arrays(st * np.cos(phi), st * np.sin(phi), np.cos(theta)),
                    axis=-1)


def direction_to_spherical(w):
    """Unit direction -> (theta, phi), phi = 0 at the poles (core.py:122-129)."""
    w = np.asarray(w, dtype=np.float64)
    theta = np.arccos(np.clip(w[..., 2], -1.0, 1.0))
    phi = np.mod(np.arctan2(w[..., 1], w[..., 0]), TWO_PI)
    phi = np.where(np.hypot(w[..., 0], w[..., 1]) < 1e-14, 0.0, phi)
    return theta[()], phi[()]


def reflect(v, n):
    """Mirror v about n: 2 (v.n) n - v (core.py:172-174)."""
    return 2.0 * dot(v, n)[..., None] * np.asarray(n) - np.asarray(v)


def normalize(v):
    v = np.asarray(v, dtype=np.float64)
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def dot(a, b):
    return np.sum(np.asarray(a) * np.asarray(b), axis=-1)


@dataclass(frozen=True)
class Frame:
    """Right-handed orthonormal frame; fields broadcast as (..., 3) arrays."""

    tangent: np.ndarray
    bitangent: np.ndarray
    normal: np.ndarray


def build_frame(n):
    """Duff et al. branchless frame about unit normal n (core.py:156-169)."""
    n = np.asarray(n, dtype=np.float64)
    s = np.copysign(1.0, n[..., 2])
    a = -1.0 / (s + n[..., 2])
    b = n[..., 0] * n[..., 1] * a
    t = np.stack([1.0 + s * n[..., 0] ** 2 * a, s * b, -s * n[..., 0]], axis=-1)
    bt = np.stack([b, s + n[..., 1] ** 2 * a, -n[..., 1]], axis=-1)
    return Frame(tangent=t, bitangent=bt, normal=n)
