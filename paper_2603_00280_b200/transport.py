"""Ratio-tracking transmittance on the GPU (reference transport.py:300-313)."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import ParameterDomainError
from .scene import ShellScene, to_c_scene


def transmittance_estimate(ray, scene: ShellScene, n_samples, rng):
    """Unbiased ratio-tracking estimate through all shell intervals along
    the ray (region |f| <= 3 sigma); returns (mean, std_error)."""
    n = int(n_samples)
    if n < 1:
        raise ParameterDomainError(f"n_samples must be >= 1, got {n}")
    torch = _lib.require_cuda()
    lib = _lib.load()
    origin, direction = ray
    o = (ctypes.c_double * 3)(*np.asarray(origin, dtype=np.float64).tolist())
    d = (ctypes.c_double * 3)(*np.asarray(direction, dtype=np.float64).tolist())
    mean = ctypes.c_double()
    se = ctypes.c_double()
    if not scene.primitives:
        return 1.0, 0.0
    cs = to_c_scene(scene)
    _lib.check(lib.mf_transmittance(ctypes.byref(cs), o, d, n, int(rng.seed) & (2**64 - 1),
                                    int(rng.stream) & (2**64 - 1), ctypes.byref(mean),
                                    ctypes.byref(se), _lib.stream_handle(torch)))
    return float(mean.value), float(se.value)
