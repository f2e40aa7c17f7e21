"""Host-side frame helpers kept for API compatibility (reference core.py:101-174).

These build the `local_frame` arguments callers pass to extinction /
phase_eval / phase_sample; the frame arithmetic of the hot path itself runs
on the device (csrc/mf_math.cuh frame_about / to_local / to_world)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


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
