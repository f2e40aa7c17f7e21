"""A defect of the reference walker, and the evidence that this build does
not share it (CPU only).

transport.py:88-91 picks the sphere root as `t1 if t1 > 1e-12 else t2`.
After a vacuum skip lands a ray on a sphere's level set, rounding leaves it
a hair outside about half the time; t1 ~ 0 then selects the FAR root and the
ray tunnels through the shell and core and escapes.  Transmittance along
fixed rays, integrated by quadrature from the pointwise extinction
(medium.py:91-95), exposes the bias; the oracle's corrected root selection
and the host build of the device walker both match the quadrature.
"""

import ctypes

import numpy as np
import pytest

from oracle import microfacet as om
from oracle import numerics as on
from oracle import tracer as ot
from paper_2603_00280_b200 import configs
from paper_2603_00280_b200.scene import to_c_scene

SCENE = configs.config3_scene()
M = SCENE.primitives[0].medium
ORIGIN = np.array([0.0, -4.0, 0.0])
TARGETS = [(0.8, 0, 0.8), (1.0, 0, 0.5), (0.3, 0, 1.1), (-1.03, 0, 0.49), (0.46195589, 0, -0.25782752)]


def exact_escape(o, d):
    t = np.linspace(0.0, 8.0, 40001)
    p = o[None, :] + t[:, None] * d[None, :]
    r = np.linalg.norm(p, axis=-1)
    f = r - 1.0
    if np.any(f < -0.6):
        return 0.0
    wl = on.to_local(on.frame_about(p / r[:, None]), np.tile(d, (len(t), 1)))
    ext = np.where((f >= -0.6) & (f <= 0.3), om.extinction_local(wl, f, M), 0.0)
    return float(np.exp(-np.trapezoid(ext, t)))


def rays():
    out = []
    for tg in TARGETS:
        d = np.array(tg) - ORIGIN
        d = (d / np.linalg.norm(d)).astype(np.float32).astype(np.float64)
        out.append(d)
    return out


def oracle_escape(d, n, policy):
    old = ot.SPHERE_ROOTS
    ot.SPHERE_ROOTS = policy
    try:
        rs = on.RayStreams(on.child_bases(9, 0, np.arange(n)), np.zeros(n, np.uint64))
        st, _, _, _, _ = ot.walk(SCENE.primitives, np.tile(ORIGIN, (n, 1)), np.tile(d, (n, 1)), rs)
    finally:
        ot.SPHERE_ROOTS = old
    return float(np.mean(st == 0))


def test_reference_root_selection_tunnels():
    n = 4000
    worst_ref = worst_fix = 0.0
    for d in rays():
        ex = exact_escape(ORIGIN, d)
        se = np.sqrt(max(ex * (1 - ex), 1e-4) / n)
        worst_ref = max(worst_ref, abs(oracle_escape(d, n, "reference") - ex) / se)
        worst_fix = max(worst_fix, abs(oracle_escape(d, n, "corrected") - ex) / se)
    assert worst_fix < 4.0
    assert worst_ref > 6.0   # the reference's own walker is measurably biased


def test_device_walker_matches_quadrature(host_math):
    cs = to_c_scene(SCENE)
    n = 200000
    for d in rays():
        o = np.ascontiguousarray(np.tile(ORIGIN, (n, 1)).T, np.float32)
        dd = np.ascontiguousarray(np.tile(d, (n, 1)).T, np.float32)
        st = np.zeros(n, np.int32)
        pos = np.zeros((3, n), np.float32)
        w = np.zeros(n, np.float32)
        viol = ctypes.c_int64()
        assert host_math.mfh_walk(ctypes.byref(cs), o.ctypes.data_as(ctypes.c_void_p),
                                  dd.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(n),
                                  ctypes.c_uint64(3), 0, st.ctypes.data_as(ctypes.c_void_p),
                                  pos.ctypes.data_as(ctypes.c_void_p),
                                  w.ctypes.data_as(ctypes.c_void_p), ctypes.c_float(1.0),
                                  ctypes.byref(viol), ctypes.c_float(0.0)) == 0
        ex = exact_escape(ORIGIN, d)
        se = np.sqrt(max(ex * (1 - ex), 1e-5) / n)
        assert abs(np.mean(st == 0) - ex) <= 4 * se, (d, np.mean(st == 0), ex)
        assert viol.value == 0
