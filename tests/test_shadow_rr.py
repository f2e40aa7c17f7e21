"""Russian roulette on the renderer's shadow-ray weights (walk(..., rr_min),
csrc/mf_transport.cuh) keeps ratio tracking unbiased (CPU, host build of the
device walker).

Ratio-mode transmittance along fixed rays through the config-3 sphere shell
(region |f| <= 3 sigma, transport.py:161-166) is integrated by quadrature
from the pointwise extinction (medium.py:91-95); the walker's mean weight
must match it within 4 standard errors with and without the roulette, and
the roulette must shorten the walks through the optically thick parts.
"""

import ctypes

import numpy as np

from oracle import microfacet as om
from oracle import numerics as on
from paper_2603_00280_b200 import configs
from paper_2603_00280_b200.scene import to_c_scene

SCENE = configs.config3_scene()
M = SCENE.primitives[0].medium
ORIGIN = np.array([0.0, -4.0, 0.0])
# from grazing the shell to straight through the sphere (two shell crossings)
TARGETS = [(1.02, 0, 0.4), (0.9, 0, 0.3), (0.5, 0, 0.2), (0.0, 0, 0.05)]


def exact_ratio_tr(o, d):
    t = np.linspace(0.0, 8.0, 80001)
    p = o[None, :] + t[:, None] * d[None, :]
    r = np.linalg.norm(p, axis=-1)
    f = r - 1.0
    wl = on.to_local(on.frame_about(p / r[:, None]), np.tile(d, (len(t), 1)))
    ext = np.where(np.abs(f) <= 0.3, om.extinction_local(wl, f, M), 0.0)
    return float(np.exp(-np.trapezoid(ext, t)))


def run(lib, d, n, rr):
    cs = to_c_scene(SCENE)
    o = np.ascontiguousarray(np.tile(ORIGIN, (n, 1)).T, np.float32)
    dd = np.ascontiguousarray(np.tile(d, (n, 1)).T, np.float32)
    st = np.zeros(n, np.int32)
    pos = np.zeros((3, n), np.float32)
    w = np.zeros(n, np.float32)
    viol = ctypes.c_int64()
    assert lib.mfh_walk(ctypes.byref(cs), o.ctypes.data_as(ctypes.c_void_p),
                        dd.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(n), ctypes.c_uint64(5),
                        1, st.ctypes.data_as(ctypes.c_void_p), pos.ctypes.data_as(ctypes.c_void_p),
                        w.ctypes.data_as(ctypes.c_void_p), ctypes.c_float(1.0),
                        ctypes.byref(viol), ctypes.c_float(rr)) == 0
    assert viol.value == 0
    return w.astype(np.float64)


def test_shadow_roulette_is_unbiased(host_math):
    n = 100000
    for tg in TARGETS:
        d = np.array(tg) - ORIGIN
        d = (d / np.linalg.norm(d)).astype(np.float32).astype(np.float64)
        ex = exact_ratio_tr(ORIGIN, d)
        for rr in (0.0, 0.05, 1.0):
            w = run(host_math, d, n, rr)
            se = max(w.std() / np.sqrt(n), 1e-7)
            assert abs(w.mean() - ex) <= 4 * se + 1e-6, (tg, rr, w.mean(), ex, se)
            if rr > 0.0:
                # surviving weights are either above the threshold or exactly it
                assert np.all((w == 0) | (w >= np.float32(rr) * (1 - 1e-6)))
