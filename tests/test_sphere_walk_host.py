"""The single-sphere tangent-majorant walker (csrc/mf_transport.cuh
sphere_walk, used by the config-3 renders) against quadrature of the
pointwise extinction (medium.py:91-95) along fixed rays -- CPU, host build
of the device code.

Collision walks: escape probability and the distribution of collision
distances (region [-6s, 3s], transport.py:161-166).  Ratio walks: the mean
weight is the transmittance over |f| <= 3s, with and without the shadow
roulette.  Also: no majorant violations, and far fewer iterations than the
stepping walker."""

import ctypes

import numpy as np
import pytest

from oracle import microfacet as om
from oracle import numerics as on
from paper_2603_00280_b200 import configs
from paper_2603_00280_b200.scene import to_c_scene

SCENE = configs.config3_scene()
M = SCENE.primitives[0].medium
ORIGIN = np.array([0.0, -4.0, 0.0])
# straight through the centre, off-centre, grazing the shell, grazing the core
TARGETS = [(0.0, 0, 0.0), (0.5, 0, 0.2), (0.9, 0, 0.3), (1.02, 0, 0.4), (1.25, 0, 0.1),
           (0.55, 0, 0.0)]


def quad(o, d, lo, t_grid=160001):
    t = np.linspace(0.0, 8.0, t_grid)
    p = o[None, :] + t[:, None] * d[None, :]
    r = np.maximum(np.linalg.norm(p, axis=-1), 1e-12)
    f = r - 1.0
    wl = on.to_local(on.frame_about(p / r[:, None]), np.tile(d, (len(t), 1)))
    ext = np.where((f >= lo) & (f <= 0.3), om.extinction_local(wl, f, M), 0.0)
    tau = np.concatenate([[0.0], np.cumsum(0.5 * (ext[1:] + ext[:-1]) * np.diff(t))])
    return t, f, tau


def run(lib, d, n, ratio, rr=0.0, sphere=1):
    cs = to_c_scene(SCENE)
    o = np.ascontiguousarray(np.tile(ORIGIN, (n, 1)).T, np.float32)
    dd = np.ascontiguousarray(np.tile(d, (n, 1)).T, np.float32)
    st = np.zeros(n, np.int32)
    steps = np.zeros(n, np.int32)
    pos = np.zeros((3, n), np.float32)
    w = np.zeros(n, np.float32)
    viol = ctypes.c_int64()
    lib.mfh_set_walker(ctypes.c_int(sphere), steps.ctypes.data_as(ctypes.c_void_p))
    try:
        assert lib.mfh_walk(ctypes.byref(cs), o.ctypes.data_as(ctypes.c_void_p),
                            dd.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(n),
                            ctypes.c_uint64(11), 1 if ratio else 0,
                            st.ctypes.data_as(ctypes.c_void_p),
                            pos.ctypes.data_as(ctypes.c_void_p),
                            w.ctypes.data_as(ctypes.c_void_p), ctypes.c_float(1.0),
                            ctypes.byref(viol), ctypes.c_float(rr)) == 0
    finally:
        lib.mfh_set_walker(ctypes.c_int(0), None)
    assert viol.value == 0
    return st, pos.T.astype(np.float64), w.astype(np.float64), steps


def rays():
    for tg in TARGETS:
        d = np.array(tg) - ORIGIN
        yield tg, (d / np.linalg.norm(d)).astype(np.float32).astype(np.float64)


def test_collision_walk_matches_quadrature(host_math):
    n = 100000
    for tg, d in rays():
        st, pos, _, steps = run(host_math, d, n, ratio=False)
        t, f, tau = quad(ORIGIN, d, -0.6)
        p_esc = float(np.exp(-tau[-1])) if not np.any(f < -0.6) else 0.0
        se = np.sqrt(max(p_esc * (1 - p_esc), 1e-5) / n)
        assert abs(np.mean(st == 0) - p_esc) <= 4 * se, (tg, np.mean(st == 0), p_esc)
        # collision distances: the CDF 1 - e^{-tau(t)} at a few distances
        hit = st == 2
        dist = np.linalg.norm(pos - ORIGIN, axis=-1)
        for q in (0.25, 0.5, 0.75):
            if not hit.any():
                break
            tq = np.quantile(dist[hit], q)
            cdf = 1.0 - np.exp(-np.interp(tq, t, tau))
            emp = float(np.mean(hit & (dist <= tq)))
            assert abs(emp - cdf) <= 4 * np.sqrt(cdf * (1 - cdf) / n) + 2e-4, (tg, q, emp, cdf)
        assert steps.mean() < 4.0, (tg, steps.mean())


@pytest.mark.parametrize("rr", [0.0, 0.05])
def test_ratio_walk_matches_quadrature(host_math, rr):
    n = 100000
    for tg, d in rays():
        _, _, w, steps = run(host_math, d, n, ratio=True, rr=rr)
        _, _, tau = quad(ORIGIN, d, -0.3)
        ex = float(np.exp(-tau[-1]))
        # 0 <= w <= 1, so Var(w) <= E[w] (1 - E[w]): a bound that holds even
        # when the rare large weights of a deep shadow are not in the sample
        se = np.sqrt(max(w.var(), ex * (1 - ex)) / n)
        assert abs(w.mean() - ex) <= 4 * se + 1e-7, (tg, rr, w.mean(), ex, se)


def test_fewer_iterations_than_stepping(host_math):
    """The tangent majorant replaces ~6 bounded steps per flight by ~1-2
    exact samples (cut the step count)."""
    n = 20000
    tot_new = tot_old = 0.0
    for tg, d in rays():
        _, _, _, s_new = run(host_math, d, n, ratio=False, sphere=1)
        _, _, _, s_old = run(host_math, d, n, ratio=False, sphere=0)
        tot_new += s_new.mean()
        tot_old += s_old.mean()
    assert tot_new < 0.5 * tot_old, (tot_new, tot_old)
