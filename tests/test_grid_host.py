"""Grid-field walker (csrc/mf_grid.cuh) built for the host (CPU only):
a constant-sigma grid of the plane f = z must reproduce the closed-form
planar transmittance (medium.py:98-124), and the majorant grid must bound
the extinction on the config-5 fields."""

import ctypes
import math

import numpy as np

from oracle import microfacet as om
from paper_2603_00280_b200 import _lib
from paper_2603_00280_b200.grid import GridMedium, GridSDF, config5_fields


def grid_scene(sdf, sigma, l_xy, l_z, n_maj, lib):
    g = _lib.MfGridField()
    g.d_sdf = sdf.ctypes.data
    g.d_sigma = sigma.ctypes.data
    maj = np.zeros(n_maj ** 3, np.float32)
    g.d_majorant = maj.ctypes.data
    g.n_sdf, g.n_sigma, g.n_maj = sdf.shape[0], sigma.shape[0], n_maj
    g.bmin[:] = (-1.6,) * 3
    g.bmax[:] = (1.6,) * 3
    g.l_xy, g.l_z = l_xy, l_z
    assert lib.mfh_grid_majorant(ctypes.byref(g), maj.ctypes.data_as(ctypes.c_void_p)) == 0
    cs = _lib.MfScene()
    cs.n_prims = cs.n_media = 1
    cs.prims[0].shape = _lib.SHAPE_GRID
    m = cs.media[0]
    m.kind, m.fresnel, m.ax, m.ay, m.az, m.sigma, m.mix_ratio = 2, 1, 1.0, 1.0, 1.0, 1.0, 0.5
    cs.camera.width = cs.camera.height = 1
    cs.camera.look_at[2] = -1.0
    cs.has_grid = 1
    cs.grid = g
    cs._keep = (sdf, sigma, maj)   # the C struct holds raw pointers into these
    return cs, maj


def run_walk(lib, cs, o, d, n, ratio=False, seed=3):
    O = np.ascontiguousarray(np.tile(o, (n, 1)).T, np.float32)
    D = np.ascontiguousarray(np.tile(d, (n, 1)).T, np.float32)
    st = np.zeros(n, np.int32)
    pos = np.zeros((3, n), np.float32)
    w = np.zeros(n, np.float32)
    v = ctypes.c_int64()
    assert lib.mfh_walk(ctypes.byref(cs), O.ctypes.data_as(ctypes.c_void_p),
                        D.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(n), ctypes.c_uint64(seed),
                        int(ratio), st.ctypes.data_as(ctypes.c_void_p),
                        pos.ctypes.data_as(ctypes.c_void_p), w.ctypes.data_as(ctypes.c_void_p),
                        ctypes.c_float(1.0), ctypes.byref(v), ctypes.c_float(0.0)) == 0
    return st, pos, w, v.value


class M:
    kind = "generalized"
    sigma = 0.05

    class a3:
        ax = ay = az = math.sqrt(2.0)


def plane(n=64):
    x = np.linspace(-1.6, 1.6, n)
    return np.ascontiguousarray(np.broadcast_to(x[None, None, :], (n, n, n)), np.float32)


def test_grid_plane_escape_and_ratio_match_closed_form(host_math):
    cs, _ = grid_scene(plane(), np.full((8, 8, 8), 0.05, np.float32), 0.05, 0.05, 32, host_math)
    n = 200000
    th = math.radians(40.0)
    d = np.array([math.sin(th), 0.0, math.cos(th)])
    st, _, _, viol = run_walk(host_math, cs, np.array([0.0, 0.0, 0.0]), d, n)
    closed = float(om.planar_transmittance(0.0, 0.15, d[2], d, M))   # escape at 3 sigma
    se = math.sqrt(closed * (1 - closed) / n)
    assert abs(np.mean(st == 0) - closed) <= 4 * se and viol == 0
    _, _, w, viol = run_walk(host_math, cs, np.array([0.0, 0.0, -0.1]), d, n, ratio=True)
    closed = float(om.planar_transmittance(-0.1, 0.15, d[2], d, M))
    assert abs(w.mean() - closed) <= 4 * w.std() / math.sqrt(n) and viol == 0


def test_grid_plane_collision_depth(host_math):
    # downward rays from above the shell: all collide inside [-6s, 3s]
    cs, _ = grid_scene(plane(), np.full((8, 8, 8), 0.05, np.float32), 0.05, 0.05, 32, host_math)
    th = math.radians(135.0)
    d = np.array([math.sin(th), 0.0, math.cos(th)])
    st, pos, _, viol = run_walk(host_math, cs, np.array([0.0, 0.0, 0.5]), d, 20000)
    assert np.all(st == 2) and viol == 0
    assert pos[2].max() <= 0.15 + 1e-5 and pos[2].min() >= -0.3 - 1e-5


def test_config5_majorant_bounds_extinction(host_math):
    sdf, sigma = config5_fields(n_sdf=64, n_sigma=32)
    cs, maj = grid_scene(sdf.values, sigma, 0.03, 0.08, 16, host_math)
    rs = np.random.default_rng(5)
    n = 20000
    o = np.array([0.0, -3.0, 0.3])
    for k in range(8):
        tgt = rs.uniform(-0.8, 0.8, 3)
        d = (tgt - o) / np.linalg.norm(tgt - o)
        st, _, _, viol = run_walk(host_math, cs, o, d, n // 8, seed=11 + k)
        assert viol == 0
        _, _, w, viol = run_walk(host_math, cs, o, d, n // 8, ratio=True, seed=21 + k)
        assert viol == 0 and np.all((w >= 0) & (w <= 1))


def test_majorant_empty_space_distances(host_math):
    """Cells without medium hold -D, D the Chebyshev distance (cells) to the
    nearest cell with medium, capped at 16 (grid_walk's empty-space jumps)."""
    sdf, sigma = config5_fields(n_sdf=64, n_sigma=32)
    n = 16
    _, maj = grid_scene(sdf.values, sigma, 0.03, 0.08, n, host_math)
    m = maj.reshape(n, n, n)
    full = np.argwhere(m > 0)
    assert len(full) and np.any(m < 0)
    for c in np.argwhere(m <= 0):
        d = int(np.min(np.max(np.abs(full - c), axis=1)))
        assert m[tuple(c)] == -min(d, 16), (c, m[tuple(c)], d)


def _mid_transmittance_rays(sdf, sigma, bounds, count, seed):
    """Rays from the config-5 camera position whose transmittance through
    the field is neither ~0 nor ~1 (coarse oracle quadrature to choose them,
    fine quadrature for the value)."""
    from oracle import gridfield as og

    rs = np.random.default_rng(seed)
    o = np.array([0.0, -4.0, 1.2])
    out = []
    for _ in range(400):
        tgt = rs.uniform(-0.9, 0.9, 3)
        d = (tgt - o) / np.linalg.norm(tgt - o)
        d = d.astype(np.float32).astype(np.float64)
        d /= np.linalg.norm(d)
        coarse = og.transmittance(sdf, sigma, bounds, 0.03, 0.08, o, d, step=2e-3)
        if 0.08 < coarse < 0.92:
            out.append((o, d, og.transmittance(sdf, sigma, bounds, 0.03, 0.08, o, d, step=4e-5)))
            if len(out) == count:
                break
    assert len(out) == count
    return out


def test_config5_transmittance_matches_oracle_quadrature(host_math):
    """The grid walker on config 5's own fields (union-of-spheres SDF, value
    noise sigma, l_xy 0.03 / l_z 0.08) against oracle/gridfield.py: ratio
    tracking through the majorant grid must reproduce exp(-int sigma_t ds)
    computed by plain float64 quadrature of the reference's coefficient
    functions on the same trilinear fields."""
    sdf, sigma = config5_fields(n_sdf=64, n_sigma=32)
    bounds = ((-1.6,) * 3, (1.6,) * 3)
    cs, _ = grid_scene(sdf.values, sigma, 0.03, 0.08, 32, host_math)
    n = 40000
    for k, (o, d, tr) in enumerate(_mid_transmittance_rays(sdf.values, sigma, bounds, 5, 9)):
        _, _, w, viol = run_walk(host_math, cs, o, d, n, ratio=True, seed=31 + k)
        w = w.astype(np.float64)
        se = w.std() / math.sqrt(n)
        assert viol == 0
        assert abs(w.mean() - tr) <= 4 * se + 2e-3, (k, w.mean(), tr, se)
        # delta tracking (collision walks, region down to -6 sigma): the escape
        # probability is the transmittance of that wider region
        from oracle import gridfield as og
        tr6 = og.transmittance(sdf.values, sigma, bounds, 0.03, 0.08, o, d, step=4e-5, lo_mult=-6.0)
        st, _, _, viol = run_walk(host_math, cs, o, d, n, seed=51 + k)
        p_esc = float(np.mean(st == 0))
        se6 = math.sqrt(max(tr6 * (1 - tr6), 1e-6) / n)
        assert viol == 0
        assert abs(p_esc - tr6) <= 4 * se6 + 2e-3, (k, p_esc, tr6, se6)
