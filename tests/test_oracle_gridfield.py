"""oracle/gridfield.py against the oracle's own planar functions (which are
pinned to the reference's golden values, tests/test_oracle_golden.py): on a
grid that holds the plane f = z with constant sigma the grid-field
quadrature must reproduce extinction_local and planar_transmittance
(medium.py:91-124); the trilinear interpolant reproduces its vertices and
its gradient matches finite differences."""

import math

import numpy as np

from oracle import gridfield as og
from oracle import microfacet as om

BOUNDS = ((-1.6,) * 3, (1.6,) * 3)


def plane_grid(n=33):
    z = np.linspace(-1.6, 1.6, n)
    return np.ascontiguousarray(np.broadcast_to(z[None, None, :], (n, n, n)), np.float64)


class M:
    kind = "generalized"
    sigma = 0.05
    mix_ratio = 0.5
    fresnel_one = True
    albedo = None

    class a3:
        ax = ay = math.sqrt(2.0) * 0.05 / 0.03
        az = math.sqrt(2.0) * 0.05 / 0.08


def test_trilinear_vertices_and_gradient():
    rs = np.random.default_rng(1)
    v = rs.normal(size=(9, 9, 9))
    x = np.linspace(-1.6, 1.6, 9)
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    pts = np.stack([X, Y, Z], axis=-1).reshape(-1, 3)
    assert np.allclose(og.trilinear(v, BOUNDS, pts), v.ravel(), atol=1e-12)
    p = rs.uniform(-1.5, 1.5, (200, 3))
    f, g = og.trilinear(v, BOUNDS, p, grad=True)
    h = 1e-6
    for a in range(3):
        e = np.zeros(3)
        e[a] = h
        fd = (og.trilinear(v, BOUNDS, p + e) - og.trilinear(v, BOUNDS, p - e)) / (2 * h)
        # central differences straddle a cell face for a few points: skip those
        cell = (p + 1.6) / 0.4
        ok = np.floor(cell[:, a] + h / 0.4) == np.floor(cell[:, a] - h / 0.4)
        assert np.allclose(fd[ok], g[ok, a], rtol=1e-6, atol=1e-6)


def test_plane_grid_matches_planar_closed_forms():
    sdf = plane_grid()
    sig = np.full((5, 5, 5), M.sigma)
    th = math.radians(40.0)
    d = np.array([math.sin(th), 0.0, -math.cos(th)])
    # pointwise extinction = rho(f) sigma(w) of the homogeneous medium
    z = np.linspace(-0.14, 0.14, 57)
    p = np.stack([np.full_like(z, 0.1), np.full_like(z, -0.2), z], axis=-1)
    st = og.extinction(sdf, sig, BOUNDS, 0.03, 0.08, p, d)
    ref = om.extinction_local(np.broadcast_to(d, p.shape), z, M)
    assert np.allclose(st, ref, rtol=1e-10, atol=0.0)
    # region rule: zero outside [-3 sigma, 3 sigma] (and [-6, 3] for flights)
    assert og.extinction(sdf, sig, BOUNDS, 0.03, 0.08, np.array([[0, 0, -0.2]]), d)[0] == 0.0
    assert og.extinction(sdf, sig, BOUNDS, 0.03, 0.08, np.array([[0, 0, -0.2]]), d, -6.0)[0] > 0.0
    # transmittance through the whole shell = the closed form over |f| <= 3 sigma
    tr = og.transmittance(sdf, sig, BOUNDS, 0.03, 0.08, np.array([0.0, 0.0, 1.0]), d, step=1e-5)
    closed = float(om.planar_transmittance(3 * M.sigma, -3 * M.sigma, d[2], d, M))
    assert abs(tr - closed) <= 2e-3 * closed + 1e-6, (tr, closed)


def test_plane_grid_single_scatter_matches_planar_quadrature():
    """single_scatter_radiance on the plane grid = the collision-depth
    quadrature of Tr_in sigma_t / |cos| phase Tr_out over [-6 sigma, 3 sigma]
    (the make_golden.py depth-1 anchor) with the planar closed forms."""

    class Ma(M):
        albedo = (0.85, 0.85, 0.85)
        fresnel_one = False

    sdf = plane_grid(65)
    sig = np.full((5, 5, 5), M.sigma)
    thv, thl = math.radians(35.0), math.radians(50.0)
    d = np.array([math.sin(thv), 0.0, -math.cos(thv)])
    tl = np.array([-math.sin(thl), 0.0, math.cos(thl)])
    got = og.single_scatter_radiance(sdf, sig, BOUNDS, 0.03, 0.08, 0.85,
                                     np.array([-0.3, 0.0, 1.0]), d, tl, 2.0, 0.0)
    s = M.sigma
    h = np.linspace(-6 * s, 3 * s, 200001)
    sig_t = om.extinction_local(np.broadcast_to(d, h.shape + (3,)), h, Ma)
    tr_in = om.planar_transmittance(3 * s, h, d[2], d, Ma)
    tr_out = om.planar_transmittance(np.maximum(h, -3 * s), 3 * s, tl[2], tl, Ma)
    ph = float(om.phase_eval_local(d[None], tl[None], Ma)[0, 0])
    ref = 2.0 * float(np.trapezoid(tr_in * sig_t / abs(d[2]) * ph * tr_out, h))
    assert abs(got - ref) <= 5e-3 * ref, (got, ref)
