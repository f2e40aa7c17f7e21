"""Heterogeneous GP field (BASELINE config 5, no reference oracle: parity is
unpinned by construction).  Self-consistency instead: a
constant-sigma grid of a plane / sphere SDF must reproduce the analytic
planar / sphere paths, and the majorant grid must never be exceeded."""

import math

import numpy as np
import pytest

import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
from paper_2603_00280_b200.grid import GridMedium, GridSDF, union_sdf

pytestmark = pytest.mark.gpu

BOUNDS = ((-1.6, -1.6, -1.6), (1.6, 1.6, 1.6))


def plane_grid(n=64):
    x = np.linspace(-1.6, 1.6, n)
    Z = np.broadcast_to(x[None, None, :], (n, n, n))
    return GridSDF(np.ascontiguousarray(Z, dtype=np.float32), BOUNDS)


def test_grid_plane_matches_planar_quadrature(cuda):
    """Constant sigma = 0.05, l = 0.05 grid of f = z reproduces config 2's
    depth-1 collision-depth quadrature (0.113098, anchors.json)."""
    sdf = plane_grid()
    med = GridMedium(sigma=np.full((16, 16, 16), 0.05, np.float32), l_xy=0.05, l_z=0.05,
                     albedo=0.8)
    base = configs.config2_scene(64, 64)
    cam = mf.Camera(position=base.camera.position, look_at=(0, 0, 0), fov_deg=40, width=64,
                    height=64, ortho=True, film_height=0.2)
    sc = mf.ShellScene(primitives=(mf.ShellPrimitive(sdf, med),), camera=cam,
                       environment=base.environment, sun=base.sun)
    img, st = mf.render_device(sc, 1024, 3, max_bounces=1, stats=True)
    v = img[..., 0].cpu().numpy().astype(np.float64)
    se = v.std() / math.sqrt(v.size)
    assert st["majorant_violations"] == 0 and st["nonfinite"] == 0
    assert abs(v.mean() - 0.113098) <= 3.5 * se + 2e-5, (v.mean(), se)


def test_grid_sphere_matches_analytic_sphere(cuda):
    """A 128^3 grid of the unit-sphere SDF with constant sigma = 0.1 renders
    config 3 (reduced) like the analytic sphere walker."""
    n = 128
    sdf = GridSDF(union_sdf(n, BOUNDS, [((0.0, 0.0, 0.0), 1.0)], None), BOUNDS)
    med = GridMedium(sigma=np.full((16, 16, 16), 0.1, np.float32), l_xy=0.05, l_z=0.05,
                     albedo=0.9)
    ref = configs.config3_scene(48, 48)
    sc = mf.ShellScene(primitives=(mf.ShellPrimitive(sdf, med),), camera=ref.camera,
                       environment=ref.environment, point=ref.point)
    a, st = mf.render_device(sc, 256, 5, max_bounces=32, stats=True)
    b, _ = mf.render_device(ref, 256, 6, max_bounces=32)
    a = a.cpu().numpy().astype(np.float64)
    b = b.cpu().numpy().astype(np.float64)
    assert st["majorant_violations"] == 0 and st["nonfinite"] == 0
    # image means (trilinear SDF error ~h^2/8R ~ 1e-4 << sigma)
    da = a[..., 0].std() / math.sqrt(a[..., 0].size)
    assert abs(a.mean() - b.mean()) <= 4 * math.sqrt(2) * da + 2e-3 * b.mean()


def test_config5_render_small(cuda):
    torch = cuda
    sc = configs.config5_scene(64, 64, n_sdf=96, n_sigma=48)
    img, st = mf.render_device(sc, 16, 4, max_bounces=64, stats=True)
    assert st["majorant_violations"] == 0, st
    assert st["nonfinite"] == 0 and st["capped"] == 0
    assert torch.isfinite(img).all() and (img >= 0).all()
    img2, _ = mf.render_device(sc, 16, 4, max_bounces=64, tile=8)
    assert torch.equal(img, img2)
    # the geometry is visible: some pixels differ from the environment
    assert (img[..., 0] != 0.2).float().mean() > 0.2


def test_grid_transmittance_matches_plane(cuda):
    """Ratio tracking through a constant grid plane equals the closed form."""
    from oracle import microfacet as om

    sdf = plane_grid()
    med = GridMedium(sigma=np.full((8, 8, 8), 0.2, np.float32), l_xy=0.2 * math.sqrt(2),
                     l_z=0.2 * math.sqrt(2), fresnel_one=True)
    cam = mf.Camera(position=(0, 0, 10), look_at=(0, 0, 0), fov_deg=40, width=4, height=4)
    sc = mf.ShellScene(primitives=(mf.ShellPrimitive(sdf, med),), camera=cam)
    th = np.deg2rad(45.0)
    d = np.array([np.sin(th), 0.0, np.cos(th)])
    mean, se = mf.transmittance_estimate((np.array([0.0, 0.0, -0.1]), d), sc, 1_000_000,
                                         mf.RandomStream(3, 1))

    class M:
        kind = "generalized"
        sigma = 0.2

        class a3:
            ax = ay = az = 1.0

    closed = float(om.planar_transmittance(-0.1, 0.6, d[2], d, M))
    assert abs(mean - closed) <= 4 * se, (mean, closed, se)
