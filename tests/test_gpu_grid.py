"""Heterogeneous GP field (BASELINE config 5, no reference oracle: parity is
unpinned by construction).  Self-consistency instead: a
constant-sigma grid of a plane / sphere SDF must reproduce the analytic
planar / sphere paths, and the majorant grid must never be exceeded."""

import dataclasses
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


def _depth1_quadrature_oracle(m, travel, to_light):
    """Oracle single-scatter value of a flat shell lit by the sun (the
    make_golden.py depth-1 quadrature, with the oracle's functions):
    int Tr_in sigma_t / |cos| phase Tr_out dh over [-6s, 3s]."""
    from oracle import microfacet as om

    s = m.sigma
    d = np.asarray(travel, dtype=np.float64)
    tl = np.asarray(to_light, dtype=np.float64)
    h = np.linspace(-6 * s, 3 * s, 200001)
    sig_t = om.extinction_local(np.broadcast_to(d, h.shape + (3,)), h, m)
    tr_in = om.planar_transmittance(3 * s, h, d[2], d, m)
    tr_out = om.planar_transmittance(np.maximum(h, -3 * s), 3 * s, tl[2], tl, m)
    ph = float(om.phase_eval_local(d[None], tl[None], m)[0, 0])
    return float(np.trapezoid(tr_in * sig_t / abs(d[2]) * ph * tr_out, h))


def test_grid_plane_config5_anisotropy(cuda):
    """Self-consistency at config 5's own anisotropy (l_xy = 0.03, l_z =
    0.08: alpha_xy = 4.71, alpha_z = 1.77 at sigma = 0.1): a
    grid plane with constant sigma reproduces (a) the oracle's depth-1
    quadrature of the analytic GENERALIZED plane and (b) the analytic
    planar path (pool kernel) at depth 64, through the grid walker's
    independent code (majorant DDA, trilinear fields, delta / ratio
    tracking)."""
    import parity

    sigma, lxy, lz = 0.1, 0.03, 0.08
    sdf = plane_grid()
    med = GridMedium(sigma=np.full((16, 16, 16), sigma, np.float32), l_xy=lxy, l_z=lz,
                     albedo=0.85)
    base = configs.config2_scene(64, 64)
    cam = mf.Camera(position=base.camera.position, look_at=(0, 0, 0), fov_deg=40, width=64,
                    height=64, ortho=True, film_height=0.2)
    sc = mf.ShellScene(primitives=(mf.ShellPrimitive(sdf, med),), camera=cam,
                       environment=base.environment, sun=base.sun)
    a3 = mf.roughness_from_kernel(mf.KernelParams(sigma, lxy, lxy, lz))
    ana = mf.MacrofacetMedium(kind=mf.NdfKind.GENERALIZED, a3=a3, sigma=sigma, albedo=0.85)
    # (a) depth 1 vs the oracle quadrature
    img, st = mf.render_device(sc, 1024, 3, max_bounces=1, stats=True)
    v = img[..., 0].cpu().numpy().astype(np.float64)
    se = v.std() / math.sqrt(v.size)
    q = _depth1_quadrature_oracle(parity.f32_medium(ana), configs.CAM_TRAVEL_C2,
                                  configs.TO_LIGHT_C2)
    assert st["majorant_violations"] == 0 and st["nonfinite"] == 0 and st["capped"] == 0
    assert abs(v.mean() - q) <= 3.5 * se + 2e-5, (v.mean(), se, q)
    # (b) depth 64 vs the analytic plane
    img, st = mf.render_device(sc, 1024, 4, max_bounces=64, stats=True)
    v = img[..., 0].cpu().numpy().astype(np.float64)
    se = v.std() / math.sqrt(v.size)
    sc_a = mf.ShellScene(primitives=(mf.ShellPrimitive(mf.Plane(0.0), ana),), camera=cam,
                         environment=base.environment, sun=base.sun)
    ref, _ = mf.render_device(sc_a, 1024, 5, max_bounces=64)
    r = ref[..., 0].cpu().numpy().astype(np.float64)
    se_r = r.std() / math.sqrt(r.size)
    assert st["majorant_violations"] == 0 and st["capped"] == 0
    assert abs(v.mean() - r.mean()) <= 3.5 * math.hypot(se, se_r), (v.mean(), r.mean(), se, se_r)


def test_config5_full_grids(cuda):
    """BASELINE config 5's own fields at full size (256^3 SDF, 128^3 value
    noise sigma, l_xy 0.03 / l_z 0.08) at a reduced film: zero majorant
    violations (the majorant grid is a sampled bound, checked at every
    tentative collision), no capped walks, finite non-negative image,
    deterministic for any tile size."""
    torch = cuda
    sc = configs.config5_scene(192, 192)
    assert sc.primitives[0].sdf.values.shape == (256, 256, 256)
    assert sc.primitives[0].medium.sigma.shape == (128, 128, 128)
    img, st = mf.render_device(sc, 64, 4, max_bounces=64, stats=True)
    assert st["majorant_violations"] == 0, st
    assert st["capped"] == 0 and st["nonfinite"] == 0, st
    assert st["track_steps"] > st["paths"]     # the walker really tracked
    assert torch.isfinite(img).all() and (img >= 0).all()
    img2, _ = mf.render_device(sc, 64, 4, max_bounces=64, tile=16)
    assert torch.equal(img, img2)


def test_grid_pool_matches_megakernel(cuda, monkeypatch):
    """The grid-field path pool runs every path with the megakernel's
    arithmetic and random stream: the same decisions (identical event
    counts) and the same image to float rounding (a few multiply-adds are
    contracted differently in the two inlining contexts); the pool itself
    is deterministic."""
    sc = configs.config5_scene(64, 48, n_sdf=96, n_sigma=48)
    a, sa = mf.render_device(sc, 16, 4, max_bounces=64, stats=True)
    a = a.cpu().numpy()
    a2, _ = mf.render_device(sc, 16, 4, max_bounces=64, tile=8)
    assert np.array_equal(a, a2.cpu().numpy())
    monkeypatch.setenv("MF_MEGAKERNEL", "1")
    b, sb = mf.render_device(sc, 16, 4, max_bounces=64, stats=True)
    b = b.cpu().numpy()
    np.testing.assert_allclose(a, b, rtol=1e-4, atol=1e-7)
    sa.pop("path_kernel_ms"), sb.pop("path_kernel_ms")
    assert sa == sb


def test_grid_walk_pool_matches_curved_pool(cuda, monkeypatch):
    """The grid pool with pooled walks (walks parked and resumed between W
    visits, tentative collisions batched) against the pool that runs whole
    walks inside its visits (MF_GRID_WALK_POOL=0): the same decisions
    (identical event counts), the same image to float rounding; colour
    scenes too; deterministic for any tile size."""
    for colour, conductor in ((False, False), (True, False), (True, True)):
        sc = configs.config5_scene(64, 48, n_sdf=96, n_sigma=48)
        if colour:
            sc = dataclasses.replace(sc, environment=mf.Environment(radiance=(0.2, 0.1, 0.05)))
        if conductor:
            # conductor Fresnel: the runtime-dispatch build (kSpec 0) of both pools
            pr = sc.primitives[0]
            med = dataclasses.replace(pr.medium, albedo=None)
            sc = dataclasses.replace(sc, primitives=(dataclasses.replace(pr, medium=med),))
        a, sa = mf.render_device(sc, 16, 4, max_bounces=64, stats=True)
        a = a.cpu().numpy()
        a2, _ = mf.render_device(sc, 16, 4, max_bounces=64, tile=8)
        assert np.array_equal(a, a2.cpu().numpy())
        monkeypatch.setenv("MF_GRID_WALK_POOL", "0")
        b, sb = mf.render_device(sc, 16, 4, max_bounces=64, stats=True)
        monkeypatch.delenv("MF_GRID_WALK_POOL")
        b = b.cpu().numpy()
        sa.pop("path_kernel_ms"), sb.pop("path_kernel_ms")
        assert sa == sb            # the same decisions: identical event counts
        # the same arithmetic up to how the compiler contracts multiply-adds
        # in the two kernels (one pixel of the conductor build: 1.9e-4)
        np.testing.assert_allclose(a, b, rtol=5e-4, atol=1e-7)


@pytest.mark.parametrize("width,height,spp,depth", [(3, 2, 1, 64), (5, 4, 3, 1), (16, 8, 4, 2),
                                                     (33, 17, 2, 9)])
def test_grid_walk_pool_small_and_shallow(cuda, monkeypatch, width, height, spp, depth):
    """Partial visits (fewer paths than a warp), paths that end at their
    first collisions (depth cap with a shadow walk still queued) and the
    first roulette bounce: same event counts and image as the curved pool."""
    sc = configs.config5_scene(width, height, n_sdf=64, n_sigma=32)
    a, sa = mf.render_device(sc, spp, 7, max_bounces=depth, stats=True)
    monkeypatch.setenv("MF_GRID_WALK_POOL", "0")
    b, sb = mf.render_device(sc, spp, 7, max_bounces=depth, stats=True)
    monkeypatch.delenv("MF_GRID_WALK_POOL")
    np.testing.assert_allclose(a.cpu().numpy(), b.cpu().numpy(), rtol=1e-4, atol=1e-7)
    sa.pop("path_kernel_ms"), sb.pop("path_kernel_ms")
    assert sa == sb
    assert sa["paths"] == width * height * spp


def test_config5_transmittance_matches_oracle_quadrature(cuda):
    """Config 5's own heterogeneous fields (128^3 union-of-spheres SDF, 64^3
    value-noise sigma, l_xy 0.03 / l_z 0.08) on the device against
    oracle/gridfield.py: the ratio-tracked transmittance (mf_transmittance:
    trilinear fetches, gradient frames, region rules, the majorant grid and
    its DDA) must equal exp(-int sigma_t ds) from plain float64 quadrature
    of the reference's coefficient functions on the same fields."""
    from paper_2603_00280_b200.grid import config5_fields
    from test_grid_host import _mid_transmittance_rays

    sdf, sigma = config5_fields(n_sdf=128, n_sigma=64)
    bounds = ((-1.6,) * 3, (1.6,) * 3)
    med = GridMedium(sigma=sigma, l_xy=0.03, l_z=0.08, albedo=0.85)
    cam = mf.Camera(position=(0.0, -4.0, 1.2), look_at=(0.0, 0.0, 0.0), fov_deg=40.0, width=4,
                    height=4)
    sc = mf.ShellScene(primitives=(mf.ShellPrimitive(sdf, med),), camera=cam)
    n = 400_000
    worst = 0.0
    for k, (o, d, tr) in enumerate(_mid_transmittance_rays(sdf.values, sigma, bounds, 8, 13)):
        mean, se = mf.transmittance_estimate((o, d), sc, n, mf.RandomStream(21 + k, 1))
        assert abs(mean - tr) <= 4 * se + 2e-3, (k, mean, tr, se)
        worst = max(worst, abs(mean - tr) / max(se, 1e-12))
    print(f"config-5 field transmittance: worst |device - quadrature| = {worst:.2f} SE over 8 rays")


def test_config5_single_scatter_matches_oracle_quadrature(cuda):
    """Depth-1 radiance on config 5's own heterogeneous fields: trace_paths
    at max_bounces = 1 (the grid flight, the collision's local medium and
    gradient frame, NEE with a tracked shadow ray, the environment on
    escape) against oracle/gridfield.single_scatter_radiance -- nested
    float64 quadrature of T sigma_t phase Tr_sun with the reference's
    coefficient functions evaluated on the same trilinear fields."""
    from oracle import gridfield as og
    from test_grid_host import _mid_transmittance_rays

    sc = configs.config5_scene(4, 4, n_sdf=128, n_sigma=64)
    pr = sc.primitives[0]
    sdf, sigma = pr.sdf.values, pr.medium.sigma
    bounds = ((-1.6,) * 3, (1.6,) * 3)
    sun_to = -np.asarray(sc.sun.direction, dtype=np.float64)
    sun_to /= np.linalg.norm(sun_to)
    n = 1 << 20
    for k, (o, d, _) in enumerate(_mid_transmittance_rays(sdf, sigma, bounds, 3, 17)):
        quad = og.single_scatter_radiance(sdf, sigma, bounds, 0.03, 0.08, 0.85, o, d, sun_to,
                                          float(sc.sun.radiance[0]),
                                          float(sc.environment.radiance[0]))
        keys = mf.PathKeys(77 + k, np.arange(n, dtype=np.uint32), np.zeros(n, dtype=np.uint32))
        rad = mf.trace_paths(np.broadcast_to(o, (n, 3)), np.broadcast_to(d, (n, 3)), sc, 1, keys)
        mc, se = float(rad[:, 0].mean()), float(rad[:, 0].std() / math.sqrt(n))
        print(f"ray {k}: device {mc:.5f} +- {se:.5f}, quadrature {quad:.5f}")
        assert abs(mc - quad) <= 4 * se + 0.01 * quad, (k, mc, quad, se)


def test_config5_white_furnace(cuda):
    """White furnace on config 5's heterogeneous fields (acceptance 11 of the
    reference, test_scene_render.py, on a grid field): a lossless medium
    (albedo 1) in a uniform environment of radiance 1 with no lights returns
    radiance 1 along every ray whatever the geometry -- the product of the
    sampling weights phase / pdf over all bounces, on local media that change
    from collision to collision, must average to 1."""
    base = configs.config5_scene(64, 48, n_sdf=128, n_sigma=64)
    pr = base.primitives[0]
    med = dataclasses.replace(pr.medium, albedo=1.0)
    sc = dataclasses.replace(base, primitives=(dataclasses.replace(pr, medium=med),),
                             environment=mf.Environment(radiance=(1.0, 1.0, 1.0)), sun=None)
    img, st = mf.render_device(sc, 256, 11, max_bounces=512, stats=True)
    v = img[..., 0].double().cpu().numpy()
    assert st["majorant_violations"] == 0 and st["capped"] == 0
    assert st["scatters"] > 0.5 * st["paths"]    # the furnace really scattered
    se = v.std() / math.sqrt(v.size)
    print(f"grid white furnace: mean {v.mean():.6f} +- {se:.6f}, pixel max |L - 1| "
          f"{np.abs(v - 1).max():.4f}, absorbed {st['absorbed'] / st['paths']:.2e}")
    assert abs(v.mean() - 1.0) <= 4 * se + 1e-3, (v.mean(), se)
