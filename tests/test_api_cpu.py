"""Host-side logic of the Python mirror (CPU only): parameter validation
with the reference's exception classes, scene flattening, the image
formats, and the no-CPU-fallback rule."""

import math

import numpy as np
import pytest

import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import _lib, configs
from paper_2603_00280_b200.render import owned_pixels
from paper_2603_00280_b200.scene import to_c_scene

ISO1 = mf.RoughnessTriple(1.0, 1.0, 1.0)


def test_parameter_validation_mirrors_reference():
    # medium.py:53-59, ndf.py:60-66
    with pytest.raises(mf.ParameterDomainError):
        mf.MacrofacetMedium(kind=mf.NdfKind.GENERALIZED, a3=ISO1, sigma=0.0)
    with pytest.raises(ValueError):  # ParameterDomainError is a ValueError
        mf.MacrofacetMedium(kind=mf.NdfKind.GENERALIZED, a3=ISO1, sigma=1.0, mix_ratio=1.5)
    with pytest.raises(mf.ParameterDomainError):
        mf.MacrofacetMedium(kind=mf.NdfKind.GENERALIZED, a3=mf.RoughnessTriple(1, 1, 0), sigma=1)
    with pytest.raises(mf.ParameterDomainError):
        mf.RoughnessTriple(-1.0, 1.0)
    with pytest.raises(mf.ParameterDomainError):
        mf.KernelParams(1.0, 0.0, 1.0, 1.0)
    m = mf.MacrofacetMedium(kind=mf.NdfKind.BECKMANN, a3=mf.RoughnessTriple(1, 1, 0.5), sigma=1)
    assert m.a3.az == 0.0  # height-field kinds drop az (medium.py:60-61)
    a = mf.roughness_from_kernel(mf.KernelParams(0.05, 0.1, 0.1, 0.1))
    assert abs(a.ax - math.sqrt(2) * 0.5) < 1e-15


def test_shell_overlap_rejected():
    # scene.py:118-129 / test_scene_render.py:68-87
    med = mf.MacrofacetMedium(kind=mf.NdfKind.GENERALIZED, a3=ISO1, sigma=1.0)
    cam = mf.Camera(position=(0, 0, 10), look_at=(0, 0, 0), fov_deg=40, width=4, height=4)
    with pytest.raises(mf.ConfigError):
        mf.ShellScene(primitives=(mf.ShellPrimitive(mf.Plane(0.0), med),
                                  mf.ShellPrimitive(mf.Sphere((0, 0, 5.0), 1.0), med)), camera=cam)
    mf.ShellScene(primitives=(mf.ShellPrimitive(mf.Plane(0.0), med),
                              mf.ShellPrimitive(mf.Sphere((0, 0, 8.0), 1.0), med)), camera=cam)


def test_scene_flattening():
    s = configs.config3_scene(64, 48)
    c = to_c_scene(s)
    assert c.n_prims == 1 and c.prims[0].shape == _lib.SHAPE_SPHERE
    assert c.prims[0].radius == 1.0 and c.camera.width == 64 and c.camera.height == 48
    assert c.has_point == 1 and tuple(c.point_intensity) == (10.0, 10.0, 10.0)
    assert c.media[0].fresnel == _lib.FRESNEL_ALBEDO and tuple(c.media[0].albedo) == (0.9,) * 3
    s2 = configs.config2_scene()
    c2 = to_c_scene(s2)
    assert c2.camera.ortho == 1 and c2.has_sun == 1
    assert abs(c2.sun_dir[2] + math.sin(math.radians(30))) < 1e-15
    # a lat-long map is uploaded to the device: no device, no fallback
    env = mf.Environment(radiance=(1, 1, 1), latlong=np.ones((2, 4, 3)))
    with pytest.raises(mf.MacrofacetError):
        to_c_scene(mf.ShellScene(primitives=(), camera=s.camera, environment=env))
    # boxes (sdf.py:55-84)
    med = mf.MacrofacetMedium(kind=mf.NdfKind.BECKMANN, a3=mf.RoughnessTriple(0.4, 0.9), sigma=0.3)
    cb = to_c_scene(mf.ShellScene(primitives=(mf.ShellPrimitive(
        mf.Box((0, 0, 0), (1.5, 1.5, 0.8)), med),), camera=s.camera))
    assert cb.prims[0].shape == _lib.SHAPE_BOX and tuple(cb.prims[0].half_extents) == (1.5, 1.5, 0.8)
    with pytest.raises(mf.ParameterDomainError):
        mf.Box((0, 0, 0), (1.0, 0.0, 1.0))


def _standin_scene(R):
    """config-2-like scene built from reference-shaped classes (module R)."""
    med = R.MacrofacetMedium(kind=R.NdfKind.GENERALIZED, a3=R.RoughnessTriple(1.2, 0.9, 0.7),
                             sigma=0.05, mix_ratio=0.4)
    sph = R.MacrofacetMedium(kind=R.NdfKind.BECKMANN, a3=R.RoughnessTriple(0.5, 0.5, 0.0),
                             sigma=0.1, fresnel_one=True)
    box = R.MacrofacetMedium(kind=R.NdfKind.GGX, a3=R.RoughnessTriple(0.3, 0.3, 0.0), sigma=0.05)
    prims = (R.ShellPrimitive(R.Plane(0.0), med), R.ShellPrimitive(R.Sphere((0, 0, 3), 1.0), sph),
             R.ShellPrimitive(R.Box((3, 0, 3), (0.5, 0.5, 0.5)), box))
    cam = R.Camera(position=(0, -6, 2), look_at=(0, 0, 1), fov_deg=40, width=32, height=24)
    return R.ShellScene(primitives=prims, camera=cam,
                        environment=R.Environment(radiance=(0.1, 0.2, 0.3)),
                        sun=R.DirectionalLight(direction=(0.3, -0.2, -0.93), radiance=(1, 1, 1)))


def _same_c_scene(a, b):
    return bytes(memoryview(a)) == bytes(memoryview(b))


def test_reference_shaped_scene_flattens_like_ours():
    """Drop-in rule: a scene built from reference-shaped
    classes flattens to exactly the C scene of the same scene built from
    this package's classes."""
    import refstandin

    a = to_c_scene(_standin_scene(refstandin))
    b = to_c_scene(_standin_scene(mf))
    assert _same_c_scene(a, b)


def test_real_reference_scene_flattens_like_ours():
    """The same with the reference package's own classes, where it is
    importable (the build container; skipped on the GPU box)."""
    import os
    import sys

    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference package not present")
    sys.path.insert(0, src)
    try:
        import macrofacet as R
    finally:
        sys.path.remove(src)
    a = to_c_scene(_standin_scene(R))
    b = to_c_scene(_standin_scene(mf))
    assert _same_c_scene(a, b)


def test_foreign_shape_error_names_the_class():
    """An SDF class the device cannot trace raises UnsupportedGeometryError
    naming it (the old message blamed Plane)."""
    import refstandin

    class Torus:
        pass

    med = refstandin.MacrofacetMedium(kind=refstandin.NdfKind.GENERALIZED,
                                      a3=refstandin.RoughnessTriple(1, 1, 1), sigma=0.1)
    sc = refstandin.ShellScene(primitives=(refstandin.ShellPrimitive(Torus(), med),),
                               camera=refstandin.Camera((0, 0, 5), (0, 0, 0), 40, 4, 4))
    with pytest.raises(mf.UnsupportedGeometryError, match="Torus"):
        to_c_scene(sc)


def test_batch_rng_matches_reference_streams():
    """BatchRng / derive_bases reproduce the reference's SplitMix64 streams
    bit for bit (rng.py:24-58, transport.py:52-67)."""
    base = mf.derive_bases(5, 7, np.arange(16))
    r = mf.BatchRng(base, np.arange(16, dtype=np.uint64))
    u = r.draw()
    assert u.shape == (16,) and np.all((u >= 0) & (u < 1))
    assert np.array_equal(r.counter, np.arange(16, dtype=np.uint64) + 1)
    s = mf.RandomStream(5, 7)
    kid = s.derive(3)
    assert np.uint64(mf.stream_base(5, kid.stream)) == base[3]


def test_no_cpu_fallback(monkeypatch):
    import torch

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(mf.MacrofacetError):
        mf.render(configs.config2_scene(8, 8), 1, 0)
    with pytest.raises(mf.MacrofacetError):
        mf.transmittance_estimate((np.zeros(3), np.array([0, 0, 1.0])), configs.config2_scene(),
                                  10, mf.RandomStream(1))


def test_render_argument_validation():
    with pytest.raises(mf.ParameterDomainError):
        mf.render_device(configs.config2_scene(8, 8), 0, 0)
    with pytest.raises(mf.ParameterDomainError):
        mf.render_device(configs.config2_scene(8, 8), 1, 0, max_bounces=0)


def test_pfm_byte_contract(tmp_path):
    # image.py:45-52 / test_scene_render.py:177-195
    img = mf.RadianceImage(pixels=np.ones((1, 1, 3)))
    path = tmp_path / "one.pfm"
    mf.write_pfm(img, path)
    blob = path.read_bytes()
    assert blob == b"PF\n1 1\n-1.0\n" + np.ones(3, dtype="<f4").tobytes()
    rs = np.random.default_rng(8)
    img = mf.RadianceImage(pixels=rs.uniform(0.0, 5.0, (7, 5, 3)))
    mf.write_pfm(img, tmp_path / "rt.pfm")
    back = mf.read_pfm(tmp_path / "rt.pfm")
    assert np.array_equal(back.pixels, img.pixels.astype(np.float32).astype(np.float64))
    mf.write_ppm(mf.RadianceImage(pixels=np.zeros((2, 3, 3))), tmp_path / "z.ppm")
    assert (tmp_path / "z.ppm").read_bytes() == b"P6\n3 2\n255\n" + bytes(18)
    with pytest.raises(mf.MacrofacetError):
        mf.RadianceImage(pixels=np.full((1, 1, 3), np.nan)).validate()


@pytest.mark.parametrize("w,h,tile,n", [(256, 256, 32, 1), (256, 256, 32, 8), (100, 37, 16, 3),
                                        (5, 7, 32, 4), (64, 64, 8, 5)])
def test_tile_ownership_partitions_image(w, h, tile, n):
    """Interleaved tile sharding: every pixel has exactly
    one owner, so a sum-reduce of disjoint buffers is exact."""
    seen = np.zeros(w * h, dtype=np.int64)
    for r in range(n):
        px = owned_pixels(w, h, tile, r, n)
        seen[px] += 1
    assert np.all(seen == 1)
