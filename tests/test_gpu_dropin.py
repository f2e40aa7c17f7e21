"""The drop-in boundary on the B200:
reference-shaped scene objects render unchanged, trace_paths takes a
BatchRng, walk() / sample_collision() run on the device walker, Box shells
and lat-long environments are traced on the device.  Statistical checks
use the float64 oracle and the reference's own analytic forms."""

import math

import numpy as np
import pytest

import paper_2603_00280_b200 as mf
from oracle import microfacet as om
from oracle import tracer
from paper_2603_00280_b200 import configs

import parity
import refstandin as R

pytestmark = pytest.mark.gpu


def _scene(M, medium_kw=None):
    med = M.MacrofacetMedium(kind=M.NdfKind.GENERALIZED, a3=M.RoughnessTriple(1.2, 0.9, 0.7),
                             sigma=0.05, **(medium_kw or {}))
    cam = M.Camera(position=(0, -6, 2), look_at=(0, 0, 0.5), fov_deg=40, width=48, height=32)
    return M.ShellScene(primitives=(M.ShellPrimitive(M.Plane(0.0), med),
                                    M.ShellPrimitive(M.Sphere((0, 0, 1.5), 0.8), med)),
                        camera=cam, environment=M.Environment(radiance=(0.3, 0.2, 0.1)),
                        sun=M.DirectionalLight(direction=(0.3, -0.2, -0.93), radiance=(1, 1, 1)))


def test_reference_shaped_scene_renders_bitwise(cuda):
    """A scene built from the reference's classes (stand-ins with the same
    names and fields) renders bit-identically to the same scene built from
    this package's classes, through render() and render_device()."""
    a = mf.render(_scene(R), spp=16, seed=7, max_bounces=8)
    b = mf.render(_scene(mf), spp=16, seed=7, max_bounces=8)
    assert np.array_equal(a.pixels, b.pixels)
    assert a.pixels.shape == (32, 48, 3) and np.all(np.isfinite(a.pixels))
    c, _ = mf.render_device(_scene(R, {"fresnel_one": True}), 16, 7, max_bounces=8)
    d, _ = mf.render_device(_scene(mf, {"fresnel_one": True}), 16, 7, max_bounces=8)
    assert cuda.equal(c, d)


def test_trace_paths_with_batch_rng(cuda):
    """trace_paths(origins, directions, scene, max_bounces, brng) with a
    BatchRng (render.py:32): deterministic in (base, counter), counters
    advance by one per path, and the single-bounce estimate matches the
    oracle's collision-depth quadrature (test_scene_render.py:222-259)."""
    sc = configs.config2_scene(8, 8)
    n = 1 << 20
    d = np.broadcast_to(np.array(configs.CAM_TRAVEL_C2), (n, 3))
    o = np.broadcast_to(np.array([0.0, 0.0, 0.2]), (n, 3))
    base = mf.derive_bases(11, 3, np.arange(n))
    b1 = mf.BatchRng(base, np.zeros(n, dtype=np.uint64))
    r1 = mf.trace_paths(o, d, sc, 1, b1)
    assert np.all(b1.counter == 1)
    r2 = mf.trace_paths(o, d, sc, 1, mf.BatchRng(base, np.zeros(n, dtype=np.uint64)))
    assert np.array_equal(r1, r2)
    r3 = mf.trace_paths(o, d, sc, 1, b1)            # advanced counters: new streams
    assert not np.array_equal(r1, r3)
    import json
    import os

    from conftest import GOLDEN

    q = json.load(open(os.path.join(GOLDEN, "anchors.json")))["config2_depth1_quadrature"]
    v = r1[:, 0]
    assert abs(v.mean() - q) <= 4 * v.std() / math.sqrt(n) + 1e-5, (v.mean(), q)


def test_walk_ratio_matches_closed_form(cuda):
    """walk(mode="ratio") on a flat shell: the mean ratio-tracking weight is
    the closed-form transmittance (medium.py:98-124) over |f| <= 3 sigma."""
    med = mf.MacrofacetMedium(kind=mf.NdfKind.GENERALIZED, a3=mf.RoughnessTriple(1, 1, 1),
                              sigma=0.2, fresnel_one=True)
    sc = mf.ShellScene(primitives=(mf.ShellPrimitive(mf.Plane(0.0), med),),
                       camera=mf.Camera((0, 0, 5), (0, 0, 0), 40, 4, 4))
    n = 1 << 18
    th = math.radians(50.0)
    d = np.array([math.sin(th), 0.0, math.cos(th)])
    o = np.broadcast_to(np.array([0.0, 0.0, -0.1]), (n, 3))
    rng = mf.BatchRng(mf.derive_bases(3, 1, np.arange(n)), np.zeros(n, dtype=np.uint64))
    state, pos, travel, w, prim = mf.walk(sc, o, np.broadcast_to(d, (n, 3)), rng, mode="ratio")
    m = parity.f32_medium(med)
    closed = float(om.planar_transmittance(-0.1, 0.6, d[2], d, m))
    assert abs(w.mean() - closed) <= 4 * w.std() / math.sqrt(n), (w.mean(), closed)
    assert np.all(prim == -1) and np.all(state == 0)
    # escaped rays end above the shell, travel = |pos - origin|
    np.testing.assert_allclose(travel, np.linalg.norm(pos - o, axis=-1), rtol=1e-4, atol=1e-5)
    assert np.all(rng.counter == 1)


def test_walk_collision_depth_law(cuda):
    """walk(mode="collision") through a flat shell from above: the
    distribution of collision heights is 1 - Tr(3 sigma -> h) (the
    reference's KS check, test_transport.py:45-116) and rays below -6 sigma
    are absorbed; outside `active`, rays are untouched."""
    sigma = 0.1
    med = mf.MacrofacetMedium(kind=mf.NdfKind.GENERALIZED, a3=mf.RoughnessTriple(0.8, 0.8, 0.5),
                              sigma=sigma, fresnel_one=True)
    sc = mf.ShellScene(primitives=(mf.ShellPrimitive(mf.Plane(0.0), med),),
                       camera=mf.Camera((0, 0, 5), (0, 0, 0), 40, 4, 4))
    n = 1 << 18
    th = math.radians(150.0)
    d = np.array([math.sin(th), 0.0, math.cos(th)])
    o = np.broadcast_to(np.array([0.0, 0.0, 1.0]), (n, 3))
    active = np.ones(n, dtype=bool)
    active[:1000] = False
    rng = mf.BatchRng(mf.derive_bases(9, 2, np.arange(n)), np.zeros(n, dtype=np.uint64))
    state, pos, travel, w, prim = mf.walk(sc, o, np.broadcast_to(d, (n, 3)), rng,
                                          active=active)
    assert np.all(state[:1000] == 0) and np.array_equal(pos[:1000], o[:1000])
    assert np.all(rng.counter[:1000] == 0) and np.all(rng.counter[1000:] == 1)
    st, h = state[1000:], pos[1000:, 2]
    m = parity.f32_medium(med)
    hits = st == 2
    assert np.all(prim[1000:][hits] == 0)
    assert np.all((h[hits] >= -6 * sigma - 1e-4) & (h[hits] <= 3 * sigma + 1e-4))
    for hq in (0.2, 0.1, 0.0, -0.1, -0.3):
        p_ref = 1.0 - float(om.planar_transmittance(3 * sigma, hq, d[2], d, m))
        p = float(np.mean(hits & (h >= hq)))
        assert abs(p - p_ref) <= 4 * math.sqrt(p_ref * (1 - p_ref) / st.size) + 1e-4, (hq, p, p_ref)
    p_abs = float(np.mean(st == 1))
    p_ref = float(om.planar_transmittance(3 * sigma, -6 * sigma, d[2], d, m))
    assert abs(p_abs - p_ref) <= 4 * math.sqrt(max(p_ref, 1e-9) / st.size) + 1e-6


def test_sample_collision_events(cuda):
    """sample_collision (transport.py:316-416): one tentative collision per
    call -- real or null -- inside the shell, with its field value, frame
    and distance; the counter advances; real events dominate where the
    majorant is tight."""
    med = mf.MacrofacetMedium(kind=mf.NdfKind.GENERALIZED, a3=mf.RoughnessTriple(1, 1, 1),
                              sigma=0.3, fresnel_one=True)
    sc = mf.ShellScene(primitives=(mf.ShellPrimitive(mf.Sphere((0, 0, 0), 1.0), med),),
                       camera=mf.Camera((0, 0, 5), (0, 0, 0), 40, 4, 4))
    rs = mf.RandomStream(4, 2)
    kinds = []
    o = np.array([0.0, 0.1, 3.0])
    d = np.array([0.0, 0.0, -1.0])
    for _ in range(200):
        ev = mf.sample_collision((o, d), sc, rs)
        kinds.append(ev.kind)
        if ev.kind is not mf.EventKind.ABSORBED_BY_EXIT:
            assert ev.prim_index == 0
            assert -0.9 - 1e-4 <= ev.local_f <= 0.9 + 1e-4
            assert abs(ev.distance - np.linalg.norm(ev.position - o)) < 1e-4
            assert abs(ev.local_f - (np.linalg.norm(ev.position) - 1.0)) < 1e-5
            np.testing.assert_allclose(ev.local_frame.normal, ev.position /
                                       np.linalg.norm(ev.position), atol=1e-5)
    assert rs.counter == 200
    real = sum(k is mf.EventKind.REAL_SCATTER for k in kinds)
    null = sum(k is mf.EventKind.NULL_SCATTER for k in kinds)
    assert real > 0 and null > 0 and real + null > 150


def _box_scene(M):
    med = M.MacrofacetMedium(kind=M.NdfKind.BECKMANN, a3=M.RoughnessTriple(0.4, 0.9, 0.0),
                             sigma=0.3)
    cam = M.Camera(position=(0, 0, 9), look_at=(0.5, 0, 0), fov_deg=35, width=8, height=8)
    return M.ShellScene(primitives=(M.ShellPrimitive(M.Box((0, 0, 0), (1.5, 1.5, 0.8)), med),),
                        camera=cam, environment=M.Environment(radiance=(1.0, 0.8, 0.6)),
                        sun=M.DirectionalLight(direction=(0.3, 0.2, -0.9), radiance=(2, 2, 2)))


def test_box_shell_matches_oracle(cuda):
    """Box shells on the device (sdf.py:55-84; Lipschitz gaps + the recede
    test, transport.py:93,105-108) vs the oracle's reference-faithful
    render of the same scene: image mean and per-pixel agreement."""
    sc = _box_scene(mf)
    img, st = mf.render_device(sc, 8192, 5, max_bounces=16, stats=True)
    assert st["majorant_violations"] == 0 and st["capped"] == 0 and st["nonfinite"] == 0
    g = img.cpu().numpy().astype(np.float64)
    ref = tracer.render(_box_scene(R), spp=256, seed=22, max_bounces=16, tile=8)
    # per-pixel oracle SE from a second oracle render
    ref2 = tracer.render(_box_scene(R), spp=256, seed=23, max_bounces=16, tile=8)
    se = np.abs(ref - ref2) / math.sqrt(2.0)
    m = 0.5 * (ref + ref2)
    se_m = math.sqrt(np.mean(se ** 2) / 2.0 / g.size)
    assert abs(g.mean() - m.mean()) <= 4 * se_m + 1e-3 * m.mean(), (g.mean(), m.mean(), se_m)
    # the same scene from the reference-shaped classes is bit-identical
    img2, _ = mf.render_device(_box_scene(R), 8192, 5, max_bounces=16)
    assert cuda.equal(img, img2)


def _env_map(h=16, w=32):
    th = (np.arange(h) + 0.5) / h * np.pi
    ph = (np.arange(w) + 0.5) / w * 2 * np.pi
    T, P = np.meshgrid(th, ph, indexing="ij")
    return np.stack([0.5 + 0.4 * np.cos(T), 0.5 + 0.3 * np.sin(P) * np.sin(T),
                     0.3 + 0.2 * np.cos(2 * P) * np.sin(T) ** 2], axis=-1)


def test_latlong_environment_matches_oracle_eval(cuda):
    """Lat-long environment on the device (scene.py:61-84): with no shells
    every camera ray escapes, so each pixel is the environment averaged
    over its footprint -- compared with the oracle's bilinear lookup
    integrated over a dense sub-pixel grid."""
    env = mf.Environment(radiance=(0, 0, 0), latlong=_env_map())
    cam = mf.Camera(position=(0, 0, 0), look_at=(1, 0.3, 0.2), fov_deg=60, width=12, height=8)
    sc = mf.ShellScene(primitives=(), camera=cam, environment=env)
    img, _ = mf.render_device(sc, 4096, 1, max_bounces=1)
    g = img.cpu().numpy().astype(np.float64)
    k = 48
    jx, jy = np.meshgrid((np.arange(k) + 0.5) / k, (np.arange(k) + 0.5) / k)
    ref = np.zeros((8, 12, 3))
    for py in range(8):
        for px in range(12):
            o, d = tracer.camera_rays(cam, np.full(k * k, px), np.full(k * k, py), jx.ravel(),
                                      jy.ravel())
            ref[py, px] = tracer.env_radiance(env, d).mean(axis=0)
    np.testing.assert_allclose(g, ref, rtol=3e-3, atol=1e-4)


def test_latlong_environment_pool_matches_megakernel(cuda, monkeypatch):
    """A lat-long map on a single plane runs the colour path pool; its image
    is bit-identical to the megakernel's."""
    base = configs.config2_scene(64, 48)
    import dataclasses

    sc = dataclasses.replace(base, environment=mf.Environment(radiance=(0, 0, 0),
                                                              latlong=_env_map()))
    a, sa = mf.render_device(sc, 32, 3, max_bounces=16, stats=True)
    a = a.cpu().numpy()
    assert a[..., 0].mean() > 0 and not np.array_equal(a[..., 0], a[..., 1])
    monkeypatch.setenv("MF_MEGAKERNEL", "1")
    b, sb = mf.render_device(sc, 32, 3, max_bounces=16, stats=True)
    assert np.array_equal(a, b.cpu().numpy())


def test_config_document_box_and_env_map_renders(cuda, tmp_path):
    """A config document naming a box shell and an env_map PFM (reference
    config.py:207-227) renders bit-identically to the same scene built
    directly from the classes."""
    from paper_2603_00280_b200.config import parse_config, scene_from_config

    env = _env_map().astype(np.float32)
    mf.write_pfm(mf.RadianceImage(env), str(tmp_path / "env.pfm"))
    text = ("[kernel]\nsigma = 0.3\nlx = 0.3\nly = 0.2\nlz = inf\n"
            "[medium]\nkind = beckmann\nfresnel = one\n"
            f"[scene]\nenv_map = {tmp_path / 'env.pfm'}\nenv_radiance = 0,0,0\n"
            "camera_position = 0,0,9\ncamera_look_at = 0.5,0,0\ncamera_fov_deg = 35\n"
            "primitive0_shape = box\nprimitive0_center = 0,0,0\n"
            "primitive0_half_extents = 1.5,1.5,0.8\n"
            "[render]\nwidth = 16\nheight = 16\n")
    sc = scene_from_config(parse_config(text))
    assert isinstance(sc.primitives[0].sdf, mf.Box)
    img, st = mf.render_device(sc, 256, 9, max_bounces=16, stats=True)
    assert st["majorant_violations"] == 0 and st["capped"] == 0 and st["nonfinite"] == 0
    direct = mf.ShellScene(primitives=(mf.ShellPrimitive(mf.Box((0, 0, 0), (1.5, 1.5, 0.8)),
                                                         sc.primitives[0].medium),),
                           camera=sc.camera,
                           environment=mf.Environment(radiance=(0, 0, 0), latlong=env))
    img2, _ = mf.render_device(direct, 256, 9, max_bounces=16)
    assert cuda.equal(img, img2)
    g = img.cpu().numpy()
    assert np.isfinite(g).all() and g.min() >= 0.0 and g.mean() > 0.05
