"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
package (/root/reference/pkg/src, importable only in the build container).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--quick]

Outputs (committed; the GPU box never reads /root/reference):
  config1_ref.npz    4096 config-1 queries evaluated by the reference
                     (extinction, phase_eval, restated pdf, _phase_sample_u)
                     on float32-exact inputs and float32-rounded parameters
  render_ref.npz     small reference renders (plane+sun, sphere+sun, box),
                     to pin the oracle's RNG consumption bit-for-bit
  anchors.json       render-level anchors: config-2 depth-1 collision-depth
                     quadrature and reference Monte-Carlo means +- SE at
                     depth 1 / 16, config-4 panel means, furnace mean
  config3_ref.npz    reduced config-3 image (sphere + point light) from the
                     oracle's composed point-light loop (reference functions
                     + the recorded NEE convention) with the corrected
                     sphere-root selection, per-pixel mean and SE
  config3_ref128.npz the same at 128x128 x 8192 spp (the per-pixel z-test
                     and relMSE of tests/test_gpu_render.py)
  config1_samples_ref.npz
                     the reference's _phase_sample_u outputs (direction,
                     pdf, weight; float32) for the first 32768 queries of
                     the full config-1 batch (configs.config1_inputs())
"""

from __future__ import annotations

import json
import math
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)
sys.path.insert(0, REF)

import macrofacet as M  # noqa: E402
from macrofacet import medium as Mmed  # noqa: E402
from macrofacet.ndf import _vndf_sample_u, projected_area_dir  # noqa: E402
from macrofacet.render import trace_paths as ref_trace_paths  # noqa: E402
from macrofacet.rng import derive_bases  # noqa: E402
from macrofacet.transport import BatchRng  # noqa: E402

from paper_2603_00280_b200 import configs  # noqa: E402

F32 = lambda v: float(np.float32(v))  # noqa: E731


def ref_medium_f32(kind, a, sigma, **kw):
    return M.MacrofacetMedium(kind=kind, a3=M.RoughnessTriple(F32(a[0]), F32(a[1]), F32(a[2])),
                              sigma=F32(sigma), **kw)


def ref_phase_pdf(wo, wi, med, frame):
    """pdf of _phase_sample_u's direction, composed from reference pieces
    (ndf.py:397-405 mixture pdf at the half vector, medium.py:186-189)."""
    wol = frame.to_local(wo)
    wil = frame.to_local(wi)
    v = -wol
    h = v + wil
    hn = np.linalg.norm(h, axis=-1)
    h = h / hn[..., None]
    sig_b = projected_area_dir(wol, M.NdfKind.BECKMANN, med.a3)
    guided = sig_b > 1e-12
    vm = np.sum(v * h, axis=-1)
    pb = np.where(guided, np.maximum(vm, 0) * M.beckmann_ndf(h, med.a3.ax, med.a3.ay)
                  / np.where(guided, sig_b, 1.0), 0.0)
    pu = np.where(vm > 0, 1.0 / (2 * np.pi), 0.0)
    r = np.where(guided, med.mix_ratio, 0.0)
    pm = r * pb + (1 - r) * pu
    return np.where(vm > 1e-12, pm / (4 * vm), 0.0)


def make_config1(n=4096):
    p, wo, wi, u = configs.config1_inputs(n=n)
    a = math.sqrt(2) * 0.05 / 0.1
    med = ref_medium_f32(M.NdfKind.GENERALIZED, (a, a, a), 0.05, fresnel_one=True)
    frame = M.build_frame(np.array([0.0, 0.0, 1.0]))
    P, WO, WI = (x.astype(np.float64) for x in (p, wo, wi))
    st = M.extinction(WO, P[:, 2], med, frame)
    ph = M.phase_eval(WO, WI, med, frame)
    pdf = ref_phase_pdf(WO, WI, med, frame)
    u1 = u[:, 0]
    half = np.float32(0.5)
    uu = np.where(u1 < half, u1 / half, (u1 - half) / half).astype(np.float32)
    U3 = np.stack([u1, uu, u[:, 1]], axis=-1).astype(np.float64)
    ws, pdf_s, w = Mmed._phase_sample_u(frame.to_local(WO), med, U3)
    np.savez_compressed(os.path.join(HERE, "config1_ref.npz"), p=p, wo=wo, wi=wi, u=u,
                        sigma_t=st, phase=ph, pdf=pdf, ws=ws, pdf_s=pdf_s, w=w)


def make_config1_samples(n=32768):
    """Reference phase samples of the first n queries of the 2^20 config-1
    batch (two-uniform convention u = (u1, u1', u2))."""
    p, wo, wi, u = configs.config1_inputs()
    wo, u = wo[:n], u[:n]
    a = math.sqrt(2) * 0.05 / 0.1
    med = ref_medium_f32(M.NdfKind.GENERALIZED, (a, a, a), 0.05, fresnel_one=True)
    frame = M.build_frame(np.array([0.0, 0.0, 1.0]))
    u1 = u[:, 0]
    half = np.float32(0.5)
    uu = np.where(u1 < half, u1 / half, (u1 - half) / half).astype(np.float32)
    U3 = np.stack([u1, uu, u[:, 1]], axis=-1).astype(np.float64)
    ws, pdf_s, w = Mmed._phase_sample_u(frame.to_local(wo.astype(np.float64)), med, U3)
    np.savez_compressed(os.path.join(HERE, "config1_samples_ref.npz"), n=n,
                        ws=ws.astype(np.float32), pdf_s=pdf_s.astype(np.float32),
                        w=w[:, 0].astype(np.float32))


def make_renders():
    iso = M.RoughnessTriple(1, 1, 1)
    med = M.MacrofacetMedium(kind=M.NdfKind.GENERALIZED, a3=iso, sigma=1.0, fresnel_one=True)
    cam = M.Camera(position=(0, 0, 10), look_at=(1.5, 0, 0), fov_deg=35, width=12, height=12)
    sun = M.DirectionalLight(direction=(0.3, 0.1, -0.9), radiance=(1, 1, 1))
    plane = M.ShellScene(primitives=(M.ShellPrimitive(M.Plane(0.0), med),), camera=cam, sun=sun)
    med2 = M.MacrofacetMedium(kind=M.NdfKind.GENERALIZED, a3=iso, sigma=0.4)
    cam2 = M.Camera(position=(0, 0, 9), look_at=(0.5, 0, 0), fov_deg=35, width=8, height=8)
    sph = M.ShellScene(primitives=(M.ShellPrimitive(M.Sphere((0, 0, 0), 2.0), med2),),
                       camera=cam2, sun=M.DirectionalLight(direction=(0.3, 0.2, -0.9),
                                                           radiance=(2, 2, 2)))
    box = M.ShellScene(primitives=(M.ShellPrimitive(
        M.Box((0, 0, 0), (1.5, 1.5, 0.8)),
        M.MacrofacetMedium(kind=M.NdfKind.BECKMANN, a3=M.RoughnessTriple(0.4, 0.9, 0),
                           sigma=0.3)),), camera=cam2)
    out = {
        "plane": M.render(plane, spp=4, seed=3).pixels,
        "sphere": M.render(sph, spp=4, seed=21).pixels,
        "box": M.render(box, spp=4, seed=22).pixels,
    }
    np.savez_compressed(os.path.join(HERE, "render_ref.npz"), **out)


# ---------------------------------------------------------------------------
# planar anchors (config 2 / 4), reference trace_paths with grey albedo

def _albedo_patch(albedo):
    orig = Mmed._fresnel_rgb

    def grey(medium, cos_i):
        return np.full(np.shape(cos_i) + (3,), float(albedo))

    Mmed._fresnel_rgb = grey
    return orig


def _planar_job(args):
    kind, a3, sigma, albedo, depth, n, seed, stream = args
    _albedo_patch(albedo)
    med = M.MacrofacetMedium(kind=M.NdfKind(kind), a3=M.RoughnessTriple(*a3), sigma=sigma)
    to_light = np.array(configs.TO_LIGHT_C2)
    sun = M.DirectionalLight(direction=tuple(-to_light), radiance=(1.0, 1.0, 1.0))
    cam = M.Camera(position=(0, 0, 10), look_at=(0, 0, 0), fov_deg=30, width=4, height=4)
    scene = M.ShellScene(primitives=(M.ShellPrimitive(M.Plane(0.0), med),), camera=cam,
                         environment=M.Environment(radiance=(0.0, 0.0, 0.0)), sun=sun)
    d = np.array(configs.CAM_TRAVEL_C2)
    o = np.broadcast_to(np.array([0.0, 0.0, 4.0 * sigma]) - d * 0.0, (n, 3))
    brng = BatchRng(derive_bases(seed, stream, np.arange(n)), np.zeros(n, dtype=np.uint64))
    rad = ref_trace_paths(o, np.broadcast_to(d, (n, 3)), scene, depth, brng)
    v = rad[:, 0]
    return float(v.sum()), float((v * v).sum()), n


def planar_mc(kind, a3, sigma, albedo, depth, n_total, seed, pool, chunk=20000):
    jobs = [(kind, a3, sigma, albedo, depth, chunk, seed, k) for k in range(n_total // chunk)]
    s = ss = cnt = 0.0
    for a, b, c in pool.map(_planar_job, jobs):
        s += a
        ss += b
        cnt += c
    mean = s / cnt
    var = ss / cnt - mean * mean
    return mean, math.sqrt(var / cnt), int(cnt)


def depth1_quadrature(kind, a3, sigma, albedo):
    """Deterministic single-scatter value: int Tr_in sigma_t/|cos| phase Tr_out dh
    over the collision band [-6s, 3s] (Tr_out over max(h, -3s) to mirror the
    ratio-mode vacuum), like test_scene_render.py:250-258."""
    orig = _albedo_patch(albedo)
    try:
        med = M.MacrofacetMedium(kind=M.NdfKind(kind), a3=M.RoughnessTriple(*a3), sigma=sigma)
        frame = M.build_frame(np.array([0.0, 0.0, 1.0]))
        d = np.array(configs.CAM_TRAVEL_C2)
        tl = np.array(configs.TO_LIGHT_C2)
        h = np.linspace(-6 * sigma, 3 * sigma, 200001)
        sig_t = M.extinction(d, h, med, frame)
        th_v = np.arccos(d[2])
        tr_in = M.planar_transmittance(3 * sigma, h, th_v, 0.0, med)
        th_l = np.arccos(tl[2])
        tr_out = M.planar_transmittance(np.maximum(h, -3 * sigma), 3 * sigma, th_l, 0.0, med)
        ph = float(M.phase_eval(d, tl, med, frame)[0])
        integ = tr_in * (sig_t / abs(d[2])) * ph * tr_out
        return float(np.trapezoid(integ, h))
    finally:
        Mmed._fresnel_rgb = orig


def make_anchors(quick=False):
    workers = os.cpu_count() or 1
    pool = mp.get_context("fork").Pool(workers)
    out = {"generated_by": "tests/golden/make_golden.py (reference package at /root/reference)",
           "conventions": "camera travel (cos45,0,-sin45), to-light (cos30,0,sin30), unit "
                          "irradiance, black env, grey albedo as F, R=0.5"}
    a = math.sqrt(2) * 0.05 / 0.05
    c2 = ("generalized", (a, a, a), 0.05, 0.8)
    out["config2_depth1_quadrature"] = depth1_quadrature(*c2)
    n = 200000 if quick else 1000000
    t = time.time()
    m, se, cnt = planar_mc(*c2, 1, n, 11, pool)
    out["config2_depth1_mc"] = {"mean": m, "se": se, "n": cnt}
    m, se, cnt = planar_mc(*c2, 16, n, 12, pool)
    out["config2_depth16_mc"] = {"mean": m, "se": se, "n": cnt}
    print(f"config2 anchors {time.time() - t:.0f}s", flush=True)
    panels = {}
    n4 = 100000 if quick else 400000
    for sigma in configs.CONFIG4_SIGMAS:
        for lz in configs.CONFIG4_LZ:
            s2 = math.sqrt(2) * sigma
            if math.isinf(lz):
                spec = ("beckmann", (s2 / 0.05, s2 / 0.05, 0.0), sigma, 0.8)
            else:
                spec = ("generalized", (s2 / 0.05, s2 / 0.05, s2 / lz), sigma, 0.8)
            t = time.time()
            m, se, cnt = planar_mc(*spec, 64, n4, 13, pool)
            key = f"sigma={sigma},lz={'inf' if math.isinf(lz) else lz}"
            panels[key] = {"mean": m, "se": se, "n": cnt, "depth1_quadrature":
                           depth1_quadrature(*spec)}
            print(f"panel {key}: {m:.6f} +- {se:.6f} ({time.time() - t:.0f}s)", flush=True)
    out["config4_depth64_mc"] = panels
    pool.close()
    with open(os.path.join(HERE, "anchors.json"), "w") as fh:
        json.dump(out, fh, indent=1)


# ---------------------------------------------------------------------------
# config 3 at reduced resolution via the oracle (pinned to the reference)

def _c3_job(args):
    from oracle import tracer

    # the reference's sphere root selection tunnels rays through shells
    # (DESIGN.md "Reference defect"); the fixture uses the corrected roots
    tracer.SPHERE_ROOTS = "corrected"

    ys, xs, spp, tile, w = args
    scene = configs.config3_scene(w, w)
    cam = scene.camera
    # per-pixel mean and second moment: trace each pixel's samples
    ye, xe = min(cam.height, ys + tile), min(cam.width, xs + tile)
    yy, xx = np.mgrid[ys:ye, xs:xe]
    pix = (yy * cam.width + xx).ravel()
    from oracle.numerics import RayStreams, stream_base
    base = stream_base(np.uint64(2), pix.astype(np.uint64))
    rs = RayStreams(np.repeat(base, spp),
                    np.tile(np.arange(spp, dtype=np.uint64), pix.size) * tracer.SAMPLE_STRIDE)
    jx = rs.draw()
    jy = rs.draw()
    o, d = tracer.camera_rays(cam, np.repeat(xx.ravel(), spp), np.repeat(yy.ravel(), spp), jx, jy)
    rad = tracer.trace_paths(o, d, scene, 32, rs).reshape(pix.size, spp, 3)
    return ys, xs, ye, xe, rad.mean(axis=1), rad.var(axis=1) / spp


def make_config3(quick=False, w=32, spp=None, name="config3_ref.npz"):
    spp = spp or (64 if quick else 256)
    tile = 8
    jobs = [(ys, xs, spp, tile, w) for ys in range(0, w, tile) for xs in range(0, w, tile)]
    pool = mp.get_context("fork").Pool(os.cpu_count() or 1)
    mean = np.zeros((w, w, 3))
    var = np.zeros((w, w, 3))
    for ys, xs, ye, xe, m, v in pool.map(_c3_job, jobs):
        mean[ys:ye, xs:xe] = m.reshape(ye - ys, xe - xs, 3)
        var[ys:ye, xs:xe] = v.reshape(ye - ys, xe - xs, 3)
    pool.close()
    np.savez_compressed(os.path.join(HERE, name), mean=mean.astype(np.float32),
                        se=np.sqrt(var).astype(np.float32), spp=spp, width=w)


if __name__ == "__main__":
    quick = "--quick" in sys.argv
    what = [a for a in sys.argv[1:] if not a.startswith("--")] or \
        ["config1", "renders", "config3", "anchors"]
    for wname in what:
        t = time.time()
        {"config1": make_config1, "renders": make_renders,
         "anchors": lambda: make_anchors(quick), "config3": lambda: make_config3(quick),
         "config3_128": lambda: make_config3(quick, 128, 8192, "config3_ref128.npz"),
         "config1_samples": make_config1_samples}[wname]()
        print(f"{wname}: {time.time() - t:.0f}s", flush=True)
