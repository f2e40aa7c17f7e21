"""Diagnostic: GPU vs oracle image means on reduced config-3 variants."""
import os, sys, time, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
from oracle import tracer
from oracle.numerics import RayStreams, stream_base
import multiprocessing as mp

def oracle_img(scene, spp, seed, depth):
    cam = scene.camera
    yy, xx = np.mgrid[0:cam.height, 0:cam.width]
    pix = (yy * cam.width + xx).ravel()
    base = stream_base(np.uint64(seed), pix.astype(np.uint64))
    rs = RayStreams(np.repeat(base, spp), np.tile(np.arange(spp, dtype=np.uint64), pix.size) * tracer.SAMPLE_STRIDE)
    jx = rs.draw(); jy = rs.draw()
    o, d = tracer.camera_rays(cam, np.repeat(xx.ravel(), spp), np.repeat(yy.ravel(), spp), jx, jy)
    rad = tracer.trace_paths(o, d, scene, depth, rs)[:, 0]
    return rad

def job(a):
    variant, depth, spp, seed = a
    sc = make(variant)
    r = oracle_img(sc, spp, seed, depth)
    return r.sum(), (r * r).sum(), r.size

def make(variant):
    sc = configs.config3_scene(16, 16)
    if variant == "sun":
        sc = mf.ShellScene(primitives=sc.primitives, camera=sc.camera, environment=mf.Environment((0.0, 0.0, 0.0)),
                           sun=mf.DirectionalLight(direction=(-1, -1, -1), radiance=(1, 1, 1)))
    elif variant == "env":
        sc = mf.ShellScene(primitives=sc.primitives, camera=sc.camera, environment=mf.Environment((1.0, 1.0, 1.0)))
    elif variant == "point0":
        sc = mf.ShellScene(primitives=sc.primitives, camera=sc.camera, environment=mf.Environment((0.0, 0.0, 0.0)), point=sc.point)
    return sc

pool = mp.get_context("fork").Pool(os.cpu_count())
for variant, depth in (("point0", 1), ("sun", 1), ("env", 1), ("env", 32), ("point0", 32)):
    t = time.time()
    res = pool.map(job, [(variant, depth, 32, 100 + k) for k in range(os.cpu_count() * 2)])
    s = sum(r[0] for r in res); ss = sum(r[1] for r in res); n = sum(r[2] for r in res)
    m = s / n; se = math.sqrt((ss / n - m * m) / n)
    sc = make(variant)
    img, st = mf.render_device(sc, 65536, 5, max_bounces=depth, stats=True)
    v = img[..., 0].cpu().numpy().astype(np.float64)
    print(f"{variant} depth {depth}: oracle {m:.6f} +- {se:.6f} (n={n}, {time.time()-t:.0f}s)  gpu {v.mean():.6f}  z={(v.mean()-m)/se:.2f}  steps/path {st['track_steps']/st['paths']:.1f}", flush=True)
