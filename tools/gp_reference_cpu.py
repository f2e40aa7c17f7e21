"""CPU time of the REFERENCE gp.ensemble_radiance on a bounded sample of the
bench's gp workload (run in the build container, where /root/reference is
importable; the GPU box cannot import it).  Writes
profiles/r02_gp_reference_cpu.json.

    PYTHONDONTWRITEBYTECODE=1 python tools/gp_reference_cpu.py"""
import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np  # noqa: E402
from macrofacet import gp  # noqa: E402
from macrofacet.ndf import KernelParams  # noqa: E402
from macrofacet.rng import RandomStream  # noqa: E402
from macrofacet.scene import Camera  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sigma, ell = 0.05, 0.05
k = KernelParams(sigma, ell, ell, ell)
w = h = 16
rounds = 2
cam = Camera(position=(0, 0, 8 * sigma + 2), look_at=(1.0, 0, 0), fov_deg=35, width=w, height=h)
t0 = time.perf_counter()
img = gp.ensemble_radiance(k, cam, rounds, rounds, RandomStream(0, 0), max_bounces=64)
dt = time.perf_counter() - t0
paths = w * h * rounds
rec = {"what": "reference gp.ensemble_radiance (numpy, one process) on the build container's CPU",
       "sample": f"{w}x{h} pixels x {rounds} rounds (realisations), kernel sigma {sigma}, "
                 f"l {ell}, CLI gp-ensemble camera, max_bounces 64",
       "paths": paths, "seconds": dt, "paths_per_s": paths / dt,
       "cpu_count": os.cpu_count(), "mean_pixel": float(img.mean())}
with open(os.path.join(ROOT, "profiles", "r02_gp_reference_cpu.json"), "w") as fh:
    json.dump(rec, fh, indent=1)
print(rec)
