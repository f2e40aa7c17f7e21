"""Per-core speed of the oracle port (oracle/tracer.py, the CPU baseline
bench.py times on the GPU box) against the reference package itself
(/root/reference, importable only in the build container), on the same
config-4 tile jobs, one process each.  Writes profiles/r02_port_vs_reference.json.
The reference renders with the grey-albedo Fresnel patch of
tests/golden/make_golden.py and the same orthographic rays."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
import macrofacet as M  # noqa: E402
from macrofacet import medium as Mmed  # noqa: E402
from macrofacet.render import trace_paths as ref_trace  # noqa: E402
from macrofacet.rng import stream_base  # noqa: E402
from macrofacet.transport import BatchRng  # noqa: E402

from oracle import tracer  # noqa: E402
from oracle.numerics import RayStreams  # noqa: E402
from oracle.numerics import stream_base as o_stream_base  # noqa: E402
from paper_2603_00280_b200 import configs  # noqa: E402

orig = Mmed._fresnel_rgb
Mmed._fresnel_rgb = lambda medium, cos_i: np.full(np.shape(cos_i) + (3,), 0.8)

out = []
for sigma, lz in ((0.05, 0.1), (0.2, 0.02)):
    sc = configs.config4_scene(sigma, lz, 64, 64)
    m = sc.primitives[0].medium
    kind = M.NdfKind(m.kind.value)
    rmed = M.MacrofacetMedium(kind=kind, a3=M.RoughnessTriple(m.a3.ax, m.a3.ay, m.a3.az),
                              sigma=m.sigma)
    rsc = M.ShellScene(primitives=(M.ShellPrimitive(M.Plane(0.0), rmed),),
                       camera=M.Camera((0, 0, 10), (0, 0, 0), 30, 4, 4),
                       environment=M.Environment(radiance=(0, 0, 0)),
                       sun=M.DirectionalLight(direction=sc.sun.direction, radiance=(1, 1, 1)))
    cam = sc.camera
    spp, tile = 16, 32
    yy, xx = np.mgrid[0:tile, 0:tile]
    pix = (yy * cam.width + xx).ravel()
    n = pix.size * spp
    # identical rays for both (the port's camera, jitter from the port's streams)
    rs = RayStreams(np.repeat(o_stream_base(np.uint64(3), pix.astype(np.uint64)), spp),
                    np.tile(np.arange(spp, dtype=np.uint64), pix.size) * tracer.SAMPLE_STRIDE)
    o, d = tracer.camera_rays(cam, np.repeat(xx.ravel(), spp), np.repeat(yy.ravel(), spp),
                              rs.draw(), rs.draw())
    t0 = time.perf_counter()
    tracer.trace_paths(o, d, sc, 64, rs)
    t_port = time.perf_counter() - t0
    brng = BatchRng(np.repeat(stream_base(3, pix.astype(np.uint64)), spp),
                    np.tile(np.arange(spp, dtype=np.uint64), pix.size) << np.uint64(28))
    t0 = time.perf_counter()
    ref_trace(o, d, rsc, 64, brng)
    t_ref = time.perf_counter() - t0
    out.append({"panel": f"sigma={sigma},l_z={lz}", "paths": int(n),
                "port_paths_per_s": n / t_port, "reference_paths_per_s": n / t_ref,
                "port_over_reference": t_ref / t_port})
    print(out[-1], flush=True)
Mmed._fresnel_rgb = orig
res = {"what": "one process, same rays, config-4 panels 32x32 px x 16 spp, depth 64",
       "host": os.uname().nodename, "cpu_count": os.cpu_count(), "results": out}
with open(os.path.join(ROOT, "profiles", "r02_port_vs_reference.json"), "w") as fh:
    json.dump(res, fh, indent=1)
