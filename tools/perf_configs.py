"""Throughput of every BASELINE config on one GPU (CUDA events, after
warm-up); writes JSON to stdout.  Reduced sizes where the full config is a
multi-GPU job (config 4 panels at 1024^2 x 64 spp, config 5 at 512^2 x 16 spp).

    python tools/perf_configs.py [config1 config2 ...]   (default: all)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_00280_b200 as mf  # noqa: E402
from paper_2603_00280_b200 import _lib, configs, roofline  # noqa: E402


def timed(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def render_case(name, scene, spp, seed, depth, reps=3):
    out = torch.empty((scene.camera.height, scene.camera.width, 3), device="cuda")
    ms = timed(lambda: mf.render_device(scene, spp, seed, max_bounces=depth, out=out), reps)
    _, st = mf.render_device(scene, spp, seed, max_bounces=depth, out=out, stats=True)
    paths = scene.camera.width * scene.camera.height * spp
    return {"case": name, "paths": paths, "ms": ms, "Mpaths_s": paths / ms / 1e3,
            "mean": float(out.mean()), "per_path": {k: v / st["paths"] for k, v in st.items()
                                                     if k not in ("paths", "path_kernel_ms")}}


torch.cuda.set_device(0)
res = []
# FP32 / MUFU issue peaks measured on this device (as bench.py)
_lib_h = _lib.load()
_f, _s = _lib.ctypes.c_double(), _lib.ctypes.c_double()
_lib.check(_lib_h.mf_measure_peaks(_lib.ctypes.byref(_f), _lib.ctypes.byref(_s),
                                   _lib.stream_handle(torch, torch.device("cuda", 0))))
PEAK = (_f.value, _s.value)
ONLY = sys.argv[1:]


def want(name):
    return not ONLY or any(name.startswith(o) for o in ONLY)



p, wo, wi, u = configs.config1_inputs()
d = torch.device("cuda", 0)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(d)  # noqa: E731
med = configs.config1_medium()
for reps in ((1, 16) if want("config1") else ()):
    P, WO, WI = (T(a.T).repeat(1, reps).contiguous() for a in (p, wo, wi))
    U1, U2 = T(u[:, 0]).repeat(reps), T(u[:, 1]).repeat(reps)
    ms = timed(lambda: mf.query_batch(med, P, WO, WI, U1, U2), 5, 2)
    n = (1 << 20) * reps
    res.append({"case": f"config1 queries N=2^{20 + (4 if reps == 16 else 0)}", "ms": ms,
                "Mqueries_s": n / ms / 1e3, "bytes_per_query": 96,
                "GB_s": n * 96 / ms / 1e6,
                "roofline": roofline.query_roofline(n, ms, PEAK[0], PEAK[1])})
if want("config2"):
    res.append(render_case("config2 256^2 x 64 spp d16", configs.config2_scene(), 64, 1, 16, 10))
if want("config3"):
    res.append(render_case("config3 512^2 x 256 spp d32", configs.config3_scene(), 256, 2, 32, 2))
for sig in (configs.CONFIG4_SIGMAS if want("config4") else ()):
    for lz in configs.CONFIG4_LZ:
        res.append(render_case(f"config4 sigma={sig} lz={lz} 1024^2 x 64 spp d64",
                               configs.config4_scene(sig, lz), 64, 3, 64, 2))
if want("config5"):
    t0 = time.time()
    sc5 = configs.config5_scene(512, 512)
    build_s = time.time() - t0
    r5 = render_case("config5 512^2 x 16 spp d64", sc5, 16, 4, 64, 2)
    r5["field_build_s"] = build_s
    res.append(r5)
print(json.dumps(res, indent=1))
