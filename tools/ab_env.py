"""A/B timing of one render under two environment settings of the library
(path-kernel time from its CUDA events; image difference reported).
    python tools/ab_env.py VAR workload [width spp]   (VAR=0 vs unset)"""
import os
import subprocess
import sys

code = r'''
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
wl, w, spp = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
torch.cuda.set_device(0)
if wl == "config4": sc, seed, mb = configs.config4_scene(0.05, 0.1, w, w), 3, 64
elif wl == "config4s2": sc, seed, mb = configs.config4_scene(0.2, 0.1, w, w), 3, 64
elif wl == "config3": sc, seed, mb = configs.config3_scene(w, w), 2, 32
elif wl == "config2": sc, seed, mb = configs.config2_scene(w, w), 1, 16
else: sc, seed, mb = configs.config5_scene(w, w), 4, 64
out = torch.empty((w, w, 3), device="cuda")
for _ in range(2): mf.render_device(sc, spp, seed, max_bounces=mb, out=out)
ts = []
for _ in range(5):
    _, st = mf.render_device(sc, spp, seed, max_bounces=mb, out=out, stats=True)
    ts.append(st["path_kernel_ms"])
np.save(sys.argv[4], out.cpu().numpy())
print(json.dumps({"ms": min(ts), "mean": float(out.mean())}))
'''
var, wl = sys.argv[1], sys.argv[2]
w = sys.argv[3] if len(sys.argv) > 3 else "512"
spp = sys.argv[4] if len(sys.argv) > 4 else "64"
res = {}
for tag, val in (("off", "0"), ("on", None)):
    env = dict(os.environ)
    if val is None:
        env.pop(var, None)
    else:
        env[var] = val
    r = subprocess.run([sys.executable, "-c", code, wl, w, spp, f"/tmp/ab_{tag}.npy"], env=env,
                       capture_output=True, text=True)
    res[tag] = r.stdout.strip() or r.stderr[-1500:]
    print(var, tag, res[tag], flush=True)
import numpy as np  # noqa: E402
a, b = np.load("/tmp/ab_off.npy"), np.load("/tmp/ab_on.npy")
print("identical" if np.array_equal(a, b) else f"max rel diff {np.max(np.abs(a - b) / np.maximum(np.abs(a), 1e-12)):.3e}")
