"""Config-3 check: the single-sphere walker (mode 3) against the general
walker (MF_GENERIC_WALK=1) -- bit-identical images -- and their times."""
import os
import subprocess
import sys

code = r'''
import os, sys, json, hashlib
sys.path.insert(0, os.getcwd())
import torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
torch.cuda.set_device(0)
sc = configs.config3_scene(256, 256)
out = torch.empty((256, 256, 3), device="cuda")
for _ in range(2): mf.render_device(sc, 64, 2, max_bounces=32, out=out)
ts = []
for _ in range(5):
    _, st = mf.render_device(sc, 64, 2, max_bounces=32, out=out, stats=True)
    ts.append(st["path_kernel_ms"])
print(json.dumps({"ms": min(ts), "hash": hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:12],
                  "steps_per_path": st["track_steps"] / st["paths"]}))
'''
for generic in ("0", "1"):
    env = dict(os.environ, MF_GENERIC_WALK=generic)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("generic" if generic == "1" else "mode3", r.stdout.strip() or r.stderr[-1500:])
