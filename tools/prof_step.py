"""Minimal driver for ncu: W warm-up + K config-2 render steps (the bench
workload) on cuda:0, nothing else.   python tools/prof_step.py [K] [W] [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2603_00280_b200 as mf  # noqa: E402
from paper_2603_00280_b200 import configs  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = sys.argv[3] if len(sys.argv) > 3 else "c2"
torch.cuda.set_device(0)
if cfg == "c2":
    scene, kw = configs.config2_scene(), dict(spp=64, seed=1, max_bounces=16)
elif cfg == "c3":
    scene, kw = configs.config3_scene(256, 256), dict(spp=16, seed=2, max_bounces=32)
else:
    raise SystemExit(f"unknown config {cfg}")
out = torch.empty((scene.camera.height, scene.camera.width, 3), device="cuda")
for _ in range(w + k):
    mf.render_device(scene, kw["spp"], kw["seed"], max_bounces=kw["max_bounces"], out=out)
torch.cuda.synchronize()
print("done", float(out.mean()))
