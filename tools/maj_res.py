import sys, os, json, dataclasses
sys.path.insert(0, os.getcwd())
import torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
torch.cuda.set_device(0)
for res in (32, 48, 64, 80, 96, 128):
    sc = configs.config5_scene(512, 512)
    pr = sc.primitives[0]
    med = dataclasses.replace(pr.medium, majorant_res=res)
    sc = dataclasses.replace(sc, primitives=(dataclasses.replace(pr, medium=med),))
    out = torch.empty((512, 512, 3), device="cuda")
    for _ in range(2): mf.render_device(sc, 16, 4, max_bounces=64, out=out)
    ts = []
    for _ in range(4):
        _, st = mf.render_device(sc, 16, 4, max_bounces=64, out=out, stats=True)
        ts.append(st["path_kernel_ms"])
    print(res, round(min(ts), 3), float(out.mean()), st["track_steps"] / st["paths"], st["majorant_violations"], flush=True)
