"""Efficiency of walker variants on config 3 (reduced): kernel time x
per-pixel variance (16 independent renders)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
torch.cuda.set_device(0)
sc = configs.config3_scene(128, 128)
variants = sys.argv[1:] or ["0:1.0001", "0:1.5", "0:2", "2:0"]
for v in variants:
    gw, ms = v.split(":")
    os.environ["MF_GENERIC_WALK"] = gw
    os.environ["MF_RATIO_MSCALE"] = ms
    mf.render_device(sc, 64, 2, max_bounces=32, stats=True)
    imgs, t, steps = [], 0.0, 0
    for k in range(16):
        img, st = mf.render_device(sc, 256, 100 + k, max_bounces=32, stats=True)
        imgs.append(img[..., 0].cpu().numpy().astype(np.float64))
        t += st["path_kernel_ms"]
        steps += st["track_steps"] / st["paths"]
    imgs = np.stack(imgs)
    var = float(imgs.var(axis=0, ddof=1).mean())
    print(f"{v:10s} ms/render {t / 16:.3f} steps/path {steps / 16:.2f} mean {imgs.mean():.6f} "
          f"pixvar {var:.3e} efficiency {1e3 / (var * t / 16):.4e}")
