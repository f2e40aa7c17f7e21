"""Config-5 / config-3 efficiency of the shadow-ray Russian-roulette threshold
(MF_SHADOW_RR build variants): path-kernel time x per-pixel variance
(variance over eight seeds of one reduced render each)."""
import json
import os
import subprocess
import sys

here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, json
sys.path.insert(0, %r)
import torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
torch.cuda.set_device(0)
out = {}
for name, sc, spp, mb in (("c5", configs.config5_scene(512, 512), 16, 64),
                          ("c3", configs.config3_scene(256, 256), 64, 32)):
    imgs, ts = [], []
    for seed in range(4, 12):
        mf.render_device(sc, spp, seed, max_bounces=mb)
        img, st = mf.render_device(sc, spp, seed, max_bounces=mb, stats=True)
        imgs.append(img[..., 0].double()); ts.append(st["path_kernel_ms"])
    x = torch.stack(imgs)
    var = x.var(dim=0, unbiased=True).mean().item()
    out[name] = {"ms": round(min(ts), 4), "var": var, "mean": x.mean().item(),
                 "ms_x_var": min(ts) * var}
print(json.dumps(out))
''' % here
for so in sys.argv[1:]:
    env = dict(os.environ, MF_LIB_PATH=os.path.abspath(so))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(so), r.stdout.strip() or r.stderr[-1500:], flush=True)
