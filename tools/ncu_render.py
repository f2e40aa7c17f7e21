"""One workload render for an ncu capture (reduced size):
    python tools/ncu_render.py config4|config3|config5 [width] [spp]
config4 renders the centre panel (sigma 0.05, l_z 0.1).  Two renders: the
first warms the slope table / scene caches, the second is the captured one
(ncu -k regex:<kernel> -s 1 -c 1)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_2603_00280_b200 as mf  # noqa: E402
from paper_2603_00280_b200 import configs  # noqa: E402

wl = sys.argv[1]
w = int(sys.argv[2]) if len(sys.argv) > 2 else 512
spp = int(sys.argv[3]) if len(sys.argv) > 3 else 64
torch.cuda.set_device(0)
if wl == "config4":
    sc, seed, mb = configs.config4_scene(0.05, 0.1, w, w), 3, 64
elif wl == "config3":
    sc, seed, mb = configs.config3_scene(w, w), 2, 32
elif wl == "config5":
    sc, seed, mb = configs.config5_scene(w, w), 4, 64
else:
    raise SystemExit(wl)
for _ in range(2):
    img, st = mf.render_device(sc, spp, seed, max_bounces=mb, stats=True)
torch.cuda.synchronize()
print(wl, w, spp, st)
