"""Config 5 at a reduced film (512^2 x 16 spp): kernel time and event
counts per path (development timing)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
torch.cuda.set_device(0)
sc = configs.config5_scene(512, 512)
res = int(os.environ.get("MF_MAJ_RES", "0"))
if res:
    import dataclasses
    med = sc.primitives[0].medium
    med.majorant_res = res
for _ in range(2):
    img, st = mf.render_device(sc, 16, 4, max_bounces=64, stats=True)
ms = []
for _ in range(3):
    img, st = mf.render_device(sc, 16, 4, max_bounces=64, stats=True)
    ms.append(st["path_kernel_ms"])
print("c5 512^2x16 res", os.environ.get("MF_MAJ_RES"), min(ms), "ms", 512 * 512 * 16 / min(ms) / 1e3, "Mpaths/s",
      {k: round(v / st["paths"], 3) for k, v in st.items() if k not in ("paths", "path_kernel_ms")},
      float(img.mean()))
