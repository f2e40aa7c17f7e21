import sys, dataclasses
sys.path.insert(0, '.')
import torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
sc = configs.config3_scene(256, 256)
for name, s in (("full", sc), ("no point light", dataclasses.replace(sc, point=None))):
    for _ in range(2):
        img, st = mf.render_device(s, 64, 2, max_bounces=32, stats=True)
    print(name, {k: round(v / st["paths"], 3) for k, v in st.items() if k not in ("paths", "path_kernel_ms")}, "ms", round(st["path_kernel_ms"], 3))
