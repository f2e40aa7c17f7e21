import os, sys, dataclasses
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
torch.cuda.set_device(0)
base = configs.config2_scene(96, 64)
for I in [(4.0,4.0,4.0),(4.0,3.0,2.0)]:
    scene = dataclasses.replace(base, point=mf.PointLight(position=(0.3, 0.2, 2.0), intensity=I))
    os.environ.pop("MF_MEGAKERNEL", None)
    a, sa = mf.render_device(scene, 16, 9, max_bounces=16, stats=True); a = a.cpu().numpy()
    a2, _ = mf.render_device(scene, 16, 9, max_bounces=16, stats=True); a2 = a2.cpu().numpy()
    os.environ["MF_MEGAKERNEL"] = "1"
    b, sb = mf.render_device(scene, 16, 9, max_bounces=16, stats=True); b = b.cpu().numpy()
    d = a != b
    print(I, "pool repeat equal", np.array_equal(a, a2), "differing pixels", d.any(-1).sum(), "max abs", np.abs(a-b).max(), sa["paths"], sb["paths"])
    sa.pop("path_kernel_ms"); sb.pop("path_kernel_ms"); print({k:(sa[k],sb[k]) for k in sa if sa[k]!=sb[k]})
