"""Diagnostic: config-3 image at 128^2 (GPU) saved for comparison with the
oracle fixture tests/golden/config3_ref128.npz."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_00280_b200 as mf  # noqa: E402
from paper_2603_00280_b200 import configs  # noqa: E402

torch.cuda.set_device(0)
out = {}
for seed in (2, 3):
    img, st = mf.render_device(configs.config3_scene(128, 128), 8192, seed, max_bounces=32,
                               stats=True)
    out[f"s{seed}"] = img.cpu().numpy()
    print(st)
if os.environ.get("MF_NO_SHADOW_RR"):
    pass
np.savez_compressed("gpurun_out/c3_gpu128.npz", **out)
