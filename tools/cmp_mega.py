"""Compare the pool kernel's config-2 image with the megakernel's (MF_MEGAKERNEL=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_00280_b200 as mf  # noqa: E402
from paper_2603_00280_b200 import configs  # noqa: E402

sc = configs.config2_scene()
a = mf.render_device(sc, 64, 1, max_bounces=16)[0].cpu().numpy()
os.environ["MF_MEGAKERNEL"] = "1"
b = mf.render_device(sc, 64, 1, max_bounces=16)[0].cpu().numpy()
d = np.abs(a - b)
print("identical" if np.array_equal(a, b) else f"DIFFER: {int((d > 0).sum())} values, max {d.max():.3e}")
