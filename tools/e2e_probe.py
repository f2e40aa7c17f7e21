"""Host-side breakdown of one render() call on config 2 (GPU box)."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_00280_b200 as mf  # noqa: E402
from paper_2603_00280_b200 import configs  # noqa: E402

scene = configs.config2_scene()
for _ in range(3):
    mf.render(scene, 64, 1, max_bounces=16)
T = {}


def tick(k, t0):
    T[k] = T.get(k, 0.0) + (time.perf_counter() - t0) * 1e3
    return time.perf_counter()


N = 20
for _ in range(N):
    torch.cuda.synchronize()
    t = time.perf_counter()
    img, st = mf.render_device(scene, 64, 1, max_bounces=16, stats=True)
    t = tick("render_device(stats)", t)
    flags = torch.stack(((~torch.isfinite(img)).any(), (img < 0.0).any()))
    t = tick("flags (async)", t)
    pixels = img.to(torch.float64).cpu().numpy()
    t = tick("double+d2h", t)
    f = flags.cpu().numpy()
    t = tick("flags d2h", t)
    out = mf.RadianceImage(pixels=pixels, meta={})
    t = tick("RadianceImage", t)
    torch.cuda.synchronize()
    t = time.perf_counter()
    mf.render(scene, 64, 1, max_bounces=16)
    t = tick("render() total", t)
print({k: round(v / N, 3) for k, v in T.items()})
