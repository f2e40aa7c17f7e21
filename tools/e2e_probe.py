"""Host-side cost of render() variants on config 2 (GPU box)."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_00280_b200 as mf  # noqa: E402
from paper_2603_00280_b200 import configs, _lib  # noqa: E402
from paper_2603_00280_b200.image import RadianceImage  # noqa: E402
from paper_2603_00280_b200.render import render_device  # noqa: E402

scene = configs.config2_scene()


def cur():
    return mf.render(scene, 64, 1, max_bounces=16)


def pinned():
    img, _ = render_device(scene, 64, 1, max_bounces=16, stats=True)
    d64 = img.to(torch.float64)
    h = torch.empty(d64.shape, dtype=torch.float64, pin_memory=True)
    h.copy_(d64, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return RadianceImage(pixels=h.numpy(), meta={})


def dev_only():
    img, _ = render_device(scene, 64, 1, max_bounces=16, stats=True)
    return img


def dev_nostats():
    img, _ = render_device(scene, 64, 1, max_bounces=16, stats=False)
    torch.cuda.synchronize()
    return img


for fn in (cur, pinned, dev_only, dev_nostats, cur, pinned, dev_only, dev_nostats):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(30):
        fn()
    torch.cuda.synchronize()
    print(fn.__name__, round((time.perf_counter() - t) / 30 * 1e3, 4), "ms")
