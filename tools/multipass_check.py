import sys; sys.path.insert(0, '.')
import torch, numpy as np
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
sc = configs.config2_scene(1024, 1024)
img, st = mf.render_device(sc, 100, 1, max_bounces=16, stats=True)   # 104.9M paths -> 2 passes
print("paths", st["paths"], "mean", float(img.double().mean()), "ms", st["path_kernel_ms"])
img2, _ = mf.render_device(sc, 100, 1, max_bounces=16)
print("deterministic", torch.equal(img, img2))
# tile sharding with ragged tiles through the pool kernel
sc2 = configs.config2_scene(333, 201)
full, _ = mf.render_device(sc2, 8, 3, max_bounces=16, tile=32)
acc = torch.zeros_like(full)
for r in range(3):
    part, _ = mf.render_device(sc2, 8, 3, max_bounces=16, tile=32, rank=r, nranks=3, shard="tiles")
    acc += part
print("tile shards exact", torch.equal(acc, full))
