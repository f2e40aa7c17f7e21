"""Host-side time of one render() call (config 2) by component."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
torch.cuda.set_device(0)
sc = configs.config2_scene()
for _ in range(5): mf.render(sc, 64, 1, max_bounces=16)
torch.cuda.synchronize()
N = 50
t0 = time.perf_counter()
for _ in range(N): mf.render(sc, 64, 1, max_bounces=16)
t_full = (time.perf_counter() - t0) / N
out = torch.empty((256, 256, 3), device="cuda")
t0 = time.perf_counter()
for _ in range(N):
    mf.render_device(sc, 64, 1, max_bounces=16, out=out)
torch.cuda.synchronize()
t_dev_async = (time.perf_counter() - t0) / N
t0 = time.perf_counter()
for _ in range(N):
    mf.render_device(sc, 64, 1, max_bounces=16, out=out, stats=True)
t_dev_stats = (time.perf_counter() - t0) / N
t0 = time.perf_counter()
for _ in range(N):
    mf.render_device(sc, 64, 1, max_bounces=16, out=out)
    torch.cuda.synchronize()
t_dev_sync = (time.perf_counter() - t0) / N
host = torch.empty((256, 256, 3), dtype=torch.float64, pin_memory=True)
t0 = time.perf_counter()
for _ in range(N):
    d64 = out.to(torch.float64); host.copy_(d64, non_blocking=True); torch.cuda.synchronize()
t_copy = (time.perf_counter() - t0) / N
print({k: round(v * 1e3, 4) for k, v in dict(render=t_full, device_async=t_dev_async,
       device_stats_sync=t_dev_stats, device_sync=t_dev_sync, to64_d2h=t_copy).items()})
import numpy as np
h32 = torch.empty((256, 256, 3), dtype=torch.float32, pin_memory=True)
t0 = time.perf_counter()
for _ in range(N):
    h32.copy_(out, non_blocking=True); torch.cuda.synchronize(); x = h32.numpy().astype(np.float64)
t_b = (time.perf_counter() - t0) / N
print({"d2h32_astype64": round(t_b * 1e3, 4)})
