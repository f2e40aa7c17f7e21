"""Where one GP-oracle ensemble step's time goes: CUPTI kernel / copy time
against the wall clock of the call (torch.profiler)."""
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2603_00280_b200 import gp  # noqa: E402
from paper_2603_00280_b200.rng import RandomStream  # noqa: E402

torch.cuda.set_device(0)
k, cam = bench.gp_workload()
gp.ensemble_radiance(k, cam, bench.GP_ROUNDS, bench.GP_ROUNDS, RandomStream(0, 0))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    gp.ensemble_radiance(k, cam, bench.GP_ROUNDS, bench.GP_ROUNDS, RandomStream(1, 0))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
agg = defaultdict(float)
for e in prof.events():
    if e.device_type.name == "CUDA":
        agg[e.name[:60]] += (e.time_range.end - e.time_range.start) / 1e3
print(f"wall {wall * 1e3:.1f} ms; device busy {sum(agg.values()):.1f} ms")
for name, ms in sorted(agg.items(), key=lambda kv: -kv[1])[:12]:
    print(f"{ms:9.2f} ms  {name}")
