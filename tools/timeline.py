"""Stream timeline of a few pipelined config-2 renders (torch.profiler /
CUPTI): kernels, memsets and copies with their gaps -- where a render's
fixed cost goes.   python tools/timeline.py [workload]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2603_00280_b200 as mf  # noqa: E402
from paper_2603_00280_b200 import configs  # noqa: E402

torch.cuda.set_device(0)
sc = configs.config2_scene()
out = torch.empty((256, 256, 3), device="cuda")
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for _ in range(3):
    mf.render_device(sc, 64, 1, max_bounces=16, out=out, wait=False).finish()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    pend = None
    for i in range(4):
        flush.fill_(float(i))
        t = mf.render_device(sc, 64, 1, max_bounces=16, out=out, wait=False)
        if pend is not None:
            pend.finish()
        pend = t
    pend.finish()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev = None
for e in ev:
    s, d = e.time_range.start - t0, e.time_range.end - e.time_range.start
    gap = (e.time_range.start - prev) if prev is not None else 0
    print(f"{s:10.1f} us  +gap {gap:7.1f}  dur {d:8.1f}  {e.name[:70]}")
    prev = e.time_range.end
