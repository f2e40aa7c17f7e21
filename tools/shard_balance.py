"""Strong-scaling load balance of the headline step on ONE GPU: the nine
config-4 panels (1024^2 x 1024 spp, depth 64, seed 3) are rendered share by
share -- rank r of N = 1, 2, 4, 8 with the bench's interleaved 32x32 tile
sharding, one rank's launches at a time (no rank waits on another) -- and
the step time an N-GPU run would see is the SLOWEST share (the NCCL reduce
of 9 x 12 MiB over NVLink adds ~0.2 ms).  Prints one JSON object:
  python tools/shard_balance.py [--spp 1024] > profiles/r02_shard_balance.json
This bounds the scaling curve from above; the N-GPU run itself is the
driver's (SCALE_rNN.json)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_00280_b200 as mf                      # noqa: E402
from paper_2603_00280_b200 import configs               # noqa: E402


def share_ms(scenes, spp, rank, nranks, outs):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    tickets = [mf.render_device(sc, spp, 3, max_bounces=64, tile=32, rank=rank, nranks=nranks,
                                out=o, wait=False) for sc, o in zip(scenes, outs)]
    b.record()
    for t in tickets:
        t.finish()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--spp", type=int, default=1024)
    ap.add_argument("--size", type=int, default=1024)
    args = ap.parse_args()
    scenes = [configs.config4_scene(s, lz, args.size, args.size)
              for s in configs.CONFIG4_SIGMAS for lz in configs.CONFIG4_LZ]
    outs = [torch.empty((args.size, args.size, 3), dtype=torch.float32, device="cuda")
            for _ in scenes]
    for _ in range(2):                                   # warm-up (tables, clocks)
        share_ms(scenes, max(args.spp // 8, 1), 0, 1, outs)
    res = {"workload": f"config4 nine panels {args.size}^2 x {args.spp} spp, depth 64, seed 3",
           "shard": "32x32 tiles interleaved over ranks", "device": torch.cuda.get_device_name(0),
           "n": {}}
    t1 = None
    for n in (1, 2, 4, 8):
        ms = [min(share_ms(scenes, args.spp, r, n, outs) for _ in range(2)) for r in range(n)]
        if n == 1:
            t1 = ms[0]
        res["n"][str(n)] = {"share_ms": [round(m, 3) for m in ms], "slowest_ms": round(max(ms), 3),
                            "speedup_bound": round(t1 / max(ms), 3),
                            "efficiency_bound": round(t1 / max(ms) / n, 4)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
