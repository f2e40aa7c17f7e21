#!/usr/bin/env python
"""Benchmark of the macrofacet hot path on B200 (contract in the task brief).

Workload (BASELINE.json configs[1], "config 2"): planar GP surface render,
256x256 pixels x 64 spp, depth 16, albedo 0.8, orthographic 45 deg camera,
sun at 30 deg, black environment, seed 1 -- one step = one full render
(4,194,304 paths) through the persistent path megakernel + per-pixel
accumulation (+ one NCCL reduce of the fp32 image when N > 1).

Multi-GPU: weak scaling by sample-range sharding -- every rank renders the
whole image for its own 64-sample range (samples [64r, 64r+64) of a
64N-spp render) and the fp32 buffers are summed by one NCCL reduce to
rank 0.  `value` = all ranks' paths / max-over-ranks device time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "config2: planar GP surface render 256x256 x 64 spp, depth 16 (BASELINE configs[1])"
METRIC = "Mpaths/s (pixel*spp/s)"
PATHS_PER_RANK = 256 * 256 * 64


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class ClockSampler:
    """SM clock and throttle reasons sampled every 5 ms through NVML while
    the timed region runs (nvidia-smi fallback)."""

    # NVML clocks-event-reason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_r = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self._stop.is_set():
                self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                     int(get_r(h))))
                self._stop.wait(0.005)
        except Exception as exc:  # pragma: no cover - diagnostic only
            self.samples.append((None, 0))
            print(f"clock sampler: {exc}", file=sys.stderr)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.05)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        sm = [s[0] for s in self.samples if s[0] is not None]
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"],
                    "samples": 0}
        reasons = sorted({name for _, bits in self.samples for name, b in self.BITS.items()
                          if bits & b})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(sm), "source": "nvml"}


# ---------------------------------------------------------------------------
# CPU baseline (oracle port of the reference path, process pool)

def cpu_baseline(seconds=15.0, workers=None):
    from oracle import harness
    from paper_2603_00280_b200 import configs

    scene = configs.config2_scene()
    workers = workers or harness.host_cores()
    pool = harness.make_pool(scene, workers)
    try:
        tile = 32 if workers <= 64 else 16
        spp, n_tiles, rate1 = harness.calibrated_sample(scene, 16, 1, seconds, workers, tile, pool)
        paths, dt = harness.timed_render(scene, spp, 1, 16, n_tiles, workers, tile, pool)
    finally:
        pool.close()
        pool.join()
    return {"value": paths / dt / 1e6, "unit": METRIC, "cores": workers, "kind": "port",
            "sample": f"{n_tiles} tiles of {tile}x{tile} px x {spp} spp of config 2 "
                      f"({paths} paths, {dt:.1f} s), oracle/tracer.py (float64 numpy restatement "
                      "of the reference walk/trace_paths, identical RNG consumption) on "
                      f"{workers} processes"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import harness
    from paper_2603_00280_b200 import configs

    scene = configs.config2_scene()
    workers = harness.host_cores()
    tile = 32 if workers <= 64 else 16
    pool = harness.make_pool(scene, workers)
    try:
        spp, n_tiles, _ = harness.calibrated_sample(scene, 16, 1, args.ref_seconds, workers, tile,
                                                    pool)
        for _ in range(args.warmup):
            harness.timed_render(scene, spp, 1, 16, n_tiles, workers, tile, pool)
        tot_paths = 0
        tot_t = 0.0
        for _ in range(args.steps):
            p, dt = harness.timed_render(scene, spp, 1, 16, n_tiles, workers, tile, pool)
            tot_paths += p
            tot_t += dt
    finally:
        pool.close()
        pool.join()
    v = tot_paths / tot_t / 1e6
    sample = (f"per step {n_tiles} tiles of {tile}x{tile} px x {spp} spp of config 2, "
              "oracle/tracer.py (float64 numpy restatement of the reference render path) on "
              f"{workers} processes")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": METRIC, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot_t / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "sample": sample},
            "cpu_baseline": {"value": v, "unit": METRIC, "cores": workers, "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# our arm

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2603_00280_b200 as mf
    from paper_2603_00280_b200 import _lib, configs, roofline
    from paper_2603_00280_b200.scene import to_c_scene

    ws, rank, local = dist_env()
    if ws != args.gpus and ws > 1:
        print(f"warning: WORLD_SIZE={ws} but --gpus {args.gpus}", file=sys.stderr)
    n = ws
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if n > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load()
    scene = configs.config2_scene()
    cs = to_c_scene(scene)
    spp_total = 64 * n
    shard = "samples"
    out = torch.empty((256, 256, 3), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        mf.render_device(scene, spp_total, 1, max_bounces=16, rank=rank, nranks=n, shard=shard,
                         out=out, c_scene=cs)
        if n > 1:
            dist.reduce(out, dst=0, op=dist.ReduceOp.SUM)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    if n > 1:
        dist.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    l0 = lib.mf_launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.fill_(float(i))          # evict L2 between steps (256 MiB > 126 MB L2)
            starts[i].record()
            step()
            ends[i].record()
        torch.cuda.synchronize()
        if n > 1:
            dist.barrier()
    launches = lib.mf_launch_count() - l0
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if n > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = n * PATHS_PER_RANK * args.steps / (ms_max * 1e-3) / 1e6

    # e2e through the public API: render() (host image, float64, validated)
    # at N=1; render_sharded() + host copy at N>1
    torch.cuda.synchronize()
    if n > 1:
        dist.barrier()
    e2e_steps = max(1, min(args.steps, 10))

    def e2e_step():
        if n == 1:
            mf.render(scene, 64, 1, max_bounces=16)
        else:
            img, _ = mf.render_sharded(scene, spp_total, 1, max_bounces=16, shard=shard)
            if rank == 0:
                img.cpu()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    if n > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if n > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = n * PATHS_PER_RANK * e2e_steps / float(e2e_t.item()) / 1e6

    result = None
    if rank == 0:
        # roofline of the dominant kernel (path megakernel), live CUDA events
        fpk = _lib.ctypes.c_double()
        spk = _lib.ctypes.c_double()
        _lib.check(lib.mf_measure_peaks(_lib.ctypes.byref(fpk), _lib.ctypes.byref(spk),
                                        _lib.stream_handle(torch, dev)))
        _, st = mf.render_device(scene, spp_total, 1, max_bounces=16, rank=0, nranks=n,
                                 shard=shard, out=out, stats=True, c_scene=cs)
        rl = roofline.roofline(st, st["path_kernel_ms"], fpk.value, spk.value, planar=True)
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_path_kernel.json")
        if os.path.exists(prof):
            try:
                with open(prof) as fh:
                    traffic = json.load(fh).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        roof = {"bound": rl["bound"], "achieved": rl["achieved"], "peak": rl["peak"],
                "unit": rl["unit"], "frac": rl["frac"], "traffic": traffic,
                "peak_source": "measured on this device by mf_measure_peaks (FFMA / MUFU.EX2 "
                               "issue microbenchmarks)",
                "fp32_frac": rl["fp32_frac"], "sfu_frac": rl["sfu_frac"],
                "fp32_per_path": rl["fp32_per_path"], "sfu_per_path": rl["sfu_per_path"],
                "kernel_ms": st["path_kernel_ms"], "kernel": "pool_kernel (single-plane path pool)"}
        cpu = None
        if n == 1 and not args.no_cpu:
            cpu = cpu_baseline(args.cpu_seconds)
        result = {
            "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "global_paths_per_step": n * PATHS_PER_RANK,
                       "spp_per_rank": 64, "shard": "samples (weak scaling)",
                       "l2": "flushed between steps (256 MiB device write)",
                       "parallelism": f"{n} GPU(s), one NCCL reduce per step" if n > 1 else "1 GPU"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": METRIC,
                    "h2d_bytes_per_step": _lib.ctypes.sizeof(_lib.MfScene)
                    + _lib.ctypes.sizeof(_lib.MfRenderParams),
                    "d2h_bytes_per_step": 256 * 256 * 3 * 8,   # float64 image
                    "api": "paper_2603_00280_b200.render()" if n == 1 else "render_sharded()"},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "stats_per_path": {k: v / max(st["paths"], 1) for k, v in st.items()
                               if k not in ("paths", "path_kernel_ms")},
        }
        print(json.dumps(result))
    if n > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=4.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
