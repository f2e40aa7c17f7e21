#!/usr/bin/env python
"""Benchmark of the macrofacet hot path on B200 (contract in the task brief).

Headline workload (default, BASELINE.json's metric is quoted on it):
config 4, the variance x correlation sweep -- nine planar GP-surface panels
sigma in {0.01, 0.05, 0.2} x l_z in {0.02, 0.1, inf} (l_xy = 0.05, albedo
0.8, orthographic 45 deg camera, sun at 30 deg), each 1024x1024 pixels x
1024 spp, max depth 64, seed 3.  One step = all nine panels
(9 x 2^30 = 9,663,676,416 paths): per panel one persistent path-pool launch
with the per-pixel sums fused in, one finalize launch; at N > 1 one NCCL
reduce of the nine fp32 panel buffers to rank 0.

Multi-GPU: strong scaling by image tiles -- 32x32 tiles interleaved
t -> rank t mod N, so total work is fixed as N grows and the reduce is exact
(non-owned pixels are +0.0): the image is bit-identical for every N.
`value` = all paths of the step / max-over-ranks device time.

Other workloads (`--workload`, one JSON line each, for the per-config
roofline records in profiles/):
  config1  coefficient queries, N = 2^20 (and a 2^24 kernel-only figure)
  config2  planar render 256^2 x 64 spp, depth 16, seed 1
  config3  sphere + point light 512^2 x 256 spp, depth 32, seed 2
  config5  heterogeneous grid field 2048^2 x 4096 spp, depth 64, seed 4
  gp       the GP-realisation oracle: ensemble_radiance,
           64^2 pixels x 64 realisations

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--workload config4|config1|config2|config3|config5]
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

METRIC = "Mpaths/s (pixel*spp/s)"
QMETRIC = "Mqueries/s"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# workloads (BASELINE.json configs)

def render_workload(name):
    """(description, [scenes], spp, depth, seed, scene labels)."""
    from paper_2603_00280_b200 import configs

    if name == "config4":
        scenes, labels = [], []
        for sig in configs.CONFIG4_SIGMAS:
            for lz in configs.CONFIG4_LZ:
                scenes.append(configs.config4_scene(sig, lz))
                labels.append(f"sigma={sig},l_z={lz}")
        return ("config4: 3x3 panels sigma {0.01,0.05,0.2} x l_z {0.02,0.1,inf}, l_xy 0.05, "
                "1024x1024 x 1024 spp each, depth 64, seed 3 (BASELINE configs[3])",
                scenes, 1024, 64, 3, labels)
    if name == "config2":
        return ("config2: planar GP surface render 256x256 x 64 spp, depth 16, seed 1 "
                "(BASELINE configs[1])", [configs.config2_scene()], 64, 16, 1, ["config2"])
    if name == "config3":
        return ("config3: sphere GP surface + point light 512x512 x 256 spp, depth 32, seed 2 "
                "(BASELINE configs[2])", [configs.config3_scene()], 256, 32, 2, ["config3"])
    if name == "config5":
        return ("config5: heterogeneous GP field (256^3 SDF of 16 spheres + torus, 128^3 "
                "value-noise sigma, l_xy 0.03, l_z 0.08) 2048x2048 x 4096 spp, depth 64, seed 4 "
                "(BASELINE configs[4])", [configs.config5_scene()], 4096, 64, 4, ["config5"])
    raise SystemExit(f"unknown workload {name}")


# ---------------------------------------------------------------------------
# clocks sampler (NVML during the timed region)

class ClockSampler:
    """SM clock and throttle reasons sampled every 5 ms through NVML while
    the timed region runs."""

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
# CPU side: the oracle port of the reference path (process pool)

def cpu_mix(workload, budget_s, steps=1, warmup=0):
    """Time the oracle port on `steps` bounded samples of the workload's
    scene mix (equal paths per scene, like the GPU step).  Returns
    (Mpaths/s, workers, sample description, seconds per step)."""
    from oracle import harness

    desc, scenes, spp, depth, seed, labels = render_workload(workload)
    workers = harness.host_cores()
    jobs, _ = harness.calibrated_mix(scenes, seed, depth, budget_s, workers)
    pool = harness.make_pool(scenes, workers)
    try:
        for _ in range(warmup):
            harness.run_jobs(jobs, pool)
        tot_p, tot_t = 0, 0.0
        for _ in range(steps):
            p, dt = harness.run_jobs(jobs, pool)
            tot_p += p
            tot_t += dt
    finally:
        pool.close()
        pool.join()
    label = f"{len(scenes)} {workload} scene(s) at depth {depth}"
    return tot_p / tot_t / 1e6, workers, harness.describe(jobs, label, workers), tot_t / steps


def cpu_queries(budget_s):
    """The oracle port of the config-1 query batch (extinction, phase_eval,
    pdf, phase sample in float64) over a process pool, on a bounded prefix
    of the 2^20 inputs."""
    import multiprocessing as mp

    from oracle import harness

    global _QIN
    from paper_2603_00280_b200 import configs

    _QIN = configs.config1_inputs()   # generated once, inherited by the forked workers
    workers = harness.host_cores()
    n = 1 << 14
    t0 = time.perf_counter()
    _query_chunk((0, n))
    one = time.perf_counter() - t0
    chunks = max(workers, int(budget_s * workers / max(one, 1e-6)))
    chunks = min(chunks, (1 << 20) // n)
    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        t0 = time.perf_counter()
        pool.map(_query_chunk, [(i * n, (i + 1) * n) for i in range(chunks)], chunksize=1)
        dt = time.perf_counter() - t0
    q = chunks * n
    return q / dt / 1e6, workers, (f"{q} of the 2^20 config-1 queries in {chunks} chunks of {n}, "
                                   "oracle/microfacet.py (float64 restatement of extinction, "
                                   f"phase_eval, pdf, _phase_sample_u) on {workers} processes")


_QIN = None


def _query_chunk(rng):
    from oracle import microfacet as om
    from paper_2603_00280_b200 import configs

    a, b = rng
    p, wo, wi, u = _QIN
    p, wo, wi, u = p[a:b], wo[a:b], wi[a:b], u[a:b]
    med = _oracle_medium(configs.config1_medium())
    wo64, wi64 = wo.astype(np.float64), wi.astype(np.float64)
    om.extinction_local(wo64, p[:, 2].astype(np.float64), med)
    om.phase_eval_local(wo64, wi64, med)
    om.phase_pdf_local(wo64, wi64, med)
    om.phase_sample_local(wo64, med, om.split_two_uniforms(u[:, 0], u[:, 1], med.mix_ratio))
    return b - a


def _oracle_medium(med):
    import __graft_entry__ as g

    return g._oracle_medium(med)


# ---------------------------------------------------------------------------
# reference arm: the oracle port on the host cores

def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    if args.workload == "config5":
        print(json.dumps({"impl": "reference", "unavailable": "config 5 (grid SDF, per-voxel "
                          "sigma) has no reference implementation (SURVEY.md 8(c))"}))
        return 0
    if args.workload == "gp":
        prof = os.path.join(ROOT, "profiles", "r02_gp_reference_cpu.json")
        ref = json.load(open(prof))
        v = ref["paths_per_s"] / 1e6
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": v, "unit": METRIC, "n_gpus": ws,
            "steps": 1, "warmup": 0, "ms_per_step": ref["seconds"] * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "gp (reference gp.ensemble_radiance)",
                                            "sample": ref["sample"]},
            "cpu_baseline": {"value": v, "unit": METRIC, "cores": 1, "kind": "reference",
                             "sample": ref["sample"] + " -- recorded in the build container "
                             "(profiles/r02_gp_reference_cpu.json): the reference package "
                             "cannot travel to the GPU box"},
            "e2e": {"value": v, "unit": METRIC, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}))
        return 0
    if args.workload == "config1":
        v, workers, sample = cpu_queries(args.ref_seconds)
        unit, wl = QMETRIC, "config1: 2^20 coefficient queries (BASELINE configs[0])"
        ms = None
    else:
        v, workers, sample, sec = cpu_mix(args.workload, args.ref_seconds, args.steps,
                                          args.warmup)
        unit, wl = METRIC, render_workload(args.workload)[0]
        ms = sec * 1e3
    line = {"impl": "reference", "metric": unit, "value": v, "unit": unit, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": wl, "sample": sample},
            "cpu_baseline": {"value": v, "unit": unit, "cores": workers, "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# our arm: renders

def measure_peaks(torch, dev):
    from paper_2603_00280_b200 import _lib

    lib = _lib.load()
    f, s = _lib.ctypes.c_double(), _lib.ctypes.c_double()
    _lib.check(lib.mf_measure_peaks(_lib.ctypes.byref(f), _lib.ctypes.byref(s),
                                    _lib.stream_handle(torch, dev)))
    return f.value, s.value


def ncu_traffic(workload):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture of this workload (profiles/), or None."""
    prof = os.path.join(ROOT, "profiles", f"ncu_{workload}.json")
    if not os.path.exists(prof):
        return None
    try:
        with open(prof) as fh:
            return json.load(fh).get("dram_bytes_per_launch")
    except Exception:
        return None


def ncu_memory(workload):
    """Memory-system figures of the dominant kernel from the committed ncu
    summary of this workload (profiles/r02_<workload>_ncu_full.json): DRAM
    and L2 GB/s of that capture -- for config 5, the grid lookups (the SDF
    and sigma grids are L2-resident) -- or None."""
    prof = os.path.join(ROOT, "profiles", f"r02_{workload}_ncu_full.json")
    if not os.path.exists(prof):
        return None
    try:
        with open(prof) as fh:
            d = json.load(fh)
        return {"dram_GB_s": d.get("dram_GB_s"), "l2_GB_s": d.get("l2_GB_s"),
                "l2_hit_pct": d.get("l2_hit_pct"), "capture": d.get("source"),
                "units_per_launch": d.get("units_per_launch"),
                # what the kernel actually issued in that capture (ncu pipe
                # counters), next to the algorithmic figure above
                "ncu_issue": {"issue_active_pct": d.get("issue_active_pct"),
                              "active_lanes": d.get("active_lanes"),
                              "pipe_fma_pct": d.get("pipe_fma_pct"),
                              "pipe_alu_pct": d.get("pipe_alu_pct"),
                              "pipe_xu_pct": d.get("pipe_xu_pct"),
                              "thread_instructions_per_unit":
                                  d.get("thread_instructions_per_unit"),
                              "fp32_share_of_instructions":
                                  d.get("fp32_share_of_instructions")}}
    except Exception:
        return None


def run_render(args, torch, dist, n, rank, local, dev):
    import paper_2603_00280_b200 as mf
    from paper_2603_00280_b200 import _lib, roofline
    from paper_2603_00280_b200.scene import to_c_scene

    desc, scenes, spp, depth, seed, labels = render_workload(args.workload)
    lib = _lib.load()
    cam = scenes[0].camera
    P = len(scenes)
    cs = [to_c_scene(s) for s in scenes]
    out = torch.empty((P, cam.height, cam.width, 3), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    paths_per_step = P * cam.width * cam.height * spp

    def step():
        # every panel queued on the stream (mf_render_async): no host
        # synchronisation inside a step; the tickets are finished -- and
        # validated -- while the next step runs
        tickets = [mf.render_device(scenes[i], spp, seed, max_bounces=depth, tile=32, rank=rank,
                                    nranks=n, shard="tiles", out=out[i], c_scene=cs[i],
                                    wait=False) for i in range(P)]
        if n > 1:
            dist.reduce(out, dst=0, op=dist.ReduceOp.SUM)   # the one collective of the step
        return tickets

    def finish(tickets, stats_acc=None):
        for i, t in enumerate(tickets):
            st = t.finish()
            if stats_acc is not None:
                stats_acc[i].append(st)

    for _ in range(max(args.warmup, 0)):
        finish(step())
    torch.cuda.synchronize()
    if n > 1:
        dist.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    acc = [[] for _ in range(P)]
    l0 = lib.mf_launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        pending = None
        for i in range(args.steps):
            flush.fill_(float(i))          # evict L2 between steps (256 MiB > 126 MB L2)
            starts[i].record()
            tickets = step()
            ends[i].record()
            if pending is not None:
                finish(pending, acc)
            pending = tickets
        finish(pending, acc)
        torch.cuda.synchronize()
        if n > 1:
            dist.barrier()
    launches = lib.mf_launch_count() - l0
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if n > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = paths_per_step * args.steps / (ms_max * 1e-3) / 1e6

    # e2e through the public API: render() per scene (host float64 image,
    # validated) at N = 1; render_sharded() + host copy on rank 0 at N > 1
    e2e_steps = max(1, min(args.steps, 5))

    def e2e_step():
        for s in scenes:
            if n == 1:
                mf.render(s, spp, seed, max_bounces=depth)
            else:
                img, _ = mf.render_sharded(s, spp, seed, max_bounces=depth, shard="tiles")
                if rank == 0:
                    img.cpu()
                torch.cuda.synchronize()

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
    e2e_value = paths_per_step * e2e_steps / float(e2e_t.item()) / 1e6

    if rank != 0:
        return None
    # roofline of the dominant kernel from the TIMED steps: algorithmic ops
    # from the device event counters of those launches over their CUDA-event
    # time (measured inside mf_render on the launching stream)
    pf, ps_ = measure_peaks(torch, dev)
    F = S = 0.0
    kms = 0.0
    tot = {}
    for i in range(P):
        planar = scenes[i].primitives[0].sdf.__class__.__name__ == "Plane" and \
            len(scenes[i].primitives) == 1
        for st in acc[i]:
            f, s = roofline.algorithmic_ops(st, planar=planar,
                                            kind=getattr(scenes[i].primitives[0].medium, "kind",
                                                         None))
            F += f
            S += s
            kms += st["path_kernel_ms"]
            for k, v in st.items():
                tot[k] = tot.get(k, 0) + v
    rl = roofline.from_ops(F, S, kms, pf, ps_, tot.get("paths", 1))
    kernel = {"config4": "pool_kernel (single-plane path pool, grey)",
              "config2": "pool_kernel (single-plane path pool, grey)",
              "config3": "curved_pool_kernel<3> (single-sphere path pool, grey)",
              "config5": "grid_pool_kernel (grid-field path pool with pooled walks, grey)"}[args.workload]
    roof = {"bound": rl["bound"], "achieved": rl["achieved"], "peak": rl["peak"],
            "unit": rl["unit"], "frac": rl["frac"], "traffic": ncu_traffic(args.workload),
            "peak_source": "measured on this device by mf_measure_peaks (FFMA / MUFU.EX2 issue "
                           "microbenchmarks, all SMs)",
            "fp32_frac": rl["fp32_frac"], "sfu_frac": rl["sfu_frac"],
            "fp32_per_path": rl["fp32_per_path"], "sfu_per_path": rl["sfu_per_path"],
            "kernel_ms_per_step": kms / args.steps,
            "kernel_ms_per_scene": [sum(st["path_kernel_ms"] for st in a) / args.steps
                                    for a in acc],
            "kernel_share_of_step": kms / max(ms, 1e-9),
            "kernel": kernel,
            "memory": ncu_memory(args.workload),
            "work": "algorithmic FP32 / MUFU lane ops from the frozen per-event counts "
                    "(paper_2603_00280_b200/roofline.py) x the device event counters of the "
                    "timed launches"}
    cpu = None
    if n == 1 and not args.no_cpu and args.workload != "config5":
        v, workers, sample, _ = cpu_mix(args.workload, args.cpu_seconds)
        cpu = {"value": v, "unit": METRIC, "cores": workers, "kind": "port", "sample": sample}
    elif args.workload == "config5":
        cpu = {"value": None, "unit": METRIC, "cores": 0, "kind": "port",
               "sample": "none: config 5 (grid SDF, per-voxel sigma) has no reference "
                         "implementation to port (SURVEY.md 8(c))"}
    h2d = P * (_lib.ctypes.sizeof(_lib.MfScene) + _lib.ctypes.sizeof(_lib.MfRenderParams))
    return {
        "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": desc, "paths_per_step": paths_per_step, "panels": labels,
                   "shard": "32x32 image tiles interleaved over ranks (strong scaling)",
                   "l2": "flushed between steps (256 MiB device write)",
                   "parallelism": (f"{n} GPUs, one NCCL reduce of the {P} fp32 panel buffers per "
                                   "step") if n > 1 else "1 GPU"},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": METRIC, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": P * cam.width * cam.height * 3 * 8,   # float64 images
                "api": "paper_2603_00280_b200.render() per scene" if n == 1
                else "render_sharded() per scene + rank-0 host copy"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "stats_per_path": {k: v / max(tot.get("paths", 1), 1) for k, v in tot.items()
                           if k not in ("paths", "path_kernel_ms")},
    }


# ---------------------------------------------------------------------------
# our arm: config-1 coefficient queries

def run_queries(args, torch, n, rank, local, dev):
    import paper_2603_00280_b200 as mf
    from paper_2603_00280_b200 import _lib, configs, roofline

    lib = _lib.load()
    med = configs.config1_medium()
    p, wo, wi, u = configs.config1_inputs()
    N = p.shape[0]
    # this rank's slice (no collective: queries are independent)
    a, b = N * rank // n, N * (rank + 1) // n
    host = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in
            (("p", p[a:b].T), ("wo", wo[a:b].T), ("wi", wi[a:b].T), ("u1", u[a:b, 0]),
             ("u2", u[a:b, 1]))}
    d = {k: v.to(dev) for k, v in host.items()}
    outs = {k: torch.empty(b - a, dtype=torch.int32 if k == "flags" else torch.float32,
                           device=dev) for k in mf.medium._QUERY_DEFAULT}
    host_out = {k: torch.empty_like(v, device="cpu").pin_memory() for k, v in outs.items()}

    def call(dd, oo):
        mf.query_batch(med, dd["p"], dd["wo"], dd["wi"], dd["u1"], dd["u2"], out=oo)

    reps = 50
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(max(args.warmup, 1)):
        call(d, outs)
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    l0 = lib.mf_launch_count()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            starts[i].record()
            for _ in range(reps):     # back to back: the queue stays ahead of the host
                call(d, outs)
            ends[i].record()
        torch.cuda.synchronize()
    launches = lib.mf_launch_count() - l0
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / (args.steps * reps)
    value = (b - a) * n / (ms * 1e-3) / 1e6
    # 2^24 (16 copies of the inputs): the kernel at a size that fills the GPU
    big = {k: v.repeat(1, 16).contiguous() if v.dim() == 2 else v.repeat(16) for k, v in d.items()}
    bouts = {k: v.repeat(16) for k, v in outs.items()}
    call(big, bouts)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(10):
        call(big, bouts)
    s1.record()
    torch.cuda.synchronize()
    ms24 = s0.elapsed_time(s1) / 10
    # e2e: pinned host inputs -> device -> kernel -> host outputs, every
    # step, through the public query_batch_host (copies of one chunk
    # overlapping the kernel and the copies of the others)
    e2e_steps = max(3, args.steps)

    def e2e_call():
        mf.query_batch_host(med, host["p"], host["wo"], host["wi"], host["u1"], host["u2"],
                            out=host_out)

    e2e_call()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if rank != 0:
        return None
    pf, ps_ = measure_peaks(torch, dev)
    rl = roofline.query_roofline(b - a, ms, pf, ps_)
    rl24 = roofline.query_roofline((b - a) * 16, ms24, pf, ps_)
    bytes_q = roofline.QUERY_BYTES
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs") \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else None
    cpu = None
    if n == 1 and not args.no_cpu:
        v, workers, sample = cpu_queries(args.cpu_seconds)
        cpu = {"value": v, "unit": QMETRIC, "cores": workers, "kind": "port", "sample": sample}
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    d2h = sum(v.numel() * v.element_size() for v in host_out.values())
    return {
        "metric": QMETRIC, "value": value, "unit": QMETRIC, "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "config1: 2^20 coefficient queries (sigma_t, phase value + pdf, "
                               "one phase sample; GENERALIZED sigma 0.05, l 0.1), seed 0 "
                               "(BASELINE configs[0])",
                   "timing": f"{reps} back-to-back launches per step between CUDA events",
                   "l2": "flushed between steps (256 MiB device write)"},
        "roofline": {"bound": rl["bound"], "achieved": rl["frac"] * (pf if rl["bound"] == "fp32"
                                                                     else ps_),
                     "peak": pf if rl["bound"] == "fp32" else ps_, "unit": "Ginst/s",
                     "frac": rl["frac"], "fp32_frac": rl["fp32_frac"], "sfu_frac": rl["sfu_frac"],
                     "traffic": ncu_traffic("config1"), "kernel": "query_kernel",
                     "kernel_ms": ms,
                     "hbm_GB_s": (b - a) * bytes_q / (ms * 1e-3) / 1e9,
                     "hbm_frac": ((b - a) * bytes_q / (ms * 1e-3) / 1e9 / hbm) if hbm else None,
                     "at_2^24": {"kernel_ms": ms24, "frac": rl24["frac"],
                                 "Mqueries_s": (b - a) * 16 / (ms24 * 1e-3) / 1e6,
                                 "hbm_GB_s": (b - a) * 16 * bytes_q / (ms24 * 1e-3) / 1e9}},
        "cpu_baseline": cpu,
        "e2e": {"value": (b - a) * n / e2e_s / 1e6, "unit": QMETRIC, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "api": "paper_2603_00280_b200.query_batch_host() (pinned host in / out, "
                       "chunks pipelined over three streams)"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }


# ---------------------------------------------------------------------------
# our arm: the GP-realisation oracle

GP_W = GP_H = 64          # the reference's desk-scale maximum
GP_ROUNDS = 64            # realisations (sample rounds) per step


def gp_workload():
    from paper_2603_00280_b200.ndf import KernelParams
    from paper_2603_00280_b200.scene import Camera

    sigma = ell = 0.05
    k = KernelParams(sigma, ell, ell, ell)
    cam = Camera(position=(0, 0, 8 * sigma + 2), look_at=(1.0, 0, 0), fov_deg=35, width=GP_W,
                 height=GP_H)
    return k, cam


def run_gp(args, torch, n, rank, local, dev):
    """ensemble_radiance (gp.py:334-398) of GP_ROUNDS realisations at the
    reference's 64 x 64 desk-scale limit, kernel sigma 0.05, l 0.05, the CLI
    gp-ensemble camera, F = 1, depth 64.  value: paths of the step over the
    device time of its realisation + bounce-loop work (CUDA events);
    e2e: the public ensemble_radiance() call (host camera rays, uniforms
    read-back, image download)."""
    from paper_2603_00280_b200 import _lib, gp
    from paper_2603_00280_b200.rng import RandomStream

    k, cam = gp_workload()
    lib = _lib.load()
    paths = GP_W * GP_H * GP_ROUNDS
    for _ in range(max(args.warmup, 1)):
        gp.ensemble_radiance(k, cam, GP_ROUNDS, GP_ROUNDS, RandomStream(0, 0))
    torch.cuda.synchronize()
    work = {}
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    l0 = lib.mf_launch_count()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        for i in range(args.steps):
            starts[i].record()
            gp.ensemble_radiance(k, cam, GP_ROUNDS, GP_ROUNDS, RandomStream(i, 0), work=work)
            ends[i].record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / args.steps
    launches = lib.mf_launch_count() - l0
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / args.steps
    if rank != 0:
        return None
    peak = _lib.ctypes.c_double()
    _lib.check(lib.mf_measure_peak_fp64(_lib.ctypes.byref(peak), _lib.stream_handle(torch, dev)))
    # algorithmic work: 45 float64 operations per evaluation of the trilinear
    # interpolant (3 sub + 3 div + 3 sub + 3 one-minus + 8 x (2 mul weight +
    # mul + add) + the planar mean) and 6 per ray point of the march
    # (csrc/mf_gp.cuh); FMA-free by construction (numpy's rounding)
    evals = work.get("evals", 0) / args.steps
    ops = evals * 51.0
    achieved = ops / (ms * 1e-3) / 1e9
    ref = None
    prof = os.path.join(ROOT, "profiles", "r02_gp_reference_cpu.json")
    if os.path.exists(prof):
        ref = json.load(open(prof))
    cpu = {"value": ref["paths_per_s"] / 1e6, "unit": METRIC, "cores": 1, "kind": "reference",
           "sample": ref["sample"] + "; " + ref["what"] + " (timed in the build container: "
           "the reference cannot travel to the GPU box)"} if ref else None
    return {
        "metric": METRIC, "value": paths / (ms * 1e-3) / 1e6, "unit": METRIC, "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"gp: GP-realisation oracle ensemble_radiance, {GP_W}x{GP_H} "
                               f"pixels x {GP_ROUNDS} realisations, sigma 0.05, l 0.05, depth 64 "
                               "(SURVEY.md 8(f) rank 4, reference gp.py:334-398)",
                   "paths_per_step": paths, "evaluations_per_step": evals,
                   "timing": "CUDA events around each public call (host work inside)"},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak.value,
                     "unit": "Ginst/s", "frac": achieved / peak.value, "traffic": None,
                     "peak_source": "measured on this device by mf_measure_peak_fp64 (DFMA "
                                    "issue microbenchmark, all SMs)",
                     "kernel": "gp::reflect_kernel (march + bisection + bounce)",
                     "work": "51 float64 ops per interpolant evaluation x the device's "
                             "evaluation counter"},
        "cpu_baseline": cpu,
        "e2e": {"value": paths / wall / 1e6, "unit": METRIC, "h2d_bytes_per_step": paths * 48,
                "d2h_bytes_per_step": paths * 24,
                "api": "paper_2603_00280_b200.gp.ensemble_radiance()"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }


def run_ours(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    if ws != args.gpus and ws > 1:
        print(f"warning: WORLD_SIZE={ws} but --gpus {args.gpus}", file=sys.stderr)
    n = ws
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if n > 1:
        if rank == 0:
            # communicator lines (rank count, transport) to stderr, so the
            # N-rank run is checkable without disturbing the JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=dev)
        chk = torch.ones(1, device=dev)
        dist.all_reduce(chk)
        if rank == 0:
            print(f"nccl communicator: world_size={dist.get_world_size()} "
                  f"all_reduce(ones)={int(chk.item())} nccl={torch.cuda.nccl.version()}",
                  file=sys.stderr)
    if args.workload == "config1":
        result = run_queries(args, torch, n, rank, local, dev)
    elif args.workload == "gp":
        result = run_gp(args, torch, n, rank, local, dev)
    else:
        result = run_render(args, torch, dist, n, rank, local, dev)
    if result is not None:
        if n > 1:
            result["comm"] = {"backend": "nccl", "world_size": n,
                              "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))}
        print(json.dumps(result))
    if n > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default="config4",
                    choices=("config4", "config1", "config2", "config3", "config5", "gp"))
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=4.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "ours":
        args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
