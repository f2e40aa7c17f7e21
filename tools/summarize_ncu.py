"""Summarise ncu captures into profiles/ (tracked).

    python tools/summarize_ncu.py <round_tag> <workload> <full.ncu-rep> [launches.csv]

Writes profiles/<tag>_<workload>_ncu_full.json (key metrics of the captured
kernel: DRAM / L2 bytes per launch, pipe utilisation, active lanes),
profiles/<tag>_<workload>_launches.json (per-kernel share of the step from
the gpu__time_duration launch list) and refreshes
profiles/ncu_<workload>.json (read by bench.py for roofline.traffic)."""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__inst_executed.sum", "smsp__thread_inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed_pipe_fma.sum", "smsp__inst_executed_pipe_xu.sum",
    "smsp__inst_executed_pipe_alu.sum",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "smsp__warp_issue_stalled_no_instruction_per_warp_active.pct",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6,
             "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = {"kernel": d.get("Kernel Name", "")}
        for m in METRICS:
            if m not in d:
                continue
            v = to_num(d[m])
            u = units.get(m, "")
            if isinstance(v, float) and u in scale:
                v *= scale[u]
                m = m + (" [ms]" if "second" in u else " [bytes]")
            k[m] = v
        res.append(k)
    return res


def to_num(v):
    try:
        return float(str(v).replace(",", ""))
    except (TypeError, ValueError):
        return v


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, mn = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = {}
    for r in rows[1:]:
        if r[mn] != "gpu__time_duration.sum":
            continue
        k = r[ki].split("(")[0]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += to_num(r[mi])
    tot = sum(a[1] for a in agg.values())
    # the render step proper: our kernels minus the one-off peak
    # microbenchmarks (roofline denominators) and torch's L2-flush fills
    step = {k: a for k, a in agg.items() if not k.startswith("at::") and "peak_" not in k
            and "slope_table" not in k}
    st = sum(a[1] for a in step.values()) or 1.0
    return {k: {"launches": a[0], "total_ns": a[1], "mean_ns": a[1] / a[0], "share": a[1] / tot,
                "step_share": (a[1] / st) if k in step else None}
            for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])}


def main():
    tag, wl, rep = sys.argv[1], sys.argv[2], sys.argv[3]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    kernels = raw_metrics(rep)
    summ = []
    for k in kernels:
        d = {m: to_num(v) for m, v in k.items()}
        if d.get("dram__bytes_read.sum [bytes]") is not None:
            d["dram_bytes_per_launch"] = (d.get("dram__bytes_read.sum [bytes]") or 0) + \
                (d.get("dram__bytes_write.sum [bytes]") or 0)
            t = d.get("gpu__time_duration.sum [ms]")
            if t:
                d["dram_GB_s"] = d["dram_bytes_per_launch"] / (t * 1e-3) / 1e9
                if d.get("lts__t_bytes.sum [bytes]") is not None:
                    d["l2_GB_s"] = d["lts__t_bytes.sum [bytes]"] / (t * 1e-3) / 1e9
        summ.append(d)
    out = {"source": os.path.basename(rep), "workload": wl, "kernels": summ}
    with open(os.path.join(ROOT, "profiles", f"{tag}_{wl}_ncu_full.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    path_k = [d for d in summ if "pool_kernel" in d["kernel"] or "path_kernel" in d["kernel"]
              or "query_kernel" in d["kernel"]]
    if path_k:
        with open(os.path.join(ROOT, "profiles", f"ncu_{wl}.json"), "w") as fh:
            json.dump({"round": tag, **path_k[0]}, fh, indent=1)
    if len(sys.argv) > 4 and os.path.exists(sys.argv[4]):
        with open(os.path.join(ROOT, "profiles", f"{tag}_{wl}_launches.json"), "w") as fh:
            json.dump(launches(sys.argv[4]), fh, indent=1)
    print(json.dumps(out, indent=1)[:4000])


if __name__ == "__main__":
    main()
