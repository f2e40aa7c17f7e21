"""Compact, committed summary of one `ncu --set full` capture of a render /
query kernel (profiles/<tag>_<workload>_ncu_full.json): time, issue
utilisation, active lanes, registers, pipe utilisation, DRAM / L2 traffic,
the warp-stall breakdown and the executed-instruction mix per unit (path or
query), next to the kernel's algorithmic FP32 / SFU count when given.

    python tools/profile_summary.py <tag> <workload> <rep.ncu-rep> <units per launch>
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

METRICS = {
    "gpu__time_duration.sum": "time_ms",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_lanes",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__warps_eligible.avg.per_cycle_active": "eligible_warps_per_cycle",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "pipe_fma_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "pipe_alu_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "pipe_xu_pct",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "lts__t_sectors.sum": "l2_sectors",
    "lts__t_sectors.sum.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
}
UNITS = {"ms": 1.0, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "nsecond": 1e-6,
         "s": 1e3, "second": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1.0}


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main():
    tag, wl, rep, units = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, v = r[0], r[1], r[2]
    out = {"source": os.path.basename(rep), "workload": wl, "units_per_launch": units,
           "kernel": v[h.index("Kernel Name")]}
    for k, name in METRICS.items():
        if k in h:
            x = num(v[h.index(k)])
            unit = u[h.index(k)]
            if x is not None and unit in UNITS and (name.endswith("ms") or "bytes" in name):
                x *= UNITS[unit]
            out[name] = x
    stalls = {}
    for i, k in enumerate(h):
        if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
            x = num(v[i])
            if x:
                stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = x
    tot = sum(stalls.values()) or 1.0
    out["stall_share"] = {k: round(x / tot, 4) for k, x in
                          sorted(stalls.items(), key=lambda kv: -kv[1])[:10]}
    out["dram_bytes_per_launch"] = (out.get("dram_read_bytes") or 0) + (out.get("dram_write_bytes") or 0)
    t = out.get("time_ms")
    if t:
        out["dram_GB_s"] = round(out["dram_bytes_per_launch"] / (t * 1e-3) / 1e9, 2)
        if out.get("l2_sectors") is not None:   # 32-byte sectors through the L2 slices
            out["l2_GB_s"] = round(out["l2_sectors"] * 32 / (t * 1e-3) / 1e9, 1)
    # executed-instruction mix per unit (sass_mix's classes)
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    import re
    from collections import Counter
    rows = list(csv.reader(io.StringIO(src)))
    hdr = rows[1]
    si, ti = hdr.index("Source"), hdr.index("Thread Instructions Executed")
    ops = Counter()
    for row in rows[2:]:
        if len(row) <= ti:
            continue
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", row[si].strip())
        if m:
            ops[m.group(2)] += float(row[ti] or 0)
    import importlib.util
    spec = importlib.util.spec_from_file_location("sm", os.path.join(ROOT, "tools", "sass_mix.py"))
    cls_map = {}
    text = open(os.path.join(ROOT, "tools", "sass_mix.py")).read()
    ns = {}
    exec(text[text.index("CLS = {"):text.index("cls = Counter()")], ns)
    for c, s in ns["CLS"].items():
        for op in s:
            cls_map[op] = c
    mix = Counter()
    for op, x in ops.items():
        mix[cls_map.get(op, "other")] += x
    tot_i = sum(ops.values())
    out["thread_instructions_per_unit"] = round(tot_i / units, 1)
    out["mix_per_unit"] = {k: round(x / units, 1) for k, x in mix.most_common()}
    out["fp32_share_of_instructions"] = round(mix["fp32"] / max(tot_i, 1), 4)
    path = os.path.join(ROOT, "profiles", f"{tag}_{wl}_ncu_full.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    # the per-workload DRAM figure bench.py reads for roofline.traffic
    with open(os.path.join(ROOT, "profiles", f"ncu_{wl}.json"), "w") as fh:
        json.dump({"round": tag, "kernel": out["kernel"],
                   "dram_bytes_per_launch": out["dram_bytes_per_launch"],
                   "source": out["source"]}, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
