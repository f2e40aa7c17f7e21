"""Warp instructions per path and active lanes by code region (grid walker
pieces, kernel, math) from an ncu capture with imported source.
    python tools/region_lanes.py <rep.ncu-rep> <paths per launch>"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, paths = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
src = open("paper_2603_00280_b200/csrc/mf_grid.cuh").read().split("\n")
# function of each mf_grid.cuh line: the last "MF_HD* ... name(" seen above it
fn_of = {}
cur = "?"
for i, line in enumerate(src, 1):
    m = re.match(r"\s*(?:template.*)?MF_HDM?\s+(?:static\s+)?[\w:<>\*& ]+?\s+(\w+)\(", line)
    if m:
        cur = m.group(1)
    fn_of[i] = cur
res = defaultdict(lambda: [0.0, 0.0])
fname, hdr = "?", None
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        wi, ti = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
        continue
    if hdr and len(r) > ti and r[0]:
        try:
            w, t = float(r[wi]), float(r[ti])
        except ValueError:
            continue
        key = "grid:" + fn_of.get(int(r[0]), "?") if fname == "mf_grid.cuh" else fname
        res[key][0] += w
        res[key][1] += t
tw = sum(v[0] for v in res.values())
print(f"warp instr per path {tw / paths:.1f}, lanes {sum(v[1] for v in res.values()) / tw:.1f}")
for k, (w, t) in sorted(res.items(), key=lambda kv: -kv[1][0]):
    if w / tw > 0.002:
        print(f"{k:28s} {w / paths:8.1f} {100 * w / tw:5.1f}%  lanes {t / w:5.1f}")
