"""Executed thread instructions of chosen SASS opcodes, attributed to the
CUDA source line they come from (ncu capture with imported source):
where the control / integer / select overhead of a kernel sits.

    python tools/op_lines.py <rep> <units> OPC[,OPC...] [top]"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep, units, ops = sys.argv[1], float(sys.argv[2]), set(sys.argv[3].split(","))
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "sass,cuda"], capture_output=True, text=True).stdout
agg, src_of = Counter(), {}
fname, line, hdr = "?", "?", None
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ti = hdr.index("Thread Instructions Executed")
        continue
    if not hdr or len(r) <= ti:
        continue
    if r[0]:
        line = f"{fname}:{r[0]}"
        src_of[line] = r[1].strip()[:80]
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[3])
    if m and m.group(2) in ops:
        agg[line] += float(r[ti] or 0)
tot = sum(agg.values())
print(f"{'/'.join(sorted(ops))}: {tot / units:.1f} thread instructions per unit")
for ln, v in agg.most_common(top):
    print(f"{v / units:7.1f}  {ln:26s} {src_of.get(ln, '')}")
