"""Executed thread instructions per path grouped by the enclosing source
function (innermost inline frame) from an ncu capture with imported
source.    python tools/func_mix.py <rep> <paths per launch> [csrc dir]"""
import csv
import io
import os
import re
import subprocess
import sys

rep, paths = sys.argv[1], float(sys.argv[2])
csrc = sys.argv[3] if len(sys.argv) > 3 else "paper_2603_00280_b200/csrc"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "sass,cuda"], capture_output=True, text=True).stdout
fn_at = {}
pat = re.compile(r"^(?:template\s*<[^>]*>\s*)?(?:MF_\w+|__device__|__global__|inline|static|"
                 r"__host__)[^;{]*?\b([A-Za-z_]\w*)\s*\(")
for f in os.listdir(csrc):
    lines = open(os.path.join(csrc, f)).read().splitlines()
    cur = "?"
    m = {}
    for i, l in enumerate(lines, 1):
        mm = pat.match(l)
        if mm and not l.rstrip().endswith(";"):
            cur = mm.group(1)
        m[i] = cur
    fn_at[f] = m
agg = {}
fname = "?"
hdr = None
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ti = hdr.index("Thread Instructions Executed")
        continue
    if hdr and len(r) > ti and r[0]:
        try:
            t = float(r[ti])
        except ValueError:
            continue
        fn = fn_at.get(fname, {}).get(int(r[0]), fname)
        key = f"{fname}:{fn}"
        agg[key] = agg.get(key, 0) + t
tot = sum(agg.values())
print(f"total {tot / paths:.1f} thread instructions per path")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:45]:
    print(f"{v / paths:8.1f} {v / tot:6.1%}  {k}")
