"""Join an ncu SASS source-page CSV with nvdisasm line info: per source line
warp instructions, thread instructions (avg active lanes) and stall samples.
    python tools/sass_lines.py ncu_sass.csv dis.txt kernel_substring [top]"""
import csv
import re
import sys
from collections import defaultdict

csv_path, dis_path, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(dis_path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and kname in l and l.endswith(":"))
off2src = {}
cur = None
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//---"):
        if off2src:
            break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        off2src[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
data = rows[2:]
ie = hdr.index("Instructions Executed")
te = hdr.index("Thread Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][0], 16)
agg = defaultdict(lambda: [0.0, 0.0, 0.0])
for r in data:
    off = int(r[0], 16) - base
    key = off2src.get(off, ("?", 0))
    a = agg[key]
    a[0] += float(r[ie] or 0)
    a[1] += float(r[te] or 0)
    a[2] += float(r[ws] or 0)
tot_w = sum(a[0] for a in agg.values())
tot_s = sum(a[2] for a in agg.values())
print(f"total warp instr {tot_w:.3e}, avg lanes {sum(a[1] for a in agg.values()) / tot_w:.2f}")
for key, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{key[0]:>20}:{key[1]:<5} warp% {100 * a[0] / tot_w:5.2f}  lanes {a[1] / max(a[0], 1):5.1f}"
          f"  stall% {100 * a[2] / max(tot_s, 1):5.2f}")
