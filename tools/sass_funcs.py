"""Per source FUNCTION (innermost, inline-aware) dynamic profile of a kernel:
warp instructions, average active lanes, stall samples, static size.
    python tools/sass_funcs.py lib.so capture.ncu-rep kernel_substring [top]"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
so, rep, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40

FDEF = re.compile(r"^\s*(?:template\s*<[^>]*>\s*)?(?:__device__|__global__|inline|static|__forceinline__|MF_\w+)[^;(]*?\b(\w+)\s*\(")
fcache = {}


def func_of(path, line):
    if path not in fcache:
        try:
            src = open(path).read().splitlines()
        except OSError:
            src = []
        names, cur = [], "?"
        for l in src:
            m = FDEF.match(l)
            if m:
                cur = m.group(1)
            names.append(cur)
        fcache[path] = names
    names = fcache[path]
    return (os.path.basename(path), names[line - 1] if 0 < line <= len(names) else "?")


tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True,
                     text=True).stdout.splitlines()
start = next(i for i, l in enumerate(dis) if l.startswith(".text.") and kname in l)
off2f = {}
cur = None
fresh = True
for l in dis[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if fresh:
            cur = func_of(m.group(1), int(m.group(2)))
            fresh = False
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        off2f[int(m.group(1), 16)] = cur
        fresh = True

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + re.split(r"I[LN]", kname)[0]], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr, data = rows[hi], rows[hi + 1:]
ia = hdr.index("Address")
ie = hdr.index("Instructions Executed")
te = hdr.index("Thread Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][ia], 16)
agg = defaultdict(lambda: [0.0, 0.0, 0.0, 0])
for r in data:
    try:
        off = int(r[ia], 16) - base
    except ValueError:
        continue
    a = agg[off2f.get(off, ("?", "?"))]
    a[0] += float(r[ie] or 0)
    a[1] += float(r[te] or 0)
    a[2] += float(r[ws] or 0)
    a[3] += 1
tw = sum(a[0] for a in agg.values())
ts = sum(a[2] for a in agg.values())
print(f"total warp instr {tw:.3e}, avg lanes {sum(a[1] for a in agg.values()) / tw:.2f}")
print(f"{'function':>40} {'warp%':>6} {'lanes':>6} {'stall%':>7} {'static':>7}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0] + ':' + k[1]:>40} {100 * a[0] / tw:6.2f} {a[1] / max(a[0], 1):6.1f} "
          f"{100 * a[2] / max(ts, 1):7.2f} {a[3]:7d}")
