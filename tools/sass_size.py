"""Static SASS size of a kernel by source function (inline-aware):
    python tools/sass_size.py lib.so kernel_substring [top]
Counts instructions whose innermost source line lies in each function, and
the number of distinct inline call sites of each function."""
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

so, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True,
                     text=True).stdout.splitlines()

FDEF = re.compile(r"^\s*(?:template\s*<[^>]*>\s*)?(?:__device__|__global__|inline|static|__forceinline__|MF_\w+)[^;(]*?\b(\w+)\s*\(")
fcache = {}


def func_of(path, line):
    if path not in fcache:
        try:
            src = open(path).read().splitlines()
        except OSError:
            src = []
        names = []
        cur = "?"
        for l in src:
            m = FDEF.match(l)
            if m:
                cur = m.group(1)
            names.append(cur)
        fcache[path] = names
    names = fcache[path]
    return names[line - 1] if 0 < line <= len(names) else "?"


start = next(i for i, l in enumerate(dis) if l.startswith(".text.") and kname in l)
count = defaultdict(int)
sites = defaultdict(set)
loc = None
n = 0
for l in dis[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if m:
        if loc is None or not l.lstrip().startswith("//## File") or True:
            pass
        f, ln = m.group(1), int(m.group(2))
        if loc is None or loc[2]:
            loc = [f, ln, False, None]
        if m.group(3):
            loc[3] = loc[3] or (m.group(3), int(m.group(4)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        if loc:
            fn = func_of(loc[0], loc[1])
            count[(os.path.basename(loc[0]), fn)] += 1
            if loc[3]:
                sites[(os.path.basename(loc[0]), fn)].add(loc[3])
            loc[2] = True
        n += 1
print(f"{n} instructions ({n * 16 / 1024:.1f} KiB)")
for k, v in sorted(count.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v:6d} {v * 16 / 1024:6.1f} KiB  sites={len(sites[k]):3d}  {k[0]}:{k[1]}")
