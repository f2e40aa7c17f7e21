"""Annotated SASS of one kernel from an ncu capture: every instruction with
its executed count (millions of warp instructions), average active lanes and
inline chain (innermost first), plus per-line and per-opcode summaries.
    python tools/prof_lines.py lib.so capture.ncu-rep kernel_substring out.txt"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

so, rep, kname, out_path = sys.argv[1:5]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True,
                     text=True).stdout.splitlines()
start = next(i for i, l in enumerate(dis) if l.startswith(".text.") and kname in l)
off2 = {}
chain, fresh = [], True
for l in dis[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if fresh:
            chain, fresh = [], False
        chain.append(os.path.basename(m.group(1)) + ":" + m.group(2))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?);", l)
    if m:
        off2[int(m.group(1), 16)] = (list(chain), m.group(2))
        fresh = True
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + re.split(r"I[LN]", kname)[0]], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr, data = rows[hi], rows[hi + 1:]
ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
te = hdr.index("Thread Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][ia], 16)
top = defaultdict(lambda: [0.0, 0.0, 0.0])
ops = defaultdict(lambda: [0.0, 0.0])
tot = tots = 0.0
with open(out_path, "w") as fo:
    for r in data:
        off = int(r[ia], 16) - base
        ch, ins = off2.get(off, ([], "?"))
        w, t, s = float(r[ie] or 0), float(r[te] or 0), float(r[ws] or 0)
        tot += w
        tots += s
        k = ch[-1] if ch else "?"
        top[k][0] += w
        top[k][1] += t
        top[k][2] += s
        op = re.sub(r"^@!?U?P[T0-9]+\s+", "", ins).split(" ")[0].split(".")[0]
        ops[op][0] += w
        ops[op][1] += t
        fo.write(f"{off:05x} {w / 1e6:8.3f} {t / max(w, 1):5.1f} {s:6.0f}  {ins:48s} "
                 f"{' <- '.join(ch[:5])}\n")
print(f"total warp instr {tot:.4e}")
print("outermost source line: warp% lanes stall%")
for k, a in sorted(top.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"  {k:24s} {100 * a[0] / tot:6.2f} {a[1] / max(a[0], 1):5.1f} {100 * a[2] / tots:6.2f}")
print("opcodes: warp% lanes")
for k, a in sorted(ops.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"  {k:10s} {100 * a[0] / tot:6.2f} {a[1] / max(a[0], 1):5.1f}")
