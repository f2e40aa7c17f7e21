"""Annotated SASS of one kernel from an ncu capture: every instruction with
its executed count (millions of warp instructions), average active lanes and
inline chain (innermost first), plus per-line and per-opcode summaries.
Out-of-line device functions the kernel calls (listed by ncu after the
kernel body) are matched to their nvdisasm sections by instruction text.
    python tools/prof_lines.py lib.so capture.ncu-rep kernel_substring out.txt"""
import csv
import io
import os
import re
import subprocess
import sys
from collections import defaultdict

so, rep, kname, out_path = sys.argv[1:5]
tmp = subprocess.run(["mktemp", "-d"], capture_output=True, text=True).stdout.strip()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True,
                     text=True).stdout.splitlines()

# every function section: name -> list of (chain, instruction text)
sections = {}
cur, chain, fresh = None, [], True
cur_callee = [None]
for l in dis:
    if l.startswith(".text."):
        cur = l[len(".text."):].rstrip(":")
        sections[cur] = []
        chain, fresh = [], True
        cur_callee[0] = None
        continue
    if cur is None:
        continue
    m = re.match(r"^\$[^$]+\$(_Z\w+):$", l)
    if m:
        # an out-of-line callee placed in the kernel's section: its inline
        # chains are unreliable past the innermost frame; tag by callee
        callee = re.sub(r"^_ZN2mf\d+", "", m.group(1))
        callee = re.match(r"[A-Za-z_]+", callee).group(0) if callee else m.group(1)
        cur_callee[0] = callee
        chain, fresh = [], True
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if fresh:
            chain, fresh = [], False
        chain.append(os.path.basename(m.group(1)) + ":" + m.group(2))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s*(.*?);", l)
    if m:
        ch = list(chain) if cur_callee[0] is None else chain[:1] + [f"<{cur_callee[0]}>"]
        sections[cur].append((ch, re.sub(r"\s+", " ", m.group(2)).strip()))
        fresh = True

txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + re.split(r"I[LN]", kname)[0]], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
hdr, data = rows[hi], rows[hi + 1:]
isrc, ie = hdr.index("Source"), hdr.index("Instructions Executed")
te = hdr.index("Thread Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
ncu_txt = [re.sub(r"\s+", " ", r[isrc]).strip().rstrip(";") for r in data]

# lay the sections over the ncu listing: the kernel first, then callees found
# by matching their first 8 instructions
kern = next(k for k in sections if kname in k)
labels = [None] * len(data)
def place(name, start):
    for j, (ch, ins) in enumerate(sections[name]):
        if start + j < len(labels):
            labels[start + j] = (name, ch, ins)
place(kern, 0)
pos = len(sections[kern])
norm = lambda s: re.sub(r"`\([^)]*\)|0x[0-9a-f]+", "", s)
while pos < len(data):
    probe = [norm(t) for t in ncu_txt[pos:pos + 8]]
    hit = None
    for name, ins in sections.items():
        if name == kern or len(ins) < 2:
            continue
        if [norm(t) for _, t in ins[:8]] == probe[:len(ins[:8])]:
            hit = name
            break
    if hit is None:
        pos += 1
        continue
    place(hit, pos)
    pos += len(sections[hit])

top = defaultdict(lambda: [0.0, 0.0, 0.0])
ops = defaultdict(lambda: [0.0, 0.0])
tot = tots = 0.0
with open(out_path, "w") as fo:
    for i, r in enumerate(data):
        w, t, s = float(r[ie] or 0), float(r[te] or 0), float(r[ws] or 0)
        fn, ch, ins = labels[i] if labels[i] else ("?", [], ncu_txt[i])
        tot += w
        tots += s
        k = (ch[-1] if ch else "?") + ("" if fn == kern else f" [{fn[:30]}]")
        top[k][0] += w
        top[k][1] += t
        top[k][2] += s
        op = re.sub(r"^@!?U?P[T0-9]+\s+", "", ins).split(" ")[0].split(".")[0]
        ops[op][0] += w
        ops[op][1] += t
        fo.write(f"{i:05d} {w / 1e6:8.3f} {t / max(w, 1):5.1f} {s:6.0f}  {ins:48s} "
                 f"{' <- '.join(ch)}{'' if fn == kern else ' [' + fn + ']'}\n")
print(f"total warp instr {tot:.4e}")
print("outermost source line: warp% lanes stall%")
for k, a in sorted(top.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"  {k:60s} {100 * a[0] / tot:6.2f} {a[1] / max(a[0], 1):5.1f} {100 * a[2] / tots:6.2f}")
print("opcodes: warp% lanes")
for k, a in sorted(ops.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"  {k:10s} {100 * a[0] / tot:6.2f} {a[1] / max(a[0], 1):5.1f}")
