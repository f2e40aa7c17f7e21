"""Per-CUDA-source-line executed thread instructions of a kernel from an
ncu capture (imported source, -lineinfo): the top lines per path.

    python tools/line_mix.py <rep.ncu-rep> <paths per launch> [top]"""
import csv
import io
import subprocess
import sys

rep, paths = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "sass,cuda"], capture_output=True, text=True).stdout
res = []
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
    if hdr and len(r) > ti and r[0] not in ("",):
        try:
            t = float(r[ti])
        except ValueError:
            continue
        if t > 0:
            res.append((t, fname, r[0], r[1].strip()[:100]))
tot = sum(x[0] for x in res)
print(f"total thread instr per path {tot / paths:.1f}")
by_file = {}
for t, f, l, s in res:
    by_file[f] = by_file.get(f, 0) + t
for f, t in sorted(by_file.items(), key=lambda kv: -kv[1]):
    print(f"  {f:22s} {t / paths:8.1f}")
for t, f, l, s in sorted(res, reverse=True)[:top]:
    print(f"{t / paths:7.1f} {f}:{l:5s} {s}")
