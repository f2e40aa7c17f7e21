"""Per-source-line warp instructions, active lanes and stall samples of a
kernel from an ncu capture (imported source, -lineinfo), sorted by warp
instructions: where divergence costs issue slots.

    python tools/line_lanes.py <rep.ncu-rep> <paths per launch> [top] [file filter]"""
import csv
import io
import subprocess
import sys

rep, paths = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
filt = sys.argv[4] if len(sys.argv) > 4 else ""
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
        wi = hdr.index("Instructions Executed")
        ti = hdr.index("Thread Instructions Executed")
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr and len(r) > ti and r[0]:
        try:
            w, t, smp = float(r[wi]), float(r[ti]), float(r[si] or 0)
        except ValueError:
            continue
        if w > 0 and filt in fname:
            res.append((w, t, smp, f"{fname}:{r[0]}", r[1].strip()[:70]))
tw = sum(x[0] for x in res)
ts = sum(x[2] for x in res)
print(f"warp instr per path {tw / paths:.1f}, lanes {sum(x[1] for x in res) / max(tw, 1):.1f}")
for w, t, smp, loc, src in sorted(res, reverse=True)[:top]:
    print(f"{w / paths:8.1f} {100 * w / tw:5.1f}% lanes {t / w:5.1f} stall {100 * smp / max(ts, 1):5.1f}%  "
          f"{loc:24s} {src}")
