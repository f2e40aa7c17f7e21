"""Print tools/time_variants.py output (gpurun_out/variants.txt) as a table."""
import json
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/variants.txt"
for line in open(path):
    n, _, j = line.partition(" ")
    try:
        d = json.loads(j)
    except Exception:
        print(line[:300].rstrip())
        continue
    keys = [k for k in ("c4_ms", "c4b_ms", "c2_ms", "c3_ms", "c5_ms", "query_2^24_ms") if k in d]
    print(f"{n:14s} " + "  ".join(f"{k[:-3]} {d[k]:.4f}" for k in keys) + "  " + " ".join(d.get("hashes", [])))
