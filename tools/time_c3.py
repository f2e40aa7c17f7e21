"""Config-3 path-kernel time (512^2 x 64 spp, library CUDA events) for
library variants given as args (tools/build_variants.sh)."""
import json
import os
import subprocess
import sys

here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, json, hashlib
sys.path.insert(0, %r)
import torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
torch.cuda.set_device(0)
sc = configs.config3_scene(512, 512)
out = torch.empty((512, 512, 3), device="cuda")
for _ in range(2): mf.render_device(sc, 64, 2, max_bounces=32, out=out)
ts = []
for _ in range(5):
    _, st = mf.render_device(sc, 64, 2, max_bounces=32, out=out, stats=True)
    ts.append(st["path_kernel_ms"])
print(json.dumps({"c3_ms": min(ts), "mean": float(out.mean()),
                  "hash": hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:10]}))
''' % here
for so in sys.argv[1:]:
    env = dict(os.environ, MF_LIB_PATH=os.path.abspath(so))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(so), r.stdout.strip() or r.stderr[-1500:], flush=True)
