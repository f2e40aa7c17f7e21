#!/bin/bash
# ncu --set full capture of the megakernel on a reduced config-3 render
# (sphere, 256^2 x 64 spp, depth 32) -- and config 5 (grid) with MF_NCU_C5=1
set -u
mkdir -p gpurun_out
cat > gpurun_out/c3.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
torch.cuda.set_device(0)
if os.environ.get("MF_NCU_C5") == "1":
    sc, spp, seed, mb = configs.config5_scene(512, 512), 16, 4, 64
else:
    sc, spp, seed, mb = configs.config3_scene(512, 512), 64, 2, 32
for _ in range(2):
    img, st = mf.render_device(sc, spp, seed, max_bounces=mb, stats=True)
torch.cuda.synchronize()
print(st)
PY
python gpurun_out/c3.py || exit 1
ncu --set full --clock-control none --import-source on -k regex:"path_kernel" -s 1 -c 1 \
    -o gpurun_out/c3_full -f python gpurun_out/c3.py > gpurun_out/ncu_c3.log 2>&1
echo "ncu rc=$?"
