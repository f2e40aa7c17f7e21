#!/bin/bash
# ncu --set full capture of the config-1 query kernel at N = 2^24
set -u
mkdir -p gpurun_out
cat > gpurun_out/q.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
torch.cuda.set_device(0)
p, wo, wi, u = configs.config1_inputs(1 << 20)
d = torch.device("cuda", 0)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(d)
rep = 16
P = T(p.T).repeat(1, rep).contiguous(); WO = T(wo.T).repeat(1, rep).contiguous()
WI = T(wi.T).repeat(1, rep).contiguous()
U1 = T(u[:, 0]).repeat(rep); U2 = T(u[:, 1]).repeat(rep)
med = configs.config1_medium()
for _ in range(3):
    r = mf.query_batch(med, P, WO, WI, U1, U2)
torch.cuda.synchronize()
print("ok", float(r["sigma_t"].mean()))
PY
python gpurun_out/q.py || exit 1
ncu --set full --clock-control none --import-source on -k regex:"query_kernel" -s 2 -c 1 \
    -o gpurun_out/q_full -f python gpurun_out/q.py > gpurun_out/ncu_q.log 2>&1
echo "ncu rc=$?"
