"""Config-1 coefficient queries for an ncu capture: 2^24 queries (16 copies
of the 2^20 inputs), two launches (the second is the captured one)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_00280_b200 as mf  # noqa: E402
from paper_2603_00280_b200 import configs  # noqa: E402

rep = int(sys.argv[1]) if len(sys.argv) > 1 else 16
torch.cuda.set_device(0)
p, wo, wi, u = configs.config1_inputs(1 << 20)
d = torch.device("cuda", 0)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(d)  # noqa: E731
P = T(p.T).repeat(1, rep).contiguous()
WO = T(wo.T).repeat(1, rep).contiguous()
WI = T(wi.T).repeat(1, rep).contiguous()
U1, U2 = T(u[:, 0]).repeat(rep), T(u[:, 1]).repeat(rep)
med = configs.config1_medium()
for _ in range(2):
    r = mf.query_batch(med, P, WO, WI, U1, U2)
torch.cuda.synchronize()
print("queries", P.shape[1])
