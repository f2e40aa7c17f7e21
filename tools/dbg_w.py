import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
from oracle import microfacet as om
import parity
torch.cuda.set_device(0)
med = configs.planar_medium(0.01, 0.05, float("inf"), 0.8)
m = parity.f32_medium(med)
rs = np.random.default_rng(44); n = 1 << 16
wo = rs.normal(size=(n, 3)); wo /= np.linalg.norm(wo, axis=-1, keepdims=True)
wi = rs.normal(size=(n, 3)); wi /= np.linalg.norm(wi, axis=-1, keepdims=True)
wo, wi = wo.astype(np.float32), wi.astype(np.float32)
sig = om.projected_area(wo.astype(np.float64), m.kind.value, m.a3.ax, m.a3.ay, m.a3.az)
keep = sig > 1e-9; wo, wi = wo[keep], wi[keep]
p = np.zeros((len(wo), 3), np.float32); p[:, 2] = rs.uniform(-6 * 0.01, 3 * 0.01, len(wo))
u = rs.uniform(size=(len(wo), 2)).astype(np.float32)
d = torch.device("cuda", 0); t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(d)
r = {k: v.cpu().numpy() for k, v in mf.query_batch(med, t(p.T), t(wo.T), t(wi.T), t(u[:, 0]), t(u[:, 1])).items()}
WO = wo.astype(np.float64)
ws_r, pdf_r, w_r = parity.oracle_sample(WO, m, u[:, 0], u[:, 1])
ws = np.stack([r["wsx"], r["wsy"], r["wsz"]], -1).astype(np.float64)
e = parity.relerr(r["w_r"], w_r[:, 0], 1e-30)
res = parity.check_samples(ws, r["pdf_s"], np.stack([r["w_r"]] * 3, -1), WO, m, u[:, 0], u[:, 1])
print(res)
idx = np.argsort(-e)[:12]
v = -WO; wm = v + ws_r; wm /= np.linalg.norm(wm, axis=-1, keepdims=True)
for i in idx:
    tan2 = (wm[i, 0] ** 2 + wm[i, 1] ** 2) / wm[i, 2] ** 2
    print(i, 'u', u[i], 'wo', WO[i], 'wm_z', wm[i, 2], 'E', tan2 / m.a3.ax ** 2, 'w_gpu', r["w_r"][i], 'w_ref', w_r[i, 0], 'rel', e[i], 'pdf', r["pdf_s"][i], pdf_r[i])
