import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
from oracle import microfacet as om
import parity, test_math_host as T, conftest, subprocess
so = os.path.join(conftest.ROOT, "tests/native/_build/libmf_host.so")
subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off", "-o", so, os.path.join(conftest.ROOT, "tests/native/mf_host_shim.cpp")], check=True)
host = ctypes.CDLL(so)
for sigma in (0.05, 0.2):
    med = configs.planar_medium(sigma, 0.05, float("inf"), 0.8); m = parity.f32_medium(med)
    rs = np.random.default_rng(44); n = 1 << 16
    wo = rs.normal(size=(n, 3)); wo /= np.linalg.norm(wo, axis=-1, keepdims=True)
    wi = rs.normal(size=(n, 3)); wi /= np.linalg.norm(wi, axis=-1, keepdims=True)
    wo, wi = wo.astype(np.float32), wi.astype(np.float32)
    sig = om.projected_area(wo.astype(np.float64), "beckmann", m.a3.ax, m.a3.ay, 0.0)
    keep = sig > 1e-9; wo, wi = wo[keep], wi[keep]
    p = np.zeros((len(wo), 3), np.float32); p[:, 2] = rs.uniform(-6 * sigma, 3 * sigma, len(wo))
    u = rs.uniform(size=(len(wo), 2)).astype(np.float32)
    d = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(d)
    r = mf.query_batch(med, t(p.T), t(wo.T), t(wi.T), t(u[:, 0]), t(u[:, 1]))
    ph = r["phase_r"].cpu().numpy()
    o = T.run_query(host, med, p, wo, wi, u)
    WO, WI = wo.astype(float), wi.astype(float)
    ref = om.phase_eval_local(WO, WI, m)[:, 0]
    tol = parity.phase_tolerance(WO, WI, m)
    e = parity.relerr(ph, ref, 1e-25); eh = parity.relerr(o[1], ref, 1e-25)
    bad = np.flatnonzero((np.abs(ref) > 1e-25) & (e > tol))
    print("sigma", sigma, "n bad", len(bad))
    for i in bad[:8]:
        v = -WO[i]; h = v + WI[i]; h /= np.linalg.norm(h)
        E = (h[0] ** 2 + h[1] ** 2) / m.a3.ax ** 2 / h[2] ** 2
        s = m.a3.ax * np.hypot(WO[i, 0], WO[i, 1]); a = WO[i, 2] / s
        print(f"  dev err {e[i]:.2e} host err {eh[i]:.2e} tol {tol[i]:.2e} E {E:.1f} a {a:.2f} vh {abs(v@h):.3g} hz {h[2]:.3g} ref {ref[i]:.3g}")
