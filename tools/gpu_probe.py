"""Quick GPU probe: parity spot checks + timings (development tool)."""
import sys, time, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
from oracle import microfacet as OM

def t_events(fn, reps=5, warm=2):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return min(ts), float(np.median(ts))

out = {}
# config 1 queries
p, wo, wi, u = configs.config1_inputs()
med = configs.config1_medium()
dev = torch.device('cuda')
P = torch.from_numpy(p.T.copy()).to(dev); WO = torch.from_numpy(wo.T.copy()).to(dev); WI = torch.from_numpy(wi.T.copy()).to(dev)
U1 = torch.from_numpy(u[:, 0].copy()).to(dev); U2 = torch.from_numpy(u[:, 1].copy()).to(dev)
res = mf.query_batch(med, P, WO, WI, U1, U2)
n = 1 << 16
st = res['sigma_t'][:n].cpu().numpy()
class M: pass
m = M(); m.kind = 'generalized'
class A: pass
m.a3 = A(); a = float(np.float32(med.a3.ax)); m.a3.ax = m.a3.ay = m.a3.az = a; m.sigma = float(np.float32(0.05)); m.mix_ratio = 0.5; m.fresnel_one = True
ref = OM.extinction_local(wo[:n].astype(np.float64), p[:n, 2].astype(np.float64), m)
ok = ref > 1e-35
out['q_sigma_t_maxrel'] = float(np.max(np.abs(st[ok] / ref[ok] - 1)))
ph = res['phase_r'][:n].cpu().numpy(); refp = OM.phase_eval_local(wo[:n].astype(np.float64), wi[:n].astype(np.float64), m)[:, 0]
ok = refp > 1e-30
out['q_phase_maxrel'] = float(np.max(np.abs(ph[ok] / refp[ok] - 1)))
for N in (1 << 20, 1 << 24):
    if N > (1 << 20):
        reps = N >> 20
        P2, WO2, WI2 = [t.repeat(1, reps).contiguous() for t in (P, WO, WI)]
        U12, U22 = U1.repeat(reps), U2.repeat(reps)
    else:
        P2, WO2, WI2, U12, U22 = P, WO, WI, U1, U2
    tmin, tmed = t_events(lambda: mf.query_batch(med, P2, WO2, WI2, U12, U22))
    out[f'query_{N}_ms'] = tmin
    out[f'query_{N}_Mq_s'] = N / tmin / 1e3
# config 2 render
sc = configs.config2_scene()
img, stats = mf.render_device(sc, 64, 1, max_bounces=16, stats=True)
out['c2_stats'] = stats
out['c2_mean'] = float(img.mean().item())
buf = torch.empty_like(img)
tmin, tmed = t_events(lambda: mf.render_device(sc, 64, 1, max_bounces=16, out=buf))
out['c2_ms'] = tmin; out['c2_Mpaths_s'] = 256 * 256 * 64 / tmin / 1e3
# determinism
a = mf.render_device(sc, 64, 1, max_bounces=16)[0].clone(); b = mf.render_device(sc, 64, 1, max_bounces=16, tile=16)[0].clone()
out['c2_det_tile'] = bool(torch.equal(a, b))
# config 2 at higher spp for mean
img2, _ = mf.render_device(sc, 1024, 7, max_bounces=16)
v = img2[..., 0].cpu().numpy()
out['c2_hi_mean'] = float(v.mean()); out['c2_hi_se'] = float(v.std() / np.sqrt(v.size))
# depth 1
img3, _ = mf.render_device(sc, 1024, 7, max_bounces=1)
v = img3[..., 0].cpu().numpy(); out['c2_d1_mean'] = float(v.mean()); out['c2_d1_se'] = float(v.std() / np.sqrt(v.size))
# config 3
sc3 = configs.config3_scene(128, 128)
img, stats = mf.render_device(sc3, 64, 2, max_bounces=32, stats=True)
out['c3_stats'] = stats; out['c3_mean'] = float(img.mean().item())
tmin, _ = t_events(lambda: mf.render_device(sc3, 64, 2, max_bounces=32), reps=3, warm=1)
out['c3_128_64_ms'] = tmin; out['c3_Mpaths_s'] = 128 * 128 * 64 / tmin / 1e3
# transmittance vs closed form
med1 = mf.MacrofacetMedium(kind=mf.NdfKind.GENERALIZED, a3=mf.RoughnessTriple(1, 1, 1), sigma=1.0, fresnel_one=True)
cam = mf.Camera(position=(0, 0, 10), look_at=(0, 0, 0), fov_deg=40, width=4, height=4)
fs = mf.ShellScene(primitives=(mf.ShellPrimitive(mf.Plane(0.0), med1),), camera=cam)
th = np.deg2rad(45.0)
mean, se = mf.transmittance_estimate((np.array([0, 0, 0.0]), np.array([np.sin(th), 0, np.cos(th)])), fs, 1000000, mf.RandomStream(2, 1))
out['tr_mean'] = mean; out['tr_se'] = se
print(json.dumps(out, indent=1))
