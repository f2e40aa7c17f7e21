"""Time config-2 / config-3 / config-5 renders and config-1 queries for library
variants given as args (path-kernel time from the library's CUDA events)."""
import os, subprocess, sys, json
here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, os, json
sys.path.insert(0, %r)
import torch, numpy as np
import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs
torch.cuda.set_device(0)
def tm(scene, spp, seed, mb, reps=10):
    # path-kernel time from the library's own CUDA events (mf_stats)
    out = torch.empty((scene.camera.height, scene.camera.width, 3), device="cuda")
    for _ in range(3): mf.render_device(scene, spp, seed, max_bounces=mb, out=out)
    ts = []
    for _ in range(reps):
        _, st = mf.render_device(scene, spp, seed, max_bounces=mb, out=out, stats=True)
        ts.append(st["path_kernel_ms"])
    import hashlib
    tm.hashes.append(hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:12])
    return min(ts), float(out.mean())
tm.hashes = []
c2 = configs.config2_scene(); c3 = configs.config3_scene(256, 256)
t2, m2 = tm(c2, 64, 1, 16); t3, m3 = tm(c3, 64, 2, 32, reps=5)
c5 = configs.config5_scene(256, 256)
t5, m5 = tm(c5, 16, 4, 64, reps=5)
c4 = configs.config4_scene(0.05, 0.1, 512, 512)
t4, m4 = tm(c4, 64, 3, 64, reps=5)
c4b = configs.config4_scene(0.2, 0.02, 512, 512)
t4b, m4b = tm(c4b, 64, 3, 64, reps=5)
_, st = mf.render_device(c2, 64, 1, max_bounces=16, stats=True)
p, wo, wi, u = configs.config1_inputs(1 << 20)
d = torch.device("cuda", 0)
rep = 16
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(d)
P = T(p.T).repeat(1, rep).contiguous(); WO = T(wo.T).repeat(1, rep).contiguous(); WI = T(wi.T).repeat(1, rep).contiguous()
U1 = T(u[:, 0]).repeat(rep); U2 = T(u[:, 1]).repeat(rep)
med = configs.config1_medium()
for _ in range(3): mf.query_batch(med, P, WO, WI, U1, U2)
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
qt = []
for _ in range(5):
    s.record(); mf.query_batch(med, P, WO, WI, U1, U2); e.record(); torch.cuda.synchronize(); qt.append(s.elapsed_time(e))
qms = min(qt)
print(json.dumps({"c4_ms": t4, "c4b_ms": t4b, "c2_ms": t2, "c2_Mpaths_s": 256*256*64/t2/1e3, "c2_mean": m2, "c3_ms": t3, "c3_Mpaths_s": 256*256*64/t3/1e3, "c3_mean": m3, "c5_ms": t5, "c5_mean": m5, "hashes": tm.hashes, "slope_iters_per_path": st["slope_iters"]/st["paths"], "query_2^24_ms": qms, "Mq_s": (1<<24)/qms/1e3}))
''' % here
for so in sys.argv[1:]:
    env = dict(os.environ, MF_LIB_PATH=os.path.abspath(so))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(so), r.stdout.strip() or r.stderr[-2000:], flush=True)
