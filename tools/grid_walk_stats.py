"""Config-5 walk statistics on the host build of the grid walker
(csrc/mf_grid.cuh compiled into the test shim with -DMF_GRID_STATS): DDA
iterations, tentative collisions and empty-space skips per walk, for camera
rays (collision walks) and sun shadow rays from their collisions (ratio
walks).  Used to choose the majorant-grid layout; not part of the product.

    python tools/grid_walk_stats.py [n_maj] [rays_per_side]"""
import ctypes
import math
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2603_00280_b200.grid import config5_fields  # noqa: E402
from test_grid_host import grid_scene  # noqa: E402

n_maj = int(sys.argv[1]) if len(sys.argv) > 1 else 64
side = int(sys.argv[2]) if len(sys.argv) > 2 else 128
so = "/tmp/libmf_gstat.so"
flags = os.environ.get("MF_GSTAT_FLAGS", "").split()
subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off",
                "-DMF_GRID_STATS", *flags, "-o", so,
                os.path.join(ROOT, "tests", "native", "mf_host_shim.cpp")], check=True)
lib = ctypes.CDLL(so)
lib.mfh_grid_stats.restype = ctypes.POINTER(ctypes.c_longlong)
gs = lib.mfh_grid_stats()

sdf, sig = config5_fields(seed=4)
sdf = sdf.values
cs, maj = grid_scene(sdf, sig, 0.03, 0.08, n_maj, lib)
print(f"n_maj {n_maj}: medium cells {np.mean(maj > 0):.3f}")

# pinhole 40 deg at (0,-4,1.2) looking at the origin (configs.config5_scene)
eye = np.array([0.0, -4.0, 1.2])
fwd = -eye / np.linalg.norm(eye)
right = np.cross(fwd, [0.0, 0.0, 1.0]); right /= np.linalg.norm(right)
up = np.cross(right, fwd)
t = math.tan(math.radians(20.0))
ys, xs = np.mgrid[0:side, 0:side]
sx = ((xs + 0.5) / side * 2 - 1) * t
sy = (1 - (ys + 0.5) / side * 2) * t
d = fwd[None] + sx.ravel()[:, None] * right[None] + sy.ravel()[:, None] * up[None]
d /= np.linalg.norm(d, axis=1, keepdims=True)
n = d.shape[0]
O = np.ascontiguousarray(np.tile(eye, (n, 1)).T, np.float32)
D = np.ascontiguousarray(d.T, np.float32)


def walk(O, D, ratio, rr=0.0):
    n = O.shape[1]
    st = np.zeros(n, np.int32)
    pos = np.zeros((3, n), np.float32)
    w = np.zeros(n, np.float32)
    v = ctypes.c_int64()
    for i in range(8):
        gs[i] = 0
    assert lib.mfh_walk(ctypes.byref(cs), O.ctypes.data_as(ctypes.c_void_p),
                        D.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(n), ctypes.c_uint64(4),
                        int(ratio), st.ctypes.data_as(ctypes.c_void_p),
                        pos.ctypes.data_as(ctypes.c_void_p), w.ctypes.data_as(ctypes.c_void_p),
                        ctypes.c_float(1.0), ctypes.byref(v), ctypes.c_float(rr)) == 0
    it, tent, skip, walks, med = (gs[i] for i in range(5))
    print(f"   medium-cell crossings/walk {med / max(walks, 1):.2f}")
    return st, pos, w, v.value, it / max(walks, 1), tent / max(walks, 1), skip / max(walks, 1), walks


st, pos, w, viol, it, tent, skip, nw = walk(O, D, False)
print(f"camera walks {nw}: collided {np.mean(st == 2):.3f}  iters/walk {it:.1f}  "
      f"tentatives/walk {tent:.2f}  skips/walk {skip:.2f}  viol {viol}")
hit = st == 2
sun = np.array([1.0, -1.0, 2.0]); sun /= np.linalg.norm(sun)
P = np.ascontiguousarray(pos[:, hit], np.float32)
S = np.ascontiguousarray(np.tile(sun, (P.shape[1], 1)).T, np.float32)
_, _, w2, viol2, it2, tent2, skip2, nw2 = walk(P, S, True, 0.05)
print(f"shadow walks {nw2}: mean Tr {w2.astype(np.float64).mean():.9f}  iters/walk {it2:.1f}  "
      f"tentatives/walk {tent2:.2f}  skips/walk {skip2:.2f}  viol {viol2}")

if os.environ.get("MF_GSTAT_HIST"):
    h = 3.2 / n_maj
    m = maj[maj > 0] * h
    for q in (0.01, 0.03, 0.1, 0.3, 1.0, 3.0):
        print(f"  cells with mu*h < {q}: {np.mean(m < q):.3f}")
    M = maj.reshape(n_maj, n_maj, n_maj)
    for b in (2, 4):
        nb = n_maj // b
        bm = np.clip(M, 0, None).reshape(nb, b, nb, b, nb, b).max(axis=(1, 3, 5))
        bt = bm * h * b
        print(f"  {b}^3 bricks: medium {np.mean(bm > 0):.3f}; thin (mu_max*size < 0.1) "
              f"{np.mean((bt > 0) & (bt < 0.1)):.3f}, < 0.3 {np.mean((bt > 0) & (bt < 0.3)):.3f}")
