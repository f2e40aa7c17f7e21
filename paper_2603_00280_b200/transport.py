"""Null-scattering transport on the GPU (reference transport.py:144-416).

    walk(scene, pos, direction, rng, mode="collision", active=None)
        -> (state, pos, travel, weight, prim)                transport.py:144-297
    transmittance_estimate(ray, scene, n_samples, rng) -> (mean, se)  :300-313
    sample_collision(ray, scene, rng) -> MediumEvent                 :316-416

Every walk runs in `walk_kernel` / `ratio_kernel` behind the C ABI
(mf_walk, mf_transmittance): delta / ratio tracking with the exact
per-step majorant (plane, sphere), the moving Lipschitz band (box) or the
majorant grid (grid fields), and the reference's region rules.  Random
numbers: ray i of a BatchRng draws from the device Philox stream keyed by
(base_i, counter_i) (rng.philox_keys); its counter then advances by one.
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import Frame, build_frame
from .errors import ParameterDomainError
from .rng import BATCH_SEED, philox_keys
from .scene import to_c_scene
from .sdf import shape_name

_MODES = {"collision": _lib.WALK_COLLISION, "ratio": _lib.WALK_RATIO}


class EventKind(enum.Enum):
    ABSORBED_BY_EXIT = "absorbed_by_exit"
    REAL_SCATTER = "real_scatter"
    NULL_SCATTER = "null_scatter"


@dataclass(frozen=True)
class MediumEvent:
    kind: EventKind
    position: np.ndarray
    distance: float
    local_f: float
    local_frame: Frame
    prim_index: int = -1


def _device_walk(scene, pos, direction, pixel, sample, seed, mode):
    torch = _lib.require_cuda()
    lib = _lib.load()
    n = pos.shape[0]
    dev = torch.device("cuda", torch.cuda.current_device())
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)  # noqa: E731
    org = t(pos.T, np.float32)
    dr = t(direction.T, np.float32)
    pix = t(pixel.view(np.int32), np.int32)
    smp = t(sample.view(np.int32), np.int32)
    state = torch.empty(n, dtype=torch.int8, device=dev)
    p_out = torch.empty((3, n), dtype=torch.float32, device=dev)
    travel = torch.empty(n, dtype=torch.float32, device=dev)
    weight = torch.empty(n, dtype=torch.float32, device=dev)
    prim = torch.empty(n, dtype=torch.int32, device=dev)
    cs = to_c_scene(scene)
    st = _lib.MfStats()
    _lib.check(lib.mf_walk(ctypes.byref(cs), org.data_ptr(), dr.data_ptr(), pix.data_ptr(),
                           smp.data_ptr(), int(seed) & (2**64 - 1), 0, int(mode), n,
                           state.data_ptr(), p_out.data_ptr(), travel.data_ptr(),
                           weight.data_ptr(), prim.data_ptr(), ctypes.byref(st),
                           _lib.stream_handle(torch, dev)))
    return (state.cpu().numpy(), p_out.cpu().numpy().T.astype(np.float64),
            travel.cpu().numpy().astype(np.float64), weight.cpu().numpy().astype(np.float64),
            prim.cpu().numpy().astype(np.int64))


def walk(scene, pos, direction, rng, mode="collision", active=None):
    """Advance rays until each reaches a terminal state (transport.py:144-297).

    Returns (state, pos, travel, weight, prim_idx): state 0 = escaped,
    1 = absorbed below the depth cap, 2 = real collision ("collision" mode
    only); weight is the ratio-tracking transparency in "ratio" mode (1.0
    otherwise); prim_idx names the scattering primitive for state 2 (-1
    otherwise).  `rng` is a BatchRng (per-ray base / counter); the counters
    of the walked rays advance by one.  Rays outside `active` are returned
    unchanged (state 0, travel 0, weight 1)."""
    if mode not in _MODES:
        raise ParameterDomainError(f"mode must be 'collision' or 'ratio', got {mode!r}")
    pos = np.asarray(pos, dtype=np.float64)
    n = pos.shape[0]
    direction = np.broadcast_to(np.asarray(direction, dtype=np.float64), (n, 3))
    out_state = np.zeros(n, dtype=np.int8)
    out_pos = np.array(pos, dtype=np.float64)
    out_travel = np.zeros(n)
    out_weight = np.ones(n)
    out_prim = np.full(n, -1, dtype=np.int64)
    prims = tuple(scene.primitives)
    ids = np.arange(n) if active is None else np.flatnonzero(active)
    if not prims or ids.size == 0:
        return out_state, out_pos, out_travel, out_weight, out_prim
    base = np.broadcast_to(np.asarray(rng.base, dtype=np.uint64), (n,))
    ctr = np.broadcast_to(np.asarray(rng.counter, dtype=np.uint64), (n,)).copy()
    pixel, sample = philox_keys(base[ids], ctr[ids], ids.size)
    st, p, tr, w, k = _device_walk(scene, pos[ids], direction[ids], pixel, sample, BATCH_SEED,
                                   _MODES[mode])
    out_state[ids], out_pos[ids], out_travel[ids], out_weight[ids] = st, p, tr, w
    out_prim[ids] = np.where(st == 2, k, -1)
    ctr[ids] += np.uint64(1)
    rng.counter = ctr
    return out_state, out_pos, out_travel, out_weight, out_prim


def transmittance_estimate(ray, scene, n_samples, rng):
    """Unbiased ratio-tracking estimate through all shell intervals along
    the ray (region |f| <= 3 sigma); returns (mean, std_error)."""
    n = int(n_samples)
    if n < 1:
        raise ParameterDomainError(f"n_samples must be >= 1, got {n}")
    torch = _lib.require_cuda()
    lib = _lib.load()
    origin, direction = ray
    o = (ctypes.c_double * 3)(*np.asarray(origin, dtype=np.float64).tolist())
    d = (ctypes.c_double * 3)(*np.asarray(direction, dtype=np.float64).tolist())
    mean = ctypes.c_double()
    se = ctypes.c_double()
    if not tuple(scene.primitives):
        return 1.0, 0.0
    cs = to_c_scene(scene)
    _lib.check(lib.mf_transmittance(ctypes.byref(cs), o, d, n, int(rng.seed) & (2**64 - 1),
                                    int(rng.stream) & (2**64 - 1), ctypes.byref(mean),
                                    ctypes.byref(se), _lib.stream_handle(torch)))
    return float(mean.value), float(se.value)


def _field_and_frame(sdf, p):
    """f and the gradient frame of one primitive at p (sdf.py:18-84,
    transport.py:138-141), on the host: a single event's bookkeeping."""
    name = shape_name(sdf)
    p = np.asarray(p, dtype=np.float64)
    if name == "Plane":
        return float(p[2] - sdf.z0), build_frame(np.array([0.0, 0.0, 1.0]))
    if name == "Sphere":
        d = p - np.asarray(sdf.center, dtype=np.float64)
        r = float(np.linalg.norm(d))
        return r - sdf.radius, build_frame(d / r if r > 0 else np.array([0.0, 0.0, 1.0]))
    if name == "Box":
        d = p - np.asarray(sdf.center, dtype=np.float64)
        q = np.abs(d) - np.asarray(sdf.half_extents, dtype=np.float64)
        out = np.maximum(q, 0.0)
        on = float(np.linalg.norm(out))
        f = on + min(float(np.max(q)), 0.0)
        if on > 0.0:
            g = np.sign(d) * out / on
        else:
            g = np.zeros(3)
            a = int(np.argmax(q))
            g[a] = 1.0 if d[a] >= 0.0 else -1.0
        return f, build_frame(g)
    raise ParameterDomainError(f"no field for {name}")


def sample_collision(ray, scene, rng):
    """Walk one ray to its next tentative collision -- classified real or
    null with probability sigma_t / majorant -- or out of the medium
    (transport.py:316-416); returns a MediumEvent.  `rng` is a
    RandomStream: the ray's device stream is keyed by (its base, counter)
    and the counter advances by one."""
    origin, direction = ray
    o = np.asarray(origin, dtype=np.float64)[None, :]
    d = np.asarray(direction, dtype=np.float64)[None, :]
    prims = tuple(scene.primitives)
    if not prims:
        return MediumEvent(EventKind.ABSORBED_BY_EXIT, o[0].copy(), 0.0, np.inf,
                           build_frame(np.array([0.0, 0.0, 1.0])), -1)
    from .rng import derive_bases

    base = derive_bases(rng.seed, rng.stream, np.array([0]))
    pixel, sample = philox_keys(base, np.uint64(rng.counter), 1)
    st, p, tr, _, k = _device_walk(scene, o, d, pixel, sample, BATCH_SEED,
                                   _lib.WALK_TENTATIVE)
    rng.counter += 1
    state, pos, travel, prim = int(st[0]), p[0], float(tr[0]), int(k[0])
    if state in (2, 3):
        f, fr = _field_and_frame(prims[prim].sdf, pos)
        kind = EventKind.REAL_SCATTER if state == 2 else EventKind.NULL_SCATTER
        return MediumEvent(kind, pos, travel, f, fr, prim)
    # escaped or below the absorption edge: the primitive nearest its
    # surface (escape) / deepest below its edge (absorption)
    vals = [(_field_and_frame(pr.sdf, pos), pr.medium.sigma) for pr in prims]
    if state == 1:
        j = int(np.argmin([v[0][0] + 6.0 * v[1] for v in vals]))
        prim_out = j
    else:
        j = int(np.argmin([abs(v[0][0]) for v in vals]))
        prim_out = -1
    return MediumEvent(EventKind.ABSORBED_BY_EXIT, pos, travel, vals[j][0][0], vals[j][0][1],
                       prim_out)
