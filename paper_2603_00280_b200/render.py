"""Volumetric path tracer on the GPU (reference render.py:32-180).

    render(scene, spp, seed, max_bounces=64, threads=None, tile=32, scene_hash="")
        -> RadianceImage                                      render.py:127-180
    render_device(...) -> (H, W, 3) float32 CUDA tensor (no host copies)
    render_sharded(...)  one rank's share + one NCCL reduce to rank 0
    trace_paths(origins, directions, scene, max_bounces, keys) render.py:32-108
    trace_path(ray, scene, max_bounces, rng)                   render.py:111-124

All path work runs in the persistent CUDA megakernel behind mf_render /
mf_trace_paths.  Every path draws from Philox4x32-10 keyed by the seed with
counter (pixel, sample, segment, call), so images are bit-identical for any
tile size, pass size, thread count or number of GPUs under tile sharding
(the reference's determinism contract, render.py:3-10, with a different
generator -- parity with the reference is statistical).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ParameterDomainError
from .image import RadianceImage
from .scene import ShellScene, to_c_scene

_SHARD = {"tiles": _lib.SHARD_TILES, "samples": _lib.SHARD_SAMPLES}


def _params(spp, seed, max_bounces, tile, shard, rank, nranks, accumulate=False):
    if spp < 1:
        raise ParameterDomainError(f"spp must be >= 1, got {spp}")
    if max_bounces < 1:
        raise ParameterDomainError(f"max_bounces must be >= 1, got {max_bounces}")
    if shard not in _SHARD:
        raise ParameterDomainError(f"shard must be 'tiles' or 'samples', got {shard!r}")
    p = _lib.MfRenderParams()
    p.seed = int(seed) & (2**64 - 1)
    p.spp = int(spp)
    p.max_bounces = int(max_bounces)
    p.tile = int(tile)
    p.shard = _SHARD[shard]
    p.rank, p.nranks = int(rank), int(nranks)
    p.accumulate = 1 if accumulate else 0
    return p


def _c_scene(scene: ShellScene, device):
    """The flattened C scene, built once per (immutable) scene and device."""
    cache = scene.__dict__.get("_c_scene_cache")
    if cache is None:
        cache = {}
        object.__setattr__(scene, "_c_scene_cache", cache)
    cs = cache.get(device)
    if cs is None:
        cs = cache[device] = to_c_scene(scene)
    return cs


class RenderTicket:
    """A render queued on its stream (render_device(wait=False), C ABI
    mf_render_async): `finish()` waits for it, validates it exactly like a
    synchronous render (majorant violations, walker caps and invalid
    radiance raise) and returns the stats dict.  Finish every ticket once;
    tickets of one stream may be finished in any order."""

    def __init__(self, handle, out, keep):
        self._h, self.out, self._keep = handle, out, keep

    def finish(self):
        if self._h is None:
            raise ParameterDomainError("render ticket already finished")
        st = _lib.MfStats()
        h, self._h = self._h, None
        _lib.check(_lib.load().mf_render_finish(h, ctypes.byref(st)))
        return st.as_dict()

    def __del__(self):
        if getattr(self, "_h", None) is not None:   # never finished: release it
            try:
                _lib.load().mf_render_finish(self._h, None)
            except Exception:
                pass


def render_device(scene, spp, seed, max_bounces=64, tile=32, rank=0, nranks=1,
                  shard="tiles", out=None, stats=False, stream=None, c_scene=None, wait=True):
    """Render into a (H, W, 3) float32 CUDA tensor holding radiance / spp for
    this rank's share.  Returns (tensor, stats dict or None); with
    wait=False the render is only queued on the stream and a RenderTicket
    comes back instead (ticket.out is the tensor; ticket.finish() validates
    and returns the stats), so several renders run back to back without a
    host synchronisation between them."""
    prm = _params(spp, seed, max_bounces, tile, shard, rank, nranks)
    torch = _lib.require_cuda()
    lib = _lib.load()
    cam = scene.camera
    if out is None:
        out = torch.empty((cam.height, cam.width, 3), dtype=torch.float32, device="cuda")
    if out.dtype != torch.float32 or not out.is_cuda or not out.is_contiguous() or \
            tuple(out.shape) != (cam.height, cam.width, 3):
        raise ParameterDomainError("out must be a contiguous (H, W, 3) float32 CUDA tensor")
    cs = c_scene if c_scene is not None else _c_scene(scene, out.device.index)
    s = stream if stream is not None else _lib.stream_handle(torch, out.device)
    if not wait:
        h = ctypes.c_void_p()
        _lib.check(lib.mf_render_async(ctypes.byref(cs), ctypes.byref(prm),
                                       ctypes.c_void_p(out.data_ptr()), ctypes.byref(h), s))
        return RenderTicket(h, out, (cs, prm))
    st = _lib.MfStats() if stats else None
    _lib.check(lib.mf_render(ctypes.byref(cs), ctypes.byref(prm), ctypes.c_void_p(out.data_ptr()),
                             ctypes.byref(st) if st is not None else None, s))
    return out, (st.as_dict() if st is not None else None)


def render(scene, spp, seed, max_bounces=64, threads=None, tile=32, scene_hash=""):
    """Render the scene camera (render.py:127-180); `threads` is accepted for
    signature compatibility and ignored (the GPU path is deterministic for
    any launch geometry)."""
    if threads is not None and threads < 1:
        raise ParameterDomainError(f"thread count must be >= 1, got {threads}")
    import torch

    # RadianceImage.validate (image.py:38-42) runs on the device: the path and
    # accumulate kernels count non-finite / negative radiance and mf_render
    # raises NumericFailureError (a MacrofacetError) for any
    img, _ = render_device(scene, spp, seed, max_bounces=max_bounces, tile=tile, stats=True)
    # float64 on the device, one copy into page-locked memory (torch's
    # caching host allocator recycles it); the array keeps its buffer alive
    d64 = img.to(torch.float64)
    host = torch.empty(d64.shape, dtype=torch.float64, pin_memory=True)
    host.copy_(d64, non_blocking=True)
    torch.cuda.current_stream(d64.device).synchronize()
    return RadianceImage(pixels=host.numpy(),
                         meta={"seed": int(seed), "spp": int(spp), "scene_hash": scene_hash})


def render_sharded(scene, spp, seed, max_bounces=64, tile=32, shard="tiles",
                   group=None, stats=False, comm=None, ordered=False):
    """One rank's share of a multi-GPU render followed by a single NCCL
    sum-reduce of the fp32 accumulation buffers to rank 0.
    The kernel writes straight into the tensor NCCL sends, on the same
    stream.  Tile sharding leaves non-owned pixels at +0.0, so the reduce is
    exact and the image is bit-identical for any rank count.

    The reduce runs through torch.distributed unless `comm` (a
    `comm.NcclComm`, the library's own communicator, C ABI `mf_reduce`) is
    given; `ordered=True` (needs `comm`) sums the ranks' buffers in rank
    order on the root, which makes sample-sharded images bit-reproducible
    for a fixed rank count.  Returns the (H, W, 3) tensor (complete on rank
    0) and this rank's stats."""
    import torch.distributed as dist

    if ordered and comm is None:
        raise ParameterDomainError("ordered reduction needs the library communicator (comm=)")
    rank = dist.get_rank(group) if comm is None else comm.rank
    nranks = dist.get_world_size(group) if comm is None else comm.nranks
    img, st = render_device(scene, spp, seed, max_bounces=max_bounces, tile=tile, rank=rank,
                            nranks=nranks, shard=shard, stats=stats)
    if comm is not None:
        comm.reduce(img, root=0, ordered=ordered)
    elif nranks > 1:
        dist.reduce(img, dst=group_root(group), op=dist.ReduceOp.SUM, group=group)
    return img, st


def group_root(group):
    """Global rank of the group's rank 0 (the reduce destination)."""
    import torch.distributed as dist

    return 0 if group is None else dist.get_global_rank(group, 0)


def sample_range(spp, rank, nranks):
    """[begin, end) of the samples rank `rank` renders under sample sharding
    (same split as mf_render)."""
    return spp * rank // nranks, spp * (rank + 1) // nranks


def owned_pixels(width, height, tile, rank, nranks):
    """Pixel indices rank `rank` renders under interleaved tile sharding:
    tile t = ty * tiles_x + tx belongs to rank t mod nranks (the same map
    as local_to_pixel in csrc/mf_kernels.cu)."""
    tx = (width + tile - 1) // tile
    ty = (height + tile - 1) // tile
    out = []
    for t in range(rank, tx * ty, nranks):
        y0, x0 = (t // tx) * tile, (t % tx) * tile
        yy, xx = np.mgrid[y0:min(height, y0 + tile), x0:min(width, x0 + tile)]
        out.append((yy * width + xx).ravel())
    return np.concatenate(out) if out else np.zeros(0, dtype=np.int64)


@dataclass
class PathKeys:
    """Random-stream keys of caller-given paths: path i draws from
    Philox(seed; pixel[i], sample[i], segment, call)."""

    seed: int
    pixel: np.ndarray
    sample: np.ndarray


def _keys_of(brng, n):
    """(seed, pixel, sample) of n paths from PathKeys or a BatchRng-like
    object (`.base` / `.counter`, transport.py:52-67 -- the reference's own
    BatchRng works); a BatchRng's counters advance by one per path."""
    if isinstance(brng, PathKeys):
        return (int(brng.seed), np.broadcast_to(np.asarray(brng.pixel, dtype=np.uint32), (n,)),
                np.broadcast_to(np.asarray(brng.sample, dtype=np.uint32), (n,)))
    if hasattr(brng, "base") and hasattr(brng, "counter"):
        from .rng import BATCH_SEED, philox_keys

        ctr = np.broadcast_to(np.asarray(brng.counter, dtype=np.uint64), (n,))
        pix, smp = philox_keys(brng.base, ctr, n)
        brng.counter = ctr + np.uint64(1)
        return BATCH_SEED, pix, smp
    raise ParameterDomainError("trace_paths needs a BatchRng (base, counter) or PathKeys")


def trace_paths(origins, directions, scene, max_bounces, brng, return_stats=False):
    """Trace caller-given rays to completion (render.py:32-108); returns
    (N, 3) radiance.  `brng`: a BatchRng (reference signature; each path's
    device stream is keyed by its (base, counter), which then advances by
    one) or PathKeys (explicit (seed, pixel, sample) keys)."""
    if max_bounces < 1:
        raise ParameterDomainError(f"max_bounces must be >= 1, got {max_bounces}")
    torch = _lib.require_cuda()
    lib = _lib.load()
    o = np.asarray(origins, dtype=np.float64)
    n = o.shape[0]
    d = np.broadcast_to(np.asarray(directions, dtype=np.float64), (n, 3))
    seed, pix, smp = _keys_of(brng, n)
    dev = torch.device("cuda", torch.cuda.current_device())
    org_t = torch.from_numpy(np.ascontiguousarray(o.T, dtype=np.float32)).to(dev)
    dir_t = torch.from_numpy(np.ascontiguousarray(d.T, dtype=np.float32)).to(dev)
    pix_t = torch.from_numpy(np.array(pix, dtype=np.uint32).view(np.int32)).to(dev)
    smp_t = torch.from_numpy(np.array(smp, dtype=np.uint32).view(np.int32)).to(dev)
    rad = torch.empty((3, n), dtype=torch.float32, device=dev)
    cs = to_c_scene(scene)
    st = _lib.MfStats()
    _lib.check(lib.mf_trace_paths(ctypes.byref(cs), org_t.data_ptr(), dir_t.data_ptr(),
                                  pix_t.data_ptr(), smp_t.data_ptr(), int(seed) & (2**64 - 1),
                                  int(max_bounces), n, rad.data_ptr(), ctypes.byref(st),
                                  _lib.stream_handle(torch, dev)))
    out = rad.cpu().numpy().T.astype(np.float64)
    return (out, st.as_dict()) if return_stats else out


def trace_path(ray, scene, max_bounces, rng):
    """Single-path convenience wrapper keyed by (rng.stream, rng.counter);
    advances rng by one path (render.py:111-124)."""
    origin, direction = ray
    keys = PathKeys(rng.seed, np.array([rng.stream & 0xFFFFFFFF]),
                    np.array([rng.counter & 0xFFFFFFFF]))
    out = trace_paths(np.asarray(origin)[None, :], np.asarray(direction)[None, :], scene,
                      max_bounces, keys)
    rng.counter += 1
    return out[0]
