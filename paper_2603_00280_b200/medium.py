"""The macrofacet medium and its pointwise operators, on the GPU.

Mirrors the reference's medium API (medium.py:35-207) -- same names,
argument meaning and exceptions -- with every evaluation performed by the
`query` CUDA kernel through the C ABI (mf_query_batch):

    extinction(wo, f, medium, local_frame)        medium.py:91-95
    phase_eval(wo, wi, medium, local_frame)       medium.py:158-178
    phase_pdf(wo, wi, medium, local_frame)        restated ndf.py:397-405 + medium.py:186-189
    phase_sample(wo, medium, local_frame, rng)    medium.py:196-207 (uniforms from `rng`)
    query_batch(...)                              the fused config-1 query

Host numpy inputs are copied to the device and results copied back;
torch CUDA tensors stay on the device (no copies) for the batched form.
Arithmetic is fp32 on the device (the reference is float64); see DESIGN.md
for the tolerance policy.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import Frame
from .errors import DegenerateVisibilityError, ParameterDomainError
from .ndf import NdfKind, RoughnessTriple
from .rng import draw_uniforms

DEFAULT_ETA = (0.2, 0.92, 1.1)
DEFAULT_K = (3.9, 2.45, 2.14)


@dataclass(frozen=True)
class MacrofacetMedium:
    """Appearance parameters of one shell volume (medium.py:35-67).

    `albedo` (not in the reference) replaces the Fresnel term by a constant
    per-channel single-scattering albedo, as BASELINE configs 2-5 require
    (grey F == albedo)."""

    kind: NdfKind
    a3: RoughnessTriple
    sigma: float
    fresnel_eta: tuple = DEFAULT_ETA
    fresnel_k: tuple = DEFAULT_K
    mix_ratio: float = 0.5
    fresnel_one: bool = False
    albedo: tuple | None = None

    def __post_init__(self):
        if not (np.isfinite(self.sigma) and self.sigma > 0.0):
            raise ParameterDomainError(f"sigma must be finite and > 0, got {self.sigma}")
        if not (0.0 <= self.mix_ratio <= 1.0):
            raise ParameterDomainError(f"mix_ratio must lie in [0, 1], got {self.mix_ratio}")
        if self.kind is NdfKind.GENERALIZED and self.a3.az <= 0.0:
            raise ParameterDomainError("GENERALIZED medium requires az > 0")
        if self.kind is not NdfKind.GENERALIZED and self.a3.az != 0.0:
            object.__setattr__(self, "a3", RoughnessTriple(self.a3.ax, self.a3.ay, 0.0))
        object.__setattr__(self, "fresnel_eta", tuple(float(v) for v in self.fresnel_eta))
        object.__setattr__(self, "fresnel_k", tuple(float(v) for v in self.fresnel_k))
        if self.albedo is not None:
            alb = self.albedo
            if np.isscalar(alb):
                alb = (alb, alb, alb)
            alb = tuple(float(v) for v in alb)
            if len(alb) != 3 or not all(0.0 <= v for v in alb):
                raise ParameterDomainError(f"albedo must be 3 non-negative values, got {alb}")
            object.__setattr__(self, "albedo", alb)

    @property
    def shell_half_width(self):
        return 3.0 * self.sigma


def to_c_medium(m) -> _lib.MfMedium:
    """Flatten a medium -- this package's MacrofacetMedium or the
    reference's (read by attribute: kind, a3, sigma, fresnel_eta,
    fresnel_k, mix_ratio, fresnel_one; `albedo` is the BASELINE extension
    and defaults to None)."""
    c = _lib.MfMedium()
    kind = getattr(m.kind, "value", m.kind)
    if kind not in _lib.KIND:
        raise ParameterDomainError(f"unknown NDF kind {m.kind!r}")
    c.kind = _lib.KIND[kind]
    albedo = getattr(m, "albedo", None)
    if albedo is not None:
        c.fresnel = _lib.FRESNEL_ALBEDO
        c.albedo[:] = tuple(float(v) for v in np.broadcast_to(albedo, (3,)))
    elif getattr(m, "fresnel_one", False):
        c.fresnel = _lib.FRESNEL_ONE
    else:
        c.fresnel = _lib.FRESNEL_CONDUCTOR
    c.ax, c.ay, c.az = float(m.a3.ax), float(m.a3.ay), float(m.a3.az)
    c.sigma = float(m.sigma)
    c.mix_ratio = float(getattr(m, "mix_ratio", 0.5))
    c.eta[:] = tuple(float(v) for v in getattr(m, "fresnel_eta", DEFAULT_ETA))
    c.k[:] = tuple(float(v) for v in getattr(m, "fresnel_k", DEFAULT_K))
    return c


def _plane_field():
    p = _lib.MfPrimitive()
    p.shape = _lib.SHAPE_PLANE
    p.z0 = 0.0
    return p


_PLANE_FIELD = _plane_field()


_C_MEDIA = {}


def _c_medium_cached(medium):
    """to_c_medium, memoised by value for hashable (frozen) media."""
    try:
        c = _C_MEDIA.get(medium)
    except TypeError:          # unhashable (a duck-typed medium): no cache
        return to_c_medium(medium)
    if c is None:
        if len(_C_MEDIA) > 256:
            _C_MEDIA.clear()
        c = _C_MEDIA[medium] = to_c_medium(medium)
    return c


# the config-1 outputs (query_batch's default) and the optional visible
# normal of the sample and its mixture density (vndf_sample)
_QUERY_DEFAULT = ("sigma_t", "phase_r", "phase_g", "phase_b", "pdf", "wsx", "wsy", "wsz", "pdf_s",
                  "w_r", "w_g", "w_b", "flags")
_QUERY_OUTS = _QUERY_DEFAULT + ("wmx", "wmy", "wmz", "pdf_m")


def query_batch(medium: MacrofacetMedium, p, wo, wi, u1, u2, field=None, f=None, frame=None,
                outputs=_QUERY_DEFAULT, stream=None, out=None):
    """Fused coefficient query (BASELINE config 1) on device tensors.

    p, wo, wi: (3, n) float32 CUDA tensors (SoA rows); u1, u2: (n,).
    Optional f (n,) and frame (9, n) override the field-derived values.
    `out`: caller-allocated {name: (n,) CUDA tensor} (float32, flags int32)
    to write into instead of allocating.
    Returns {name: CUDA tensor} for the requested outputs."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    n = int(u1.numel())
    dev = u1.device
    for t in (p, wo, wi, u1, u2):
        if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
            raise ParameterDomainError("query_batch expects contiguous float32 CUDA tensors")
    for t in (p, wo, wi):
        if t.dim() != 2 or t.shape[0] != 3 or t.shape[1] != n:
            raise ParameterDomainError("p / wo / wi must be (3, n) tensors")
    # SoA rows by pointer arithmetic (no per-row tensor views: the host path
    # of a 2^20 batch must stay shorter than its ~50 us kernel)
    qi = _lib.MfQueryIn()
    row = 4 * n
    a = p.data_ptr()
    qi.px, qi.py, qi.pz = a, a + row, a + 2 * row
    a = wo.data_ptr()
    qi.wox, qi.woy, qi.woz = a, a + row, a + 2 * row
    a = wi.data_ptr()
    qi.wix, qi.wiy, qi.wiz = a, a + row, a + 2 * row
    qi.u1, qi.u2 = u1.data_ptr(), u2.data_ptr()
    qi.f = f.data_ptr() if f is not None else None
    qi.frame = frame.data_ptr() if frame is not None else None
    qo = _lib.MfQueryOut()
    if out is None:
        out = {}
        for name in outputs:
            dt = torch.int32 if name == "flags" else torch.float32
            out[name] = torch.empty(n, dtype=dt, device=dev)
    for name, t in out.items():
        if name not in _QUERY_OUTS:
            raise ParameterDomainError(f"unknown query output {name!r}")
        want = torch.int32 if name == "flags" else torch.float32
        if t.dtype != want or not t.is_cuda or not t.is_contiguous() or t.numel() != n:
            raise ParameterDomainError(f"output {name!r} must be a contiguous ({n},) "
                                       f"{want} CUDA tensor")
        setattr(qo, name, t.data_ptr())
    fld = field if field is not None else _PLANE_FIELD
    cm = _c_medium_cached(medium)
    s = stream if stream is not None else _lib.stream_handle(torch, dev)
    _lib.check(lib.mf_query_batch(ctypes.byref(cm), ctypes.byref(fld), ctypes.byref(qi),
                                  ctypes.byref(qo), n, s))
    return out


_STREAMS = {}   # the pipeline's three streams per device, created once


def query_batch_host(medium: MacrofacetMedium, p, wo, wi, u1, u2, out=None,
                     outputs=_QUERY_DEFAULT, chunk=1 << 19, device=None):
    """The fused coefficient query from HOST tensors to host tensors
    (BASELINE config 1 end to end): chunks of `chunk` queries flow through
    three CUDA streams -- copy in, query_kernel, copy out -- so the PCIe
    transfers of one chunk overlap the kernel and the transfers of the
    others.  p / wo / wi: (3, n) float32 CPU tensors (pinned for the copies
    to run asynchronously), u1 / u2: (n,).  `out`: {name: (n,) CPU tensor}
    (pinned) to write into; returns it."""
    torch = _lib.require_cuda()
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    n = int(u1.numel())
    if out is None:
        out = {name: torch.empty(n, dtype=torch.int32 if name == "flags" else torch.float32,
                                 pin_memory=True) for name in outputs}
    cur = torch.cuda.current_stream(dev)
    streams = _STREAMS.get(dev)
    if streams is None:
        streams = _STREAMS[dev] = [torch.cuda.Stream(dev) for _ in range(3)]
    for st in streams:
        st.wait_stream(cur)
    for c, a in enumerate(range(0, n, chunk)):
        b = min(n, a + chunk)
        st = streams[c % 3]
        with torch.cuda.stream(st):
            d = []
            for t in (p, wo, wi):        # (3, m) device buffers from the contiguous host rows
                x = torch.empty((3, b - a), dtype=torch.float32, device=dev)
                for k in range(3):
                    x[k].copy_(t[k, a:b], non_blocking=True)
                d.append(x)
            d1 = u1[a:b].to(dev, non_blocking=True)
            d2 = u2[a:b].to(dev, non_blocking=True)
            r = query_batch(medium, d[0], d[1], d[2], d1, d2, outputs=tuple(out),
                            stream=_lib.stream_handle(torch, dev))
            for name, t in r.items():
                out[name][a:b].copy_(t, non_blocking=True)
            for t in (*d, d1, d2, *r.values()):   # keep the chunk's buffers until done
                t.record_stream(st)
    for st in streams:
        cur.wait_stream(st)
    cur.synchronize()
    return out


def _frame_rows(local_frame: Frame, shape):
    rows = []
    for v in (local_frame.tangent, local_frame.bitangent, local_frame.normal):
        v = np.broadcast_to(np.asarray(v, dtype=np.float64), shape + (3,))
        rows.extend([v[..., 0], v[..., 1], v[..., 2]])
    return rows


def _host_query(medium, wo, wi, f, local_frame, u, outputs):
    """Broadcast host arrays, run the device query, return host arrays."""
    torch = _lib.require_cuda()
    wo = np.asarray(wo, dtype=np.float64)
    wi = np.asarray(wi, dtype=np.float64) if wi is not None else wo
    f = np.asarray(f if f is not None else 0.0, dtype=np.float64)
    shape = np.broadcast_shapes(wo.shape[:-1], wi.shape[:-1], f.shape,
                                np.shape(local_frame.normal)[:-1])
    if u is not None:
        shape = np.broadcast_shapes(shape, np.shape(u)[:-1])
    n = int(np.prod(shape)) if shape else 1
    dev = torch.device("cuda", torch.cuda.current_device())

    def col(a):
        return torch.from_numpy(np.ascontiguousarray(
            np.broadcast_to(a, shape).reshape(-1), dtype=np.float32)).to(dev)

    wob = np.broadcast_to(wo, shape + (3,))
    wib = np.broadcast_to(wi, shape + (3,))
    zero = torch.zeros(n, dtype=torch.float32, device=dev)
    p = torch.stack([zero, zero, col(f)])
    wo_t = torch.stack([col(wob[..., k]) for k in range(3)]).contiguous()
    wi_t = torch.stack([col(wib[..., k]) for k in range(3)]).contiguous()
    if u is None:
        u1 = torch.full((n,), 0.5, dtype=torch.float32, device=dev)
        u2 = u1
    else:
        ub = np.broadcast_to(np.asarray(u, dtype=np.float64), shape + (2,))
        u1, u2 = col(ub[..., 0]), col(ub[..., 1])
    fr = torch.stack([col(r) for r in _frame_rows(local_frame, shape)]).contiguous()
    res = query_batch(medium, p, wo_t, wi_t, u1, u2, f=col(f), frame=fr, outputs=outputs)
    return {k: v.cpu().numpy().reshape(shape) for k, v in res.items()}, shape


def extinction(wo, f, medium: MacrofacetMedium, local_frame: Frame):
    """rho(f) * sigma(wo_local) (medium.py:91-95), on the GPU."""
    r, _ = _host_query(medium, wo, None, f, local_frame, None, ("sigma_t",))
    return r["sigma_t"].astype(np.float64)[()]


def phase_eval(wo, wi, medium: MacrofacetMedium, local_frame: Frame):
    """Phase function per steradian, 3 channels (medium.py:158-178), on the GPU.

    Raises DegenerateVisibilityError where sigma(wo) < 1e-12, like the
    reference's vndf_eval (ndf.py:312-313)."""
    r, shape = _host_query(medium, wo, wi, None, local_frame, None,
                           ("phase_r", "phase_g", "phase_b", "flags"))
    if np.any(r["flags"] & 1):
        raise DegenerateVisibilityError("projected area is numerically zero toward wo")
    return np.stack([r["phase_r"], r["phase_g"], r["phase_b"]], axis=-1).astype(np.float64)


def phase_pdf(wo, wi, medium: MacrofacetMedium, local_frame: Frame):
    """Density of phase_sample's direction (not exported by the reference;
    restated from ndf.py:397-405 and medium.py:186-189), on the GPU."""
    r, _ = _host_query(medium, wo, wi, None, local_frame, None, ("pdf",))
    return r["pdf"].astype(np.float64)[()]


def phase_sample(wo, medium: MacrofacetMedium, local_frame: Frame, rng, n=None):
    """Scattered direction, pdf and per-channel weight (medium.py:196-207).

    Uniform pairs (u1, u2) come from `rng.uniform` (two per sample, the
    config-1 convention); the direction is returned in world space."""
    wo = np.asarray(wo, dtype=np.float64)
    shape = wo.shape[:-1] if n is None else (n,)
    u = draw_uniforms(rng, shape + (2,))
    if n is not None and wo.ndim == 1:
        wo = np.broadcast_to(wo, (n, 3))
    r, _ = _host_query(medium, wo, None, None, local_frame, u,
                       ("wsx", "wsy", "wsz", "pdf_s", "w_r", "w_g", "w_b", "flags"))
    if np.any(r["flags"] & 1):
        raise DegenerateVisibilityError("projected area is zero toward wo")
    wi = np.stack([r["wsx"], r["wsy"], r["wsz"]], axis=-1).astype(np.float64)
    w = np.stack([r["w_r"], r["w_g"], r["w_b"]], axis=-1).astype(np.float64)
    return wi, r["pdf_s"].astype(np.float64), w
