"""ctypes binding of the C ABI in include/macrofacet_b200.h.

The shared library `libmacrofacet_b200.so` (sm_100a kernels) is built
in-tree by `__graft_entry__.build()` / `python -m paper_2603_00280_b200.build`.
There is no CPU fallback: if the library or a CUDA device is missing, every
compute entry point raises MacrofacetError.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (DegenerateVisibilityError, InternalConsistencyError, MacrofacetError,
                     NumericFailureError, ParameterDomainError, UnsupportedGeometryError)

LIB_NAME = "libmacrofacet_b200.so"
LIB_PATH = os.environ.get("MF_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

MF_MAX_PRIMS = 8
MF_MAX_MEDIA = 8

KIND = {"beckmann": 0, "ggx": 1, "generalized": 2}
REDUCE_NCCL, REDUCE_ORDERED = 0, 1
CURVE = {"lambda": 0, "projected-area": 1, "ndf": 2, "vndf": 3, "transmittance": 4, "density": 5,
         "fresnel": 6, "gdf": 7}
COMM_ID_BYTES = 128
FRESNEL_CONDUCTOR, FRESNEL_ONE, FRESNEL_ALBEDO = 0, 1, 2
SHAPE_PLANE, SHAPE_SPHERE, SHAPE_GRID, SHAPE_BOX = 0, 1, 2, 3
WALK_COLLISION, WALK_RATIO, WALK_TENTATIVE = 0, 1, 2
ABI_VERSION = 4
SHARD_TILES, SHARD_SAMPLES = 0, 1

_d3 = ctypes.c_double * 3


class MfMedium(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("fresnel", ctypes.c_int32),
                ("ax", ctypes.c_double), ("ay", ctypes.c_double), ("az", ctypes.c_double),
                ("sigma", ctypes.c_double), ("mix_ratio", ctypes.c_double),
                ("eta", _d3), ("k", _d3), ("albedo", _d3)]


class MfPrimitive(ctypes.Structure):
    _fields_ = [("shape", ctypes.c_int32), ("medium", ctypes.c_int32), ("z0", ctypes.c_double),
                ("center", _d3), ("radius", ctypes.c_double), ("half_extents", _d3)]


class MfCamera(ctypes.Structure):
    _fields_ = [("ortho", ctypes.c_int32), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("position", _d3), ("look_at", _d3), ("fov_deg", ctypes.c_double),
                ("film_height", ctypes.c_double)]


class MfGridField(ctypes.Structure):
    _fields_ = [("d_sdf", ctypes.c_void_p), ("d_sigma", ctypes.c_void_p),
                ("d_majorant", ctypes.c_void_p), ("n_sdf", ctypes.c_int32),
                ("n_sigma", ctypes.c_int32), ("n_maj", ctypes.c_int32), ("bmin", _d3),
                ("bmax", _d3), ("l_xy", ctypes.c_double), ("l_z", ctypes.c_double)]


class MfScene(ctypes.Structure):
    _fields_ = [("n_prims", ctypes.c_int32), ("n_media", ctypes.c_int32),
                ("prims", MfPrimitive * MF_MAX_PRIMS), ("media", MfMedium * MF_MAX_MEDIA),
                ("camera", MfCamera), ("env", _d3),
                ("d_env_map", ctypes.c_void_p), ("env_width", ctypes.c_int32),
                ("env_height", ctypes.c_int32),
                ("has_sun", ctypes.c_int32), ("sun_dir", _d3), ("sun_radiance", _d3),
                ("has_point", ctypes.c_int32), ("point_pos", _d3), ("point_intensity", _d3),
                ("has_grid", ctypes.c_int32), ("grid", MfGridField)]


class MfRenderParams(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("spp", ctypes.c_int32),
                ("max_bounces", ctypes.c_int32), ("tile", ctypes.c_int32),
                ("shard", ctypes.c_int32), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("accumulate", ctypes.c_int32)]


STAT_FIELDS = ("paths", "segments", "scatters", "nee", "slope_iters", "track_steps", "escaped",
               "absorbed", "majorant_violations", "degenerate", "nonfinite", "capped")


class MfStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in STAT_FIELDS] + [("path_kernel_ms", ctypes.c_double)]

    def as_dict(self):
        d = {n: int(getattr(self, n)) for n in STAT_FIELDS}
        d["path_kernel_ms"] = float(self.path_kernel_ms)
        return d


_vp = ctypes.c_void_p


class MfGpGrid(ctypes.Structure):
    _fields_ = [("d_grid", ctypes.c_void_p), ("n", ctypes.c_int32), ("spacing", ctypes.c_double),
                ("origin", ctypes.c_double), ("planar", ctypes.c_int32),
                ("d_bound", ctypes.c_void_p)]


class MfQueryIn(ctypes.Structure):
    _fields_ = [(n, _vp) for n in ("px", "py", "pz", "wox", "woy", "woz", "wix", "wiy", "wiz",
                                   "u1", "u2", "f", "frame")]


class MfQueryOut(ctypes.Structure):
    _fields_ = [(n, _vp) for n in ("sigma_t", "phase_r", "phase_g", "phase_b", "pdf", "wsx",
                                   "wsy", "wsz", "pdf_s", "w_r", "w_g", "w_b", "flags", "wmx",
                                   "wmy", "wmz", "pdf_m")]


# exported symbols and their signatures (must match include/macrofacet_b200.h)
SIGNATURES = {
    "mf_query_batch": (ctypes.c_int, [ctypes.POINTER(MfMedium), ctypes.POINTER(MfPrimitive),
                                      ctypes.POINTER(MfQueryIn), ctypes.POINTER(MfQueryOut),
                                      ctypes.c_int64, _vp]),
    "mf_render": (ctypes.c_int, [ctypes.POINTER(MfScene), ctypes.POINTER(MfRenderParams), _vp,
                                 ctypes.POINTER(MfStats), _vp]),
    "mf_render_async": (ctypes.c_int, [ctypes.POINTER(MfScene), ctypes.POINTER(MfRenderParams),
                                       _vp, ctypes.POINTER(_vp), _vp]),
    "mf_render_finish": (ctypes.c_int, [_vp, ctypes.POINTER(MfStats)]),
    "mf_gp_noise": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_uint64, ctypes.c_int64, _vp, _vp]),
    "mf_gp_uniform": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_uint64, ctypes.c_int64, _vp,
                                     _vp]),
    "mf_gp_eval": (ctypes.c_int, [ctypes.POINTER(MfGpGrid), _vp, _vp, ctypes.c_int64, _vp, _vp,
                                  _vp]),
    "mf_gp_first_hit": (ctypes.c_int, [ctypes.POINTER(MfGpGrid), _vp, _vp, _vp, ctypes.c_int64,
                                       ctypes.c_double, _vp, ctypes.c_double, _vp, _vp, _vp, _vp,
                                       _vp]),
    "mf_gp_reflect_paths": (ctypes.c_int, [ctypes.POINTER(MfGpGrid), _vp, _vp, _vp, _vp, _vp,
                                           ctypes.c_int64, ctypes.c_int32, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_int32, _vp, _vp, _vp, _vp]),
    "mf_measure_peak_fp64": (ctypes.c_int, [ctypes.POINTER(ctypes.c_double), _vp]),
    "mf_special_f64": (ctypes.c_int, [ctypes.c_int, _vp, ctypes.c_int64, _vp, _vp]),
    "mf_gp_camera_rays": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_int32, ctypes.c_int32, _vp, ctypes.c_int32, _vp,
                                         _vp, _vp]),
    "mf_gp_round_sum": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int32, _vp, _vp]),
    "mf_gdf_radial": (ctypes.c_int, [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_int32, _vp, _vp,
                                     ctypes.POINTER(ctypes.c_double), _vp]),
    "mf_trace_paths": (ctypes.c_int, [ctypes.POINTER(MfScene), _vp, _vp, _vp, _vp,
                                      ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64, _vp,
                                      ctypes.POINTER(MfStats), _vp]),
    "mf_walk": (ctypes.c_int, [ctypes.POINTER(MfScene), _vp, _vp, _vp, _vp, ctypes.c_uint64,
                               ctypes.c_uint32, ctypes.c_int32, ctypes.c_int64, _vp, _vp, _vp,
                               _vp, _vp, ctypes.POINTER(MfStats), _vp]),
    "mf_transmittance": (ctypes.c_int, [ctypes.POINTER(MfScene), ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_double), ctypes.c_int64,
                                        ctypes.c_uint64, ctypes.c_uint64,
                                        ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_double), _vp]),
    "mf_grid_majorant": (ctypes.c_int, [ctypes.POINTER(MfGridField), _vp, _vp]),
    "mf_measure_peaks": (ctypes.c_int, [ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_double), _vp]),
    "mf_comm_unique_id": (ctypes.c_int, [ctypes.POINTER(ctypes.c_ubyte)]),
    "mf_comm_init": (ctypes.c_int, [ctypes.POINTER(ctypes.c_ubyte), ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_void_p)]),
    "mf_comm_destroy": (ctypes.c_int, [_vp]),
    "mf_reduce": (ctypes.c_int, [_vp, _vp, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, _vp]),
    "mf_curve": (ctypes.c_int, [ctypes.POINTER(MfMedium), ctypes.c_int, _vp, _vp, _vp,
                                ctypes.c_int64, ctypes.POINTER(ctypes.c_double), _vp, _vp]),
    "mf_last_error": (ctypes.c_char_p, []),
    "mf_abi_version": (ctypes.c_int, []),
    "mf_launch_count": (ctypes.c_uint64, []),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the CUDA library; raise MacrofacetError if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise MacrofacetError(
                f"{LIB_NAME} is not built ({LIB_PATH}); run "
                "`python -c 'import __graft_entry__ as g; g.build()'` -- there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.mf_abi_version() != ABI_VERSION:
            raise MacrofacetError("libmacrofacet_b200 ABI version mismatch")
        _lib = lib
        return lib


_STATUS = {
    1: ParameterDomainError,
    2: DegenerateVisibilityError,
    3: InternalConsistencyError,
    4: InternalConsistencyError,
    5: NumericFailureError,
    6: UnsupportedGeometryError,
    7: MacrofacetError,
}


def check(status):
    """Raise the reference exception class for a non-zero C-ABI status."""
    if status == 0:
        return
    msg = load().mf_last_error().decode("utf-8", "replace")
    raise _STATUS.get(status, MacrofacetError)(msg)


def require_cuda():
    """torch + a CUDA device are required (device buffers, streams)."""
    import torch

    if not torch.cuda.is_available():
        raise MacrofacetError("no CUDA device: the macrofacet B200 path has no CPU fallback")
    return torch


def stream_handle(torch, device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
