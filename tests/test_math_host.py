"""The device math (csrc/mf_math.cuh, mf_query.cuh) compiled for the host
and checked against scipy / mpmath / the float64 oracle (CPU only).

The same source runs on sm_100a; tests/test_gpu_query.py repeats the
query checks on the B200 through the C ABI."""

import ctypes

import mpmath as mp
import numpy as np
import pytest
from scipy import special as sps

from oracle import microfacet as om
from paper_2603_00280_b200 import _lib, configs
from paper_2603_00280_b200.medium import to_c_medium

import parity

SQPI = np.sqrt(np.pi)


def special(lib, which, x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(x)
    assert lib.mfh_special(ctypes.c_int(which), x.ctypes.data_as(ctypes.c_void_p),
                           out.ctypes.data_as(ctypes.c_void_p), ctypes.c_int64(x.size)) == 0
    return out.astype(np.float64)


def rel(a, b):
    return np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))


X = np.concatenate([np.linspace(0, 5, 5001), np.geomspace(5, 1e5, 801)]).astype(np.float32)


def test_erfcx_family(host_math):
    x = X.astype(np.float64)
    assert rel(special(host_math, 0, X), sps.erfcx(x)) < 4e-7
    mp.mp.dps = 50
    ie = np.array([float(1 / mp.sqrt(mp.pi) - mp.mpf(float(xx)) * mp.erfc(mp.mpf(float(xx)))
                         * mp.exp(mp.mpf(float(xx)) ** 2)) for xx in x[::7]])
    assert rel(special(host_math, 1, X[::7]), ie) < 1e-6


def test_bterm_against_mpmath(host_math):
    mp.mp.dps = 40
    xs = np.concatenate([np.linspace(0, 6, 61), np.geomspace(6, 2000, 40)]).astype(np.float32)
    ref = []
    for xx in xs.astype(np.float64):
        x = mp.mpf(float(xx))
        erfcx = mp.exp(x * x) * mp.erfc(x)
        ref.append(float((1 + x * x) - mp.sqrt(mp.pi) * x * (x * x + mp.mpf(3) / 2) * erfcx))
    assert rel(special(host_math, 2, xs), np.array(ref)) < 3e-6


def test_erfc_erfinv_ndtri(host_math):
    xs = np.linspace(-9, 9, 4001).astype(np.float32)
    assert rel(special(host_math, 3, xs), sps.erfc(xs.astype(np.float64))) < 4e-7
    p = np.concatenate([np.geomspace(1e-30, 0.49, 3000),
                        1 - np.geomspace(6e-8, 0.49, 3000)]).astype(np.float32)
    assert rel(special(host_math, 4, p), sps.ndtri(p.astype(np.float64))) < 2e-6
    assert rel(special(host_math, 8, p), -sps.erfcinv(2 * p.astype(np.float64))) < 2e-6


def test_mills_and_log_ndtr(host_math):
    u = np.linspace(-40, 12, 20001).astype(np.float32)
    ud = u.astype(np.float64)
    ref = np.exp(-0.5 * ud * ud - sps.log_ndtr(ud)) / np.sqrt(2 * np.pi)
    assert rel(special(host_math, 5, u), ref) < 2e-6
    u2 = np.linspace(-12, 8, 20001).astype(np.float32)
    assert rel(special(host_math, 6, u2), sps.log_ndtr(u2.astype(np.float64))) < 2e-6
    L = sps.log_ndtr(np.linspace(-7, 4, 1001)).astype(np.float32)
    Ld = L.astype(np.float64)
    ref = np.where(Ld < -np.log(2), sps.ndtri(np.exp(Ld)), -sps.ndtri(-np.expm1(Ld)))
    assert np.max(np.abs(special(host_math, 7, L) - ref)) < 2e-6


def test_density_matches_oracle(host_math):
    # rho(f) sigma = phi/Phi (medium.py:70-88), including the deep series region
    u = np.linspace(-60, 10, 7001).astype(np.float32)
    got = special(host_math, 5, u)
    ref = om.density(u.astype(np.float64), 1.0)
    tol = np.maximum(2e-6, 4 * u.astype(np.float64) ** 2 * 2.0 ** -24)
    assert np.all(np.abs(got - ref) <= tol * ref)


def run_query(lib, med, p, wo, wi, u, field=None):
    cm = to_c_medium(med)
    fld = field or _lib.MfPrimitive()
    ins = [np.ascontiguousarray(a, dtype=np.float32) for a in
           (p[:, 0], p[:, 1], p[:, 2], wo[:, 0], wo[:, 1], wo[:, 2], wi[:, 0], wi[:, 1], wi[:, 2],
            u[:, 0], u[:, 1])]
    n = len(u)
    outs = [np.zeros(n, np.float32) for _ in range(16)]
    ip = (ctypes.c_void_p * 11)(*[a.ctypes.data for a in ins])
    op = (ctypes.c_void_p * 16)(*[a.ctypes.data for a in outs])
    assert lib.mfh_query(ctypes.byref(cm), ctypes.byref(fld), ip, op, ctypes.c_int64(n)) == 0
    return outs


def test_config1_queries_host(host_math):
    p, wo, wi, u = configs.config1_inputs(n=1 << 15)
    med = configs.config1_medium()
    m = parity.f32_medium(med)
    o = run_query(host_math, med, p, wo, wi, u)
    P, WO, WI = (a.astype(np.float64) for a in (p, wo, wi))
    r = parity.check_sigma_t(o[0], P[:, 2], m.sigma, om.extinction_local(WO, P[:, 2], m))
    assert r["n_bad"] == 0, r
    assert r["max_rel_in_band"] < 1e-5
    r = parity.check_rel(o[1], om.phase_eval_local(WO, WI, m)[:, 0],
                         tol=parity.phase_tolerance(WO, WI, m))
    assert r["n_bad"] == 0, r
    r = parity.check_rel(o[4], om.phase_pdf_local(WO, WI, m), tol=parity.pdf_tolerance(WO, WI))
    assert r["n_bad"] == 0, r
    ws = np.stack([o[5], o[6], o[7]], axis=-1)
    w = np.stack([o[9], o[10], o[11]], axis=-1)
    r = parity.check_samples(ws, o[8], w, WO, m, u[:, 0], u[:, 1])
    assert r["frac_dir_within_1e-5"] >= 0.9999, r
    assert r["frac_pdf_within_1e-5"] >= 0.995 and r["frac_w_within_1e-5"] >= 0.995, r
    assert r["n_dir_bad"] == 0 and r["n_pdf_bad"] == 0 and r["n_w_bad"] == 0, r


@pytest.mark.parametrize("sigma,lz", [(0.01, 0.02), (0.2, 0.02), (0.05, 0.1), (0.2, 0.1),
                                      (0.05, float("inf"))])
def test_config4_media_host(host_math, sigma, lz):
    """Rough / height-field media of the config-4 sweep (generalized NDF's
    downward branch, Beckmann limit) on random directions at f = 0."""
    med = configs.planar_medium(sigma, 0.05, lz, 0.8)
    m = parity.f32_medium(med)
    rs = np.random.default_rng(4)
    n = 8192
    wo = rs.normal(size=(n, 3))
    wo /= np.linalg.norm(wo, axis=-1, keepdims=True)
    wi = rs.normal(size=(n, 3))
    wi /= np.linalg.norm(wi, axis=-1, keepdims=True)
    wo, wi = wo.astype(np.float32), wi.astype(np.float32)
    # keep views the reference can evaluate (sigma(wo) >= 1e-12, ndf.py:312)
    sig = om.projected_area(wo.astype(np.float64), m.kind.value, m.a3.ax, m.a3.ay, m.a3.az)
    keep = sig > 1e-9
    wo, wi = wo[keep], wi[keep]
    p = np.zeros((len(wo), 3), np.float32)
    u = rs.uniform(size=(len(wo), 2)).astype(np.float32)
    o = run_query(host_math, med, p, wo, wi, u)
    WO, WI = wo.astype(np.float64), wi.astype(np.float64)
    r = parity.check_rel(o[1], om.phase_eval_local(WO, WI, m)[:, 0], floor=1e-25,
                         tol=parity.phase_tolerance(WO, WI, m))
    assert r["n_bad"] == 0, r
    r = parity.check_rel(o[0], om.extinction_local(WO, np.zeros(len(WO)), m), floor=1e-25)
    assert r["n_bad"] == 0, r


def test_uniforms_strictly_inside_unit_interval(host_math):
    """The device uniform u01 never returns 0 or 1 (1.0f made erfinv(2u-1)
    infinite and stalled the walker on NaN directions)."""
    host_math.mfh_u01.restype = ctypes.c_float
    host_math.mfh_u01.argtypes = [ctypes.c_uint32]
    lo = host_math.mfh_u01(0)
    hi = host_math.mfh_u01(0xFFFFFFFF)
    assert 0.0 < lo < 1e-6 and 1.0 - 1e-6 < hi < 1.0


def test_query_clamps_boundary_uniforms(host_math):
    med = configs.config1_medium()
    p = np.zeros((4, 3), np.float32)
    wo = np.tile(np.array([0.6, 0.0, -0.8], np.float32), (4, 1))
    u = np.array([[0.0, 0.0], [1.0, 1.0], [0.25, 1.0], [0.75, 0.0]], np.float32)
    o = run_query(host_math, med, p, wo, wo, u)
    for k in (5, 6, 7, 8, 9):
        assert np.all(np.isfinite(o[k]))
