"""Closed-form curves on the B200 (C ABI mf_curve, `curves` CLI) vs the
float64 oracle, the device validation suites (`validate` CLI), and their
error statuses."""

import numpy as np
import pytest

from oracle import microfacet as om
from paper_2603_00280_b200 import cli, curves, validate
from paper_2603_00280_b200.errors import (DegenerateVisibilityError, GrazingSingularityError,
                                          UnsupportedGeometryError)
from paper_2603_00280_b200.medium import MacrofacetMedium
from paper_2603_00280_b200.ndf import NdfKind, RoughnessTriple

import parity

pytestmark = pytest.mark.gpu

ULP = 2.0 ** -24
MEDIA = [
    (NdfKind.GENERALIZED, RoughnessTriple(0.7071, 0.7071, 0.7071)),
    (NdfKind.GENERALIZED, RoughnessTriple(1.4142, 1.4142, 2.8284)),
    (NdfKind.GENERALIZED, RoughnessTriple(5.657, 5.657, 0.707)),
    (NdfKind.BECKMANN, RoughnessTriple(0.283, 0.283, 0.0)),
    (NdfKind.GGX, RoughnessTriple(0.5, 0.8, 0.0)),
]


def _dirs(n, seed):
    w = np.random.default_rng(seed).normal(size=(n, 3))
    w /= np.linalg.norm(w, axis=-1, keepdims=True)
    return w.astype(np.float32).astype(np.float64)


def _f32(a3):
    return tuple(float(np.float32(v)) for v in (a3.ax, a3.ay, a3.az))


def _ndf_tol(wm, kind, a3):
    ax, ay, az = _f32(a3)
    lat = (wm[:, 0] / ax) ** 2 + (wm[:, 1] / ay) ** 2
    if kind is NdfKind.GENERALIZED:
        e = lat / az ** 2 / np.maximum(lat + (wm[:, 2] / az) ** 2, 1e-300)
    else:
        e = lat / np.maximum(wm[:, 2] ** 2, 1e-300)
    return np.maximum(1e-5, 8 * ULP * (1 + e))


@pytest.mark.parametrize("kind,a3", MEDIA)
def test_projected_area_lambda_ndf_vs_oracle(cuda, kind, a3):
    w = _dirs(1 << 16, 11)
    ax, ay, az = _f32(a3)
    k = kind.value
    m = parity.Obj(kind=k, a3=parity.Obj(ax=ax, ay=ay, az=az))
    ref = om.projected_area(w, k, ax, ay, az)
    got = curves.projected_area_dir(w, kind, a3)
    tol = 1e-5 + (parity.area_conditioning(w, m) if kind is not NdfKind.GGX else 0.0)
    res = parity.check_rel(got, ref, tol=tol, floor=1e-30)
    assert res["n_bad"] == 0, res
    ref_d = om.ndf(w, k, ax, ay, az)
    got_d = curves.ndf_dir(w, kind, a3)
    res = parity.check_rel(got_d, ref_d, tol=_ndf_tol(w, kind, a3), floor=1e-30)
    assert res["n_bad"] == 0, res
    if kind is not NdfKind.GGX:
        ok = np.abs(w[:, 2]) > 1e-3
        lam = curves.generalized_lambda_dir(w[ok], RoughnessTriple(a3.ax, a3.ay, a3.az))
        res = parity.check_rel(lam, om.projected_area_erf(w[ok], ax, ay, az) / w[ok, 2],
                               tol=np.asarray(tol)[ok] if np.ndim(tol) else tol, floor=1e-30)
        assert res["n_bad"] == 0, res


@pytest.mark.parametrize("kind,a3", MEDIA[:4])
def test_vndf_and_transmittance_vs_oracle(cuda, kind, a3):
    ax, ay, az = _f32(a3)
    k = kind.value
    m = parity.Obj(kind=k, a3=parity.Obj(ax=ax, ay=ay, az=az))
    wm = _dirs(1 << 15, 12)
    for inc in (10.0, 45.0, 80.0, 120.0):
        th = np.deg2rad(inc)
        wo = np.array([np.sin(th), 0.0, -np.cos(th)])
        wo32 = wo.astype(np.float32).astype(np.float64)
        got = curves.vndf_eval(wm, wo32, kind, a3)
        ref = om.vndf(wm, np.broadcast_to(wo32, wm.shape), k, ax, ay, az)
        # + the cancellation of the clamped cosine <-wo, wm> near the terminator
        cos = np.abs(wm @ wo32)
        tol = (_ndf_tol(wm, kind, a3) + parity.area_conditioning(wo32, m)
               + 4 * ULP / np.maximum(cos, 1e-30))
        res = parity.check_rel(got, ref, tol=tol, floor=1e-30)
        assert res["n_bad"] == 0, (inc, res)
    med = MacrofacetMedium(kind=kind, a3=a3, sigma=0.05, fresnel_one=True)
    mm = parity.f32_medium(med)
    for inc in (20.0, 60.0, 100.0, 160.0):
        th = np.deg2rad(inc)
        h0 = 0.02
        h1 = h0 + np.linspace(-0.3, 0.3, 257) * np.cos(th)
        h1 = h1.astype(np.float32).astype(np.float64)
        got = curves.planar_transmittance(h0, h1, th, 0.0, med)
        w = np.array([np.sin(th), 0.0, np.cos(th)])
        ref = om.planar_transmittance(h0, h1, np.cos(th), w, mm)
        # Tr = exp(-x): relative error ~ |x| times that of x
        x = np.abs(np.log(np.maximum(ref, 1e-300)))
        res = parity.check_rel(got, ref, tol=1e-5 * (1 + x), floor=1e-30)
        assert res["n_bad"] == 0, (inc, res)


def test_curve_errors(cuda):
    med = MacrofacetMedium(kind=NdfKind.GENERALIZED, a3=RoughnessTriple(1, 1, 1), sigma=1.0)
    with pytest.raises(UnsupportedGeometryError):
        curves.planar_transmittance(0.0, 1.0, np.pi / 2, 0.0, med)
    ggx = MacrofacetMedium(kind=NdfKind.GGX, a3=RoughnessTriple(1, 1, 0), sigma=1.0)
    with pytest.raises(UnsupportedGeometryError):
        curves.planar_transmittance(0.0, 1.0, 0.3, 0.0, ggx)
    with pytest.raises(GrazingSingularityError):
        curves.generalized_lambda(np.pi / 2, 0.0, RoughnessTriple(1, 1, 1))
    with pytest.raises(DegenerateVisibilityError):
        # upward view of a Beckmann height field: sigma(wo) == 0
        curves.vndf_eval(np.array([[0.0, 0.0, 1.0]]), np.array([0.0, 0.0, 1.0]),
                         NdfKind.BECKMANN, RoughnessTriple(0.1, 0.1, 0.0))


def test_validate_suites_pass(cuda):
    lines = []
    assert validate.run_suites(list(validate.SUITES), out=lines.append), "\n".join(lines)
    assert len(lines) == 15   # 13 + the two multiplicativity checks


def test_cli_curves_and_validate(cuda, tmp_path, capsys):
    out = tmp_path / "lam.csv"
    assert cli.main(["curves", "lambda", "--steps", "10", "--out", str(out)]) == 0
    text = out.read_text().splitlines()
    assert text[0].startswith("# macrofacet ") and text[1] == "# seed = 0"
    assert text[2].startswith("# params: ") and text[3] == "theta_deg,lambda_unitless"
    rows = np.array([[float(v) for v in r.split(",")] for r in text[4:]])
    assert rows.shape == (10, 2)
    ref = om.projected_area_erf(np.stack([np.sin(np.deg2rad(rows[:, 0])), 0 * rows[:, 0],
                                          np.cos(np.deg2rad(rows[:, 0]))], -1), 1, 1, 1) \
        / np.cos(np.deg2rad(rows[:, 0]))
    np.testing.assert_allclose(rows[:, 1], ref, rtol=1e-5)
    for kind in ("projected-area", "ndf", "vndf", "transmittance"):
        assert cli.main(["curves", kind, "--steps", "7", "--stop", "60",
                         "--out", str(tmp_path / f"{kind}.csv")]) == 0
    assert cli.main(["validate", "furnace"]) == 0
    assert cli.main(["validate", "furnace", "--tol", "white_furnace_mean=0"]) == 4
    assert cli.main(["validate", "nope"]) == 1
