"""The GP-realisation oracle on the device (paper_2603_00280_b200.gp,
csrc/mf_gp.cuh) against the reference's own outputs on the same streams
(tests/golden/gp_ref.npz from tests/golden/make_golden_gp.py): the noise is
drawn bit for bit, the FFT filtering agrees to float64 rounding (cuFFT vs
numpy), and every march / bisection decision follows, so hit flags,
transmittance rows, normal histograms and the multiplicativity counts are
identical and positions / radiances agree to ~1e-12."""

import numpy as np
import pytest

from paper_2603_00280_b200 import gp
from paper_2603_00280_b200.ndf import KernelParams
from paper_2603_00280_b200.rng import RandomStream
from paper_2603_00280_b200.scene import Camera

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    return np.load(f"{GOLDEN}/gp_ref.npz")


@pytest.fixture(scope="module")
def kernel(ref):
    s, lx, ly, lz = ref["kernel"]
    return KernelParams(sigma=float(s), lx=float(lx), ly=float(ly), lz=float(lz))


@pytest.fixture(scope="module")
def real(cuda, kernel):
    return gp.realize_gp(kernel, "planar", None, RandomStream(11))


def test_realisation_field_and_gradient(real, ref):
    g = real.grid
    assert g.shape == (int(ref["grid_n"]),) * 3
    scale = np.sqrt(ref["grid_sumsq"] / g.size)
    np.testing.assert_allclose(g[3], ref["grid_slice"], rtol=0, atol=1e-12 * scale)
    assert abs(g.sum() - ref["grid_sum"]) <= 1e-9 * scale * g.size ** 0.5
    np.testing.assert_allclose(real.field_at(ref["probes"]), ref["field"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(real.gradient_at(ref["probes"]), ref["gradient"], rtol=0,
                               atol=1e-10)


def test_first_hit(real, ref):
    fh = gp.first_hit(real, ref["fh_o"], ref["fh_d"], 1.2)
    assert np.array_equal(fh.hit, ref["fh_hit"])
    assert fh.hit.any() and not fh.hit.all()
    h = fh.hit
    np.testing.assert_allclose(fh.travel[h], ref["fh_travel"][h], rtol=0, atol=1e-11)
    assert np.all(np.isinf(fh.travel[~h]))
    np.testing.assert_allclose(fh.position, ref["fh_pos"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(fh.normal, ref["fh_normal"], rtol=0, atol=1e-8)


def test_empirical_transmittance(cuda, kernel, ref):
    rows = np.array(gp.empirical_transmittance(kernel, 0.1, 0.8, 0.3, np.linspace(0.0, 1.0, 9),
                                               64, RandomStream(12)))
    np.testing.assert_array_equal(rows, ref["tr_rows"])


def test_empirical_vndf(cuda, kernel, ref):
    dens, (te, pe) = gp.empirical_vndf(kernel, (0.3, 0.0, -1.0), 6, 8, 8, RandomStream(13),
                                       rays_per_realization=64)
    np.testing.assert_allclose(dens, ref["vndf"], rtol=1e-12, atol=0)
    assert te.shape == (7,) and pe.shape == (9,)


def test_multiplicativity_probe(cuda, kernel, ref):
    got = np.array(gp.multiplicativity_probe(kernel, (0.0, 0.0, 0.15), (0.5, 0.0, -1.0), 0.2,
                                             0.5, 256, RandomStream(14), n_boot=200))
    np.testing.assert_allclose(got, ref["mult"], rtol=1e-12, atol=1e-15)


def test_ensemble_radiance(cuda, kernel, ref):
    cam = Camera(position=(0.0, -1.0, 1.0), look_at=(0.0, 0.0, 0.0), fov_deg=30.0, width=8,
                 height=6)
    img = gp.ensemble_radiance(kernel, cam, 3, 3, RandomStream(15), env_radiance=1.0,
                               fresnel=((0.2, 0.3, 0.4), (3.0, 3.1, 3.2)), max_bounces=8)
    assert img.shape == (6, 8, 3)
    np.testing.assert_allclose(img, ref["ensemble"], rtol=1e-10, atol=1e-12)


def test_desk_scale_limits(cuda, kernel):
    from paper_2603_00280_b200.errors import ConfigError, ParameterDomainError

    with pytest.raises(ConfigError):
        gp.ensemble_radiance(kernel, Camera((0, -1, 1), (0, 0, 0), 30.0, 65, 64), 1, 1,
                             RandomStream(1))
    with pytest.raises(ParameterDomainError):
        gp.empirical_transmittance(kernel, 0.1, 0.5, 0.0, [0.1], 10, RandomStream(1))
    with pytest.raises(ParameterDomainError):
        gp.realize_gp(kernel, "sphere", None, RandomStream(1))


def test_cli_oracle(cuda, tmp_path):
    """`oracle` subcommand (cli.py:193-265) on the device: CSV / PFM outputs
    and the reference's caps."""
    from paper_2603_00280_b200 import cli
    from paper_2603_00280_b200.image import read_pfm

    out = tmp_path / "tr.csv"
    assert cli.main(["oracle", "gp-transmittance", "--realizations", "64", "--steps", "5",
                     "--t-max", "0.5", "--z0", "0.05", "--out", str(out)]) == 0
    rows = [l for l in out.read_text().splitlines() if l and not l.startswith("#")]
    assert rows[0].startswith("t_world") and len(rows) == 6
    vals = np.array([[float(x) for x in r.split(",")] for r in rows[1:]])
    assert vals[0, 1] == 1.0 and np.all(np.diff(vals[:, 1]) <= 0)
    pfm = tmp_path / "ens.pfm"
    assert cli.main(["oracle", "gp-ensemble", "--realizations", "4", "--spp", "2", "--width",
                     "8", "--height", "8", "--out", str(pfm)]) == 0
    img = read_pfm(pfm)
    assert img.pixels.shape == (8, 8, 3) and np.all(np.isfinite(img.pixels))
    assert cli.main(["oracle", "gp-vndf", "--realizations", "5000", "--out",
                     str(tmp_path / "v.csv")]) == 1


def test_validate_multiplicativity(cuda):
    from paper_2603_00280_b200 import validate

    lines = []
    assert validate.run_suites(["multiplicativity"], out=lines.append), lines
