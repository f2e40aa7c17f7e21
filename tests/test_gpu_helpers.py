"""The reference's remaining public helpers of the path (its __init__
exports), device-backed, against the float64 oracle: density, conductor
Fresnel, the Beckmann / GGX NDFs, the gradient density, the float64
special functions and vndf_sample (the sampler's pdf is the exact mixture
density of the returned normal)."""

import math

import numpy as np
import pytest

import paper_2603_00280_b200 as mf
from oracle import microfacet as om
from oracle import numerics as on

pytestmark = pytest.mark.gpu


def test_density_and_fresnel(cuda):
    f = np.linspace(-0.3, 0.15, 301)
    got = mf.density(f, 0.05)
    ref = om.density(f, 0.05)
    np.testing.assert_allclose(got, ref, rtol=2e-6)
    c = np.linspace(0.0, 1.0, 101)
    got = mf.fresnel_conductor(c, 0.2, 3.0)
    np.testing.assert_allclose(got, om.fresnel_conductor(c, 0.2, 3.0), rtol=2e-6, atol=1e-7)
    rgb = mf.fresnel_conductor(0.5, np.array([0.2, 1.1, 1.5]), np.array([3.0, 2.5, 2.0]))
    assert rgb.shape == (3,)
    np.testing.assert_allclose(rgb, [om.fresnel_conductor(0.5, e, k) for e, k in
                                     ((0.2, 3.0), (1.1, 2.5), (1.5, 2.0))], rtol=2e-6)
    with pytest.raises(mf.ParameterDomainError):
        mf.density(f, 0.0)


def test_ndfs_and_gdf(cuda):
    rs = np.random.default_rng(3)
    wm = rs.normal(size=(512, 3))
    wm[:, 2] = np.abs(wm[:, 2])
    wm /= np.linalg.norm(wm, axis=1, keepdims=True)
    np.testing.assert_allclose(mf.beckmann_ndf(wm, 0.4, 0.6), om.beckmann_d(wm, 0.4, 0.6),
                               rtol=1e-5, atol=1e-12)
    np.testing.assert_allclose(mf.ggx_ndf(wm, 0.4, 0.6), om.ggx_d(wm, 0.4, 0.6), rtol=1e-5)
    a3 = mf.RoughnessTriple(0.5, 0.7, 0.3)
    g = rs.normal(size=(512, 3)) * 0.4 + [0, 0, 1]
    e = (g[:, 0] / 0.5) ** 2 + (g[:, 1] / 0.7) ** 2 + ((g[:, 2] - 1) / 0.3) ** 2
    ref = np.exp(-e) / (math.pi ** 1.5 * 0.5 * 0.7 * 0.3)
    np.testing.assert_allclose(mf.gdf_pdf(g, a3), ref, rtol=2e-5, atol=1e-30)
    with pytest.raises(mf.ParameterDomainError):
        mf.gdf_pdf(g, mf.RoughnessTriple(0.5, 0.5, 0.0))
    s = mf.sample_gdf(a3, mf.RandomStream(4), 20000)
    np.testing.assert_allclose(s.mean(axis=0), [0, 0, 1], atol=0.02)
    np.testing.assert_allclose(s.std(axis=0), [0.5 / 2 ** 0.5, 0.7 / 2 ** 0.5, 0.3 / 2 ** 0.5],
                               rtol=0.03)


def test_float64_special_functions(cuda):
    x = np.linspace(-6.0, 6.0, 2001)
    assert np.max(np.abs(mf.erf(x) + mf.erfc(x) - 1.0)) < 1e-14
    assert np.array_equal(mf.erf(-x), -mf.erf(x))
    np.testing.assert_allclose(mf.erfc(np.array([5.0, 10.0, 20.0])),
                               on.erfc(np.array([5.0, 10.0, 20.0])), rtol=1e-13)
    np.testing.assert_allclose(mf.gauss_cdf(x, 0.3, 2.0), on.gauss_cdf(x - 0.3, 2.0), rtol=1e-13)
    np.testing.assert_allclose(mf.gauss_pdf(x, 0.3, 2.0), on.gauss_pdf(x - 0.3, 2.0), rtol=1e-13)
    th, ph = mf.direction_to_spherical(mf.spherical_to_direction(0.7, 2.1))
    assert abs(th - 0.7) < 1e-12 and abs(ph - 2.1) < 1e-12
    v, n = np.array([0.3, 0.4, 0.866]), np.array([0.0, 0.0, 1.0])
    np.testing.assert_allclose(mf.reflect(v, n), [-0.3, -0.4, 0.866])


def test_vndf_sample(cuda):
    a3 = mf.RoughnessTriple(0.6, 0.6, 0.4)
    wo = np.array([0.5, 0.1, -0.86])
    wo /= np.linalg.norm(wo)
    wm, pdf = mf.vndf_sample(wo, mf.NdfKind.GENERALIZED, a3, 0.5, mf.RandomStream(7), n=4096)
    assert wm.shape == (4096, 3) and pdf.shape == (4096,)
    np.testing.assert_allclose(np.linalg.norm(wm, axis=1), 1.0, atol=1e-6)
    ref = om.mixture_pdf(wm, np.broadcast_to(wo, wm.shape), 0.6, 0.6, 0.5)
    np.testing.assert_allclose(pdf, ref, rtol=5e-5)
    # the unbiased weight vndf / pdf integrates to one
    w = om.vndf(wm, np.broadcast_to(wo, wm.shape), "generalized", 0.6, 0.6, 0.4) / pdf
    assert abs(w.mean() - 1.0) < 4 * w.std() / np.sqrt(len(w))


def test_ndf_from_gdf_quadrature(cuda):
    """The radial quadrature (ndf.py:254-293) on the device in float64: the
    reference suite's pinned value at the pole for alpha = 1 (test_ndf.py:
    170-177) and agreement with the closed-form generalized NDF."""
    iso1 = mf.RoughnessTriple(1.0, 1.0, 1.0)
    assert abs(mf.ndf_from_gdf_quadrature(0.0, 0.0, iso1) - 0.7992537597222495) < 1e-10
    a3 = mf.RoughnessTriple(0.8, 0.5, 0.3)
    for th, ph in ((0.3, 0.2), (1.2, 2.0), (2.5, 4.0)):
        q = mf.ndf_from_gdf_quadrature(th, ph, a3)
        d = float(mf.generalized_ndf(th, ph, a3))
        assert abs(d / q - 1.0) < 2e-5, (th, ph, q, d)
    with pytest.raises(mf.ParameterDomainError):
        mf.ndf_from_gdf_quadrature(0.1, 0.0, mf.RoughnessTriple(1.0, 1.0, 0.0))
