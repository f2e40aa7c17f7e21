"""GP-realisation oracle, host side (CPU only): grid rules and the
reference's normal stream (rng.py:87-97) against the golden fixture."""

import numpy as np
import pytest

from paper_2603_00280_b200 import gp
from paper_2603_00280_b200.errors import ConfigError
from paper_2603_00280_b200.ndf import KernelParams
from paper_2603_00280_b200.rng import RandomStream

from conftest import GOLDEN


def test_default_grid_and_validation():
    k = KernelParams(sigma=0.05, lx=0.1, ly=0.1, lz=0.08)
    spec = gp.default_grid(k)
    ref = np.load(f"{GOLDEN}/gp_ref.npz")
    assert spec.n == int(ref["grid_n"]) and spec.n % 2 == 0
    assert spec.spacing == 0.02 and spec.origin == -0.5 * spec.extent
    with pytest.raises(ConfigError, match="extent"):
        gp._validate_grid(k, gp.GridSpec(n=8, spacing=0.02))
    with pytest.raises(ConfigError, match="spacing"):
        gp._validate_grid(k, gp.GridSpec(n=64, spacing=0.03))


def test_normal_stream_matches_reference():
    ref = np.load(f"{GOLDEN}/gp_ref.npz")
    rs = RandomStream(16, 3)
    z = rs.normal((7,))
    np.testing.assert_allclose(z, ref["normals"], rtol=1e-15, atol=0)
    assert rs.counter == int(ref["normals_counter"])
    assert gp._noise_draws(7) == int(ref["normals_counter"])
