"""Config schema and CLI (CPU only; rendering itself is covered on the GPU)."""

import math

import pytest

import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import cli, configs
from paper_2603_00280_b200.config import (config_hash, parse_config, scene_from_config,
                                          serialize_config)

from conftest import ROOT


def test_config_round_trip_and_errors():
    text = open(f"{ROOT}/configs/config2.cfg").read()
    v = parse_config(text)
    assert parse_config(serialize_config(v)) == v
    assert len(config_hash(v)) == 16
    with pytest.raises(mf.ConfigError):
        parse_config("[kernel]\nsigma = 1\nlx = 1\nax = 1\n")      # config.py:102-106
    with pytest.raises(mf.ConfigError):
        parse_config("[nope]\n")
    with pytest.raises(mf.ConfigError):
        parse_config("[render]\nwidth = 1\nwidth = 2\n")
    with pytest.raises(mf.ConfigError):
        parse_config("[scene]\nprimitive0_colour = red\n")


def test_configs_match_the_baseline_scenes():
    s2 = scene_from_config(parse_config(open(f"{ROOT}/configs/config2.cfg").read()))
    ref2 = configs.config2_scene()
    assert s2.camera.ortho and s2.camera.width == 256
    for a, b in zip(s2.camera.position, ref2.camera.position):
        assert abs(a - b) < 1e-12
    m2, r2 = s2.primitives[0].medium, ref2.primitives[0].medium
    assert m2.kind == r2.kind and abs(m2.a3.ax - r2.a3.ax) < 1e-15 and m2.albedo == r2.albedo
    for a, b in zip(s2.sun.direction, ref2.sun.direction):
        assert abs(a - b) < 1e-12
    s3 = scene_from_config(parse_config(open(f"{ROOT}/configs/config3.cfg").read()))
    assert isinstance(s3.primitives[0].sdf, mf.Sphere) and s3.point.intensity == (10.0,) * 3
    lz_inf = parse_config("[kernel]\nsigma = 0.05\nlx = 0.05\nly = 0.05\nlz = inf\n")
    m = scene_from_config(lz_inf).primitives[0].medium
    assert m.kind is mf.NdfKind.BECKMANN and m.a3.az == 0.0
    assert abs(m.a3.ax - math.sqrt(2)) < 1e-12


def test_config_box_and_env_map(tmp_path):
    """Box shells and lat-long PFM environments (reference config.py:207-227)."""
    import numpy as np

    px = np.arange(4 * 8 * 3, dtype=np.float32).reshape(4, 8, 3)
    mf.write_pfm(mf.RadianceImage(px), str(tmp_path / "env.pfm"))
    text = ("[kernel]\nsigma = 0.05\nlx = 0.05\nly = 0.05\nlz = 0.1\n"
            f"[scene]\nenv_map = {tmp_path / 'env.pfm'}\n"
            "primitive0_shape = box\nprimitive0_center = 0,1,2\n"
            "primitive0_half_extents = 1,2,0.5\n")
    sc = scene_from_config(parse_config(text))
    box = sc.primitives[0].sdf
    assert isinstance(box, mf.Box)
    assert box.center == (0.0, 1.0, 2.0) and box.half_extents == (1.0, 2.0, 0.5)
    assert np.array_equal(sc.environment.latlong, px)
    with pytest.raises(mf.IoError):
        scene_from_config(parse_config(f"[scene]\nenv_map = {tmp_path / 'missing.pfm'}\n"))


def test_cli_exit_codes(tmp_path, capsys):
    # cli.py:324-343 exit codes: config error 1, I/O error 3
    bad = tmp_path / "bad.cfg"
    bad.write_text("[kernel]\nnonsense = 1\n")
    assert cli.main(["render", str(bad), "--out", str(tmp_path / "x.pfm")]) == 1
    assert cli.main(["render", str(tmp_path / "missing.cfg"), "--out", "x.pfm"]) == 3
    assert cli.main(["bogus"]) == 1


def test_cli_curves_validate_host_paths(tmp_path, capsys):
    """Argument errors and the CSV layout need no GPU; without a device the
    compute subcommands fail loudly (no CPU fallback) with exit code 2."""
    from paper_2603_00280_b200 import cli

    assert cli.main(["validate", "nope"]) == 1
    assert cli.main(["validate", "all", "--tol", "x"]) == 1
    assert cli.main(["curves", "bogus", "--out", str(tmp_path / "x.csv")]) == 1
    out = tmp_path / "t.csv"
    cli.write_csv(str(out), ["a", "b"], [(0.1, 1.0 / 3.0)], {"z": 1, "k": "lambda"}, seed=7)
    lines = out.read_text().splitlines()
    assert lines[1:] == ["# seed = 7", "# params: k=lambda z=1", "a,b",
                         "0.10000000000000001,0.33333333333333331"]
    import torch

    if not torch.cuda.is_available():
        assert cli.main(["curves", "lambda", "--out", str(tmp_path / "l.csv")]) == 2
