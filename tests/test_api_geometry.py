"""Host geometry of the scene description (CPU only): the SDF objects'
sdf / gradient (sdf.py:18-84) and shell_intersect (scene.py:132-200)
against closed forms."""

import numpy as np

import paper_2603_00280_b200 as mf


def test_sdf_methods():
    p = np.array([[0.3, -0.2, 0.5], [2.0, 0.0, 0.0], [0.0, 0.0, -0.1]])
    assert np.allclose(mf.Plane(0.1).sdf(p), p[:, 2] - 0.1)
    assert np.allclose(mf.Plane(0.1).gradient(p), [[0, 0, 1]] * 3)
    s = mf.Sphere((0.0, 0.0, 0.0), 1.0)
    assert np.allclose(s.sdf(p), np.linalg.norm(p, axis=1) - 1.0)
    assert np.allclose(s.gradient(p[1]), [1.0, 0.0, 0.0])
    b = mf.Box((0.0, 0.0, 0.0), (1.0, 0.5, 0.25))
    assert np.isclose(b.sdf([2.0, 0.0, 0.0]), 1.0)
    assert np.isclose(b.sdf([0.0, 0.0, 0.0]), -0.25)
    assert np.isclose(b.sdf([2.0, 1.5, 0.0]), np.hypot(1.0, 1.0))
    assert np.allclose(b.gradient([0.0, 0.0, 0.1]), [0, 0, 1])
    assert np.allclose(b.gradient([3.0, 0.0, 0.0]), [1, 0, 0])


def test_shell_intersect_sphere_and_plane():
    med = mf.MacrofacetMedium(kind=mf.NdfKind.GENERALIZED, a3=mf.RoughnessTriple(1.0, 1.0, 1.0),
                              sigma=0.05)
    cam = mf.Camera((0, -4, 0), (0, 0, 0), 40.0, 4, 4)
    sc = mf.ShellScene(primitives=(mf.ShellPrimitive(mf.Sphere((0, 0, 0), 1.0), med),),
                       camera=cam)
    iv, deep = mf.shell_intersect([0.0, -4.0, 0.0], [0.0, 1.0, 0.0], sc)
    # the shell |r - 1| <= 0.15 entered at 2.85 and left into the core at
    # 3.15 (deep); past the centre the ray recedes from the sphere and the
    # march ends, as the reference's recede test does (scene.py:185-190)
    assert deep and len(iv) == 1 and iv[0][2] == 0
    np.testing.assert_allclose(iv[0][:2], [2.85, 3.15], atol=1e-9)
    iv, deep = mf.shell_intersect([0.0, -4.0, 2.0], [0.0, 1.0, 0.0], sc)
    assert iv == [] and not deep
    pl = mf.ShellScene(primitives=(mf.ShellPrimitive(mf.Plane(0.0), med),), camera=cam)
    d = np.array([0.6, 0.0, -0.8])
    iv, deep = mf.shell_intersect([0.0, 0.0, 1.0], d, pl, t_max=10.0)
    np.testing.assert_allclose([iv[0][0], iv[0][1]], [0.85 / 0.8, 1.15 / 0.8], atol=1e-9)
    assert deep and len(iv) == 1
