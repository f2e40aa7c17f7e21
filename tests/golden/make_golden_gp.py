"""Golden fixtures of the Gaussian-random-field oracle (reference gp.py) by
running the REFERENCE package (/root/reference/pkg/src, importable only in
the build container):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_gp.py

Output (committed; the GPU box never reads /root/reference): gp_ref.npz with
  - a planar realisation (kernel sigma 0.05, l = 0.1 / 0.1 / 0.08; seed 11):
    grid checksum and a slice, field_at / gradient_at at 256 probes;
  - first_hit of 256 rays through it;
  - empirical_transmittance (64 realisations, seed 12);
  - empirical_vndf (8 realisations x 64 rays, seed 13);
  - multiplicativity_probe (256 realisations, 200 bootstrap draws, seed 14);
  - ensemble_radiance (8 x 6 pixels, 3 rounds, conductor Fresnel, seed 15);
  - RandomStream(16, 3).normal(7) and the counter after it.
tests/test_gpu_gp.py compares the device oracle with these.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from macrofacet import gp  # noqa: E402
from macrofacet.ndf import KernelParams  # noqa: E402
from macrofacet.rng import RandomStream  # noqa: E402
from macrofacet.scene import Camera  # noqa: E402

KERNEL = dict(sigma=0.05, lx=0.1, ly=0.1, lz=0.08)


def main():
    k = KernelParams(**KERNEL)
    out = {"kernel": np.array([k.sigma, k.lx, k.ly, k.lz])}
    real = gp.realize_gp(k, "planar", None, RandomStream(11))
    out["grid_n"] = np.array(real.spec.n)
    out["grid_sum"] = np.array(real.grid.sum())
    out["grid_sumsq"] = np.array((real.grid ** 2).sum())
    out["grid_slice"] = real.grid[3, :, :].copy()
    ps = np.random.default_rng(5)
    probes = ps.uniform(-0.6, 0.6, (256, 3))
    probes[:, 2] *= 0.3
    out["probes"] = probes
    out["field"] = real.field_at(probes)
    out["gradient"] = real.gradient_at(probes)
    o = np.column_stack([ps.uniform(-0.3, 0.3, 256), ps.uniform(-0.3, 0.3, 256),
                         np.full(256, 0.25)])
    d = ps.normal(size=(256, 3))
    d[:, 2] = -np.abs(d[:, 2]) - 0.2
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    fh = gp.first_hit(real, o, d, 1.2)
    out.update(fh_o=o, fh_d=d, fh_hit=fh.hit, fh_pos=fh.position, fh_normal=fh.normal,
               fh_travel=fh.travel)
    out["tr_rows"] = np.array(gp.empirical_transmittance(
        k, 0.1, 0.8, 0.3, np.linspace(0.0, 1.0, 9), 64, RandomStream(12)))
    dens, _ = gp.empirical_vndf(k, (0.3, 0.0, -1.0), 6, 8, 8, RandomStream(13),
                                rays_per_realization=64)
    out["vndf"] = dens
    out["mult"] = np.array(gp.multiplicativity_probe(
        k, (0.0, 0.0, 0.15), (0.5, 0.0, -1.0), 0.2, 0.5, 256, RandomStream(14), n_boot=200))
    cam = Camera(position=(0.0, -1.0, 1.0), look_at=(0.0, 0.0, 0.0), fov_deg=30.0, width=8,
                 height=6)
    out["ensemble"] = gp.ensemble_radiance(k, cam, 3, 3, RandomStream(15), env_radiance=1.0,
                                           fresnel=((0.2, 0.3, 0.4), (3.0, 3.1, 3.2)),
                                           max_bounces=8)
    rs = RandomStream(16, 3)
    out["normals"] = rs.normal((7,))
    out["normals_counter"] = np.array(rs.counter)
    np.savez_compressed(os.path.join(HERE, "gp_ref.npz"), **out)
    print({k: np.asarray(v).shape for k, v in out.items()})


if __name__ == "__main__":
    main()
