"""The N > 1 host path on CPU with gloo, world_size 2 (the GPU box used by
this build has one GPU): render_sharded's single sum-reduce of per-rank
accumulation buffers, with the kernel replaced by a deterministic stand-in
that writes each rank's owned pixels exactly like mf_render does."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import importlib

from paper_2603_00280_b200 import configs

R = importlib.import_module("paper_2603_00280_b200.render")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_pixels(w, h):
    # stand-in radiance: any deterministic function of the pixel index
    idx = np.arange(w * h, dtype=np.float64)
    return np.stack([np.sin(idx), np.cos(idx) ** 2, idx / (w * h)], axis=-1).astype(np.float32)


def _worker(rank, world, port, shard, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scene = configs.config2_scene(40, 24)
    w, h = scene.camera.width, scene.camera.height
    full = _fake_pixels(w, h)

    def fake_render_device(scene, spp, seed, max_bounces=64, tile=32, rank=0, nranks=1,
                           shard="tiles", out=None, stats=False, stream=None, c_scene=None):
        img = np.zeros((h * w, 3), np.float32)
        if shard == "tiles":
            px = R.owned_pixels(w, h, tile, rank, nranks)
            img[px] = full[px]
        else:
            b, e = R.sample_range(spp, rank, nranks)
            img[:] = full * np.float32((e - b) / spp)
        return torch.from_numpy(img.reshape(h, w, 3)), ({"paths": 1} if stats else None)

    R.render_device = fake_render_device
    img, _ = R.render_sharded(scene, 8, 1, tile=8, shard=shard)
    if rank == 0:
        q.put(img.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("shard", ["tiles", "samples"])
def test_render_sharded_gloo_world2(shard):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shard, q)) for r in range(2)]
    for p in procs:
        p.start()
    img = q.get(timeout=90)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    full = _fake_pixels(40, 24).reshape(24, 40, 3)
    if shard == "tiles":
        assert np.array_equal(img, full)  # disjoint tiles: the reduce is exact
    else:
        np.testing.assert_allclose(img, full, rtol=1e-6, atol=1e-7)


def test_sample_ranges_partition():
    for spp in (1, 7, 64, 4096):
        for n in (1, 2, 3, 8):
            rs = [R.sample_range(spp, r, n) for r in range(n)]
            assert rs[0][0] == 0 and rs[-1][1] == spp
            assert all(rs[i][1] == rs[i + 1][0] for i in range(n - 1))
