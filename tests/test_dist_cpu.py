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


class _GlooOrderedComm:
    """Stand-in for comm.NcclComm with mf_reduce's MF_REDUCE_ORDERED
    semantics (root sums the ranks' buffers in rank order) over gloo."""

    def __init__(self):
        self.rank, self.nranks = dist.get_rank(), dist.get_world_size()
        self.calls = []

    def reduce(self, t, root=0, ordered=False):
        self.calls.append(ordered)
        parts = [torch.empty_like(t) for _ in range(self.nranks)]
        dist.all_gather(parts, t)
        if self.rank == root:
            acc = parts[0].clone()
            for p in parts[1:]:
                acc += p
            t.copy_(acc)
        return t


def _worker(rank, world, port, shard, q, ordered=False):
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
    comm = _GlooOrderedComm() if ordered else None
    img, _ = R.render_sharded(scene, 8, 1, tile=8, shard=shard, comm=comm, ordered=ordered)
    if rank == 0:
        q.put(img.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("shard,ordered", [("tiles", False), ("samples", False),
                                           ("samples", True)])
def test_render_sharded_gloo_world2(shard, ordered):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shard, q, ordered))
             for r in range(2)]
    for p in procs:
        p.start()
    img = q.get(timeout=90)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    full = _fake_pixels(40, 24).reshape(24, 40, 3)
    if shard == "tiles":
        assert np.array_equal(img, full)  # disjoint tiles: the reduce is exact
    elif ordered:
        # rank-order sum of the two halves, bit for bit
        b0, e0 = R.sample_range(8, 0, 2)
        b1, e1 = R.sample_range(8, 1, 2)
        want = full * np.float32((e0 - b0) / 8) + full * np.float32((e1 - b1) / 8)
        assert np.array_equal(img, want.astype(np.float32))
    else:
        np.testing.assert_allclose(img, full, rtol=1e-6, atol=1e-7)


def test_sample_ranges_partition():
    for spp in (1, 7, 64, 4096):
        for n in (1, 2, 3, 8):
            rs = [R.sample_range(spp, r, n) for r in range(n)]
            assert rs[0][0] == 0 and rs[-1][1] == spp
            assert all(rs[i][1] == rs[i + 1][0] for i in range(n - 1))


def _uid_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_00280_b200 import _lib, comm

    uid = comm.exchange_unique_id(_lib.load())
    q.put((rank, bytes(uid)))
    dist.barrier()
    dist.destroy_process_group()


def test_comm_unique_id_exchange_gloo_world2():
    """NcclComm's unique-id exchange: rank 0 creates it through the C ABI
    (mf_comm_unique_id, NCCL resolved at run time), both ranks hold it."""
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_uid_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=90) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got[0] == got[1] and len(got[0]) == 128 and any(got[0])
