"""The N > 1 path with the REAL kernels: two processes
(gloo, world size 2) each render their share of a config-4 panel with
mf_render on cuda:0 -- the box has one GPU, and the ranks' kernels never
wait on each other -- and combine the per-rank fp32 buffers the way
render_sharded does: one sum onto rank 0 (tile sharding: exact, so the
image is bit-identical to the one-rank render) or the rank-order sum of
MF_REDUCE_ORDERED (sample sharding: reproducible for a fixed rank count).
Plus the tile-shard emulation of N = 2, 4, 8 on config 4."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import configs

pytestmark = pytest.mark.gpu

W, H, SPP, SEED, DEPTH = 96, 64, 64, 3, 64


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene():
    return configs.config4_scene(0.05, 0.1, W, H)


class _GlooDeviceComm:
    """render_sharded's `comm` interface over gloo for CUDA tensors: the
    buffer goes to the host, rank 0 receives every rank's buffer and sums
    them in rank order (MF_REDUCE_ORDERED) or lets gloo sum them (the
    plain reduce), and the result is copied back."""

    def __init__(self):
        self.rank, self.nranks = dist.get_rank(), dist.get_world_size()

    def reduce(self, t, root=0, ordered=False):
        h = t.cpu()
        if ordered:
            parts = [torch.empty_like(h) for _ in range(self.nranks)]
            dist.all_gather(parts, h)
            acc = parts[0].clone()
            for p in parts[1:]:
                acc += p
        else:
            dist.reduce(h, dst=root, op=dist.ReduceOp.SUM)
            acc = h
        if self.rank == root:
            t.copy_(acc.to(t.device))
        return t


def _worker(rank, world, port, shard, ordered, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = _GlooDeviceComm()
    img, st = mf.render_sharded(_scene(), SPP, SEED, max_bounces=DEPTH, tile=16, shard=shard,
                                comm=comm, ordered=ordered, stats=True)
    torch.cuda.synchronize()
    q.put((rank, img.cpu().numpy().copy(), st["paths"]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("shard,ordered", [("tiles", False), ("samples", True)])
def test_two_ranks_real_kernels(cuda, shard, ordered):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shard, ordered, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, (img, n)) for r, img, n in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # every path rendered exactly once across the two ranks
    assert got[0][1] + got[1][1] == W * H * SPP
    full, _ = mf.render_device(_scene(), SPP, SEED, max_bounces=DEPTH, tile=16)
    full = full.cpu().numpy()
    img = got[0][0]
    if shard == "tiles":
        assert np.array_equal(img, full)      # disjoint tiles: exact, any rank count
    else:
        # rank-order sum of the two sample halves, reproduced here bit for bit
        parts = [mf.render_device(_scene(), SPP, SEED, max_bounces=DEPTH, rank=r, nranks=2,
                                  shard="samples")[0].cpu().numpy() for r in range(2)]
        assert np.array_equal(img, parts[0] + parts[1])
        np.testing.assert_allclose(img, full, rtol=2e-6, atol=1e-7)


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_config4_tile_sharding_is_exact(cuda, nranks):
    """The 1/2/4/8-GPU config-4 bench split (32x32 tiles, one sum) emulated
    shard by shard on one GPU: bit-identical to the one-rank panel."""
    sc = configs.config4_scene(0.2, 0.02, 256, 128)
    full, _ = mf.render_device(sc, 32, SEED, max_bounces=DEPTH, tile=32)
    full = full.clone()
    acc = torch.zeros_like(full)
    for r in range(nranks):
        part, st = mf.render_device(sc, 32, SEED, max_bounces=DEPTH, tile=32, rank=r,
                                    nranks=nranks, stats=True)
        assert st["paths"] == 256 * 128 * 32 // nranks
        acc += part
    assert torch.equal(acc, full)
