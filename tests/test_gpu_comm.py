"""The library's NCCL communicator (C ABI mf_comm_* / mf_reduce) on one GPU:
a one-rank communicator, both reduce modes, render_sharded through it, and
the error statuses.  The N > 1 host logic is covered with gloo in
test_dist_cpu.py (the GPU box has a single GPU)."""

import pytest
import torch
import torch.distributed as dist

import paper_2603_00280_b200 as mf
from paper_2603_00280_b200 import _lib, configs
from paper_2603_00280_b200.comm import NcclComm
from paper_2603_00280_b200.errors import ParameterDomainError

pytestmark = pytest.mark.gpu


@pytest.fixture
def group(cuda, tmp_path):
    dist.init_process_group("gloo", init_method=f"file://{tmp_path}/store", rank=0, world_size=1)
    yield None
    dist.destroy_process_group()


def test_reduce_modes_one_rank(group):
    with NcclComm() as comm:
        assert comm.nranks == 1 and comm.rank == 0 and comm.handle
        x = torch.randn(3 * 1000 + 7, device="cuda")
        ref = x.clone()
        comm.reduce(x, root=0)
        torch.cuda.synchronize()
        assert torch.equal(x, ref)
        comm.reduce(x, root=0, ordered=True)
        torch.cuda.synchronize()
        assert torch.equal(x, ref)
        with pytest.raises(ParameterDomainError):
            comm.reduce(x, root=1)
        with pytest.raises(ParameterDomainError):
            comm.reduce(x.double())
        lib = _lib.load()
        with pytest.raises(ParameterDomainError):
            _lib.check(lib.mf_reduce(_lib.ctypes.c_void_p(comm.handle),
                                     _lib.ctypes.c_void_p(x.data_ptr()), x.numel(), 0, 7,
                                     _lib.stream_handle(torch)))


def test_render_sharded_through_library_comm(group):
    scene = configs.config2_scene(64, 48)
    ref, _ = mf.render_device(scene, 8, 5, max_bounces=8)
    with NcclComm() as comm:
        for ordered in (False, True):
            img, st = mf.render_sharded(scene, 8, 5, max_bounces=8, shard="samples", comm=comm,
                                        ordered=ordered, stats=True)
            torch.cuda.synchronize()
            assert torch.equal(img, ref)
            assert st["paths"] == 64 * 48 * 8
