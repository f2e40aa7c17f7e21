"""NCCL communicator of the library (C ABI mf_comm_* / mf_reduce).

The reference has no multi-process path: `render()` joins a thread pool
over tiles (render.py:168-176).  Across GPUs that join becomes one sum of
the per-rank fp32 accumulation buffers onto rank 0.
`render_sharded` can run it through torch.distributed or through the
library's own communicator here:

    comm = NcclComm()                   # collective over the default group
    comm.reduce(img, root=0)            # in-place ncclReduce(sum)
    comm.reduce(img, root=0, ordered=True)   # rank-order sum, reproducible
    comm.close()

The unique id is created by rank 0 (`mf_comm_unique_id`) and broadcast
through the torch.distributed group (any backend); every rank must have
selected its CUDA device first.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .errors import ParameterDomainError


class NcclComm:
    def __init__(self, group=None):
        import torch.distributed as dist

        torch = _lib.require_cuda()
        self._lib = _lib.load()
        self.group = group
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        dev = torch.device("cuda", torch.cuda.current_device())
        uid = exchange_unique_id(self._lib, group, dev)
        handle = ctypes.c_void_p()
        _lib.check(self._lib.mf_comm_init(uid, self.nranks, self.rank, ctypes.byref(handle)))
        self._handle = handle

    @property
    def handle(self):
        """The ncclComm_t (as an integer) -- usable by other NCCL callers."""
        if self._handle is None:
            raise ParameterDomainError("communicator is closed")
        return self._handle.value

    def reduce(self, tensor, root=0, ordered=False, stream=None):
        """Sum `tensor` (contiguous float32 CUDA) over ranks onto `root`, in
        place, on `stream` (default: the current stream)."""
        torch = _lib.require_cuda()
        if tensor.dtype != torch.float32 or not tensor.is_cuda or not tensor.is_contiguous():
            raise ParameterDomainError("reduce needs a contiguous float32 CUDA tensor")
        s = stream if stream is not None else _lib.stream_handle(torch, tensor.device)
        mode = _lib.REDUCE_ORDERED if ordered else _lib.REDUCE_NCCL
        _lib.check(self._lib.mf_reduce(ctypes.c_void_p(self.handle),
                                       ctypes.c_void_p(tensor.data_ptr()),
                                       tensor.numel(), int(root), mode, s))
        return tensor

    def close(self):
        if self._handle is not None:
            _lib.check(self._lib.mf_comm_destroy(self._handle))
            self._handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def exchange_unique_id(lib, group=None, device=None):
    """Rank 0 of `group` creates the NCCL unique id, every rank receives it
    (torch.distributed broadcast; works over gloo too)."""
    import torch.distributed as dist

    uid = (ctypes.c_ubyte * _lib.COMM_ID_BYTES)()
    if dist.get_rank(group) == 0:
        _lib.check(lib.mf_comm_unique_id(uid))
    box = [bytes(uid)]
    src = 0 if group is None else dist.get_global_rank(group, 0)
    dist.broadcast_object_list(box, src=src, group=group, device=device)
    return (ctypes.c_ubyte * _lib.COMM_ID_BYTES).from_buffer_copy(box[0])
