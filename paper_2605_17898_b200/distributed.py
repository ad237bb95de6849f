"""Multi-GPU setup: one process per GPU (torchrun), row-sharded K.

``init()`` builds this rank's library context with an NCCL communicator. The
128-byte NCCL unique id is made on rank 0 by the library and broadcast over
whatever ``torch.distributed`` process group the launcher initialised (gloo is
enough: PyTorch is plumbing here, the data path is the library's own NCCL
all-gather over NVLink).
"""

from __future__ import annotations

import ctypes as C
import os

from . import _lib


def init(device=None, force_comm=False):
    """This rank's context; ``force_comm`` opens a one-rank NCCL communicator
    at world 1 so the row-sharded schedule runs on a single GPU."""
    import torch.distributed as dist

    rank = dist.get_rank() if dist.is_initialized() else int(os.environ.get("RANK", "0"))
    world = dist.get_world_size() if dist.is_initialized() else int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", rank)) if device is None else int(device)
    if world == 1:
        if force_comm:
            buf = C.create_string_buffer(128)
            _lib.check(_lib.lib().lgp_comm_unique_id(buf))
            ctx = _lib.Context(local, 0, 1, buf.raw)
        else:
            ctx = _lib.Context(local)
    else:
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed must be initialised for a multi-rank context")
        obj = [None]
        if rank == 0:
            buf = C.create_string_buffer(128)
            _lib.check(_lib.lib().lgp_comm_unique_id(buf))
            obj[0] = buf.raw
        dist.broadcast_object_list(obj, src=0)
        ctx = _lib.Context(local, rank, world, obj[0])
    _lib.set_default_context(ctx)
    return ctx


def partition(n, world, rank):
    """[r0, r1) rows of an n-row operator owned by `rank` (lgp_partition)."""
    r0, r1 = C.c_int64(), C.c_int64()
    _lib.check(_lib.lib().lgp_partition(int(n), int(world), int(rank), C.byref(r0), C.byref(r1)))
    return r0.value, r1.value
