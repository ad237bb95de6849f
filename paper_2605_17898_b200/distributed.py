"""Multi-GPU setup: one process per GPU, row-sharded K, no PyTorch.

``init()`` builds this rank's library context with an NCCL communicator. Rank
and world come from the launcher's environment (``RANK`` / ``WORLD_SIZE`` /
``LOCAL_RANK``: torchrun, or ``bench.py --gpus N``'s own launcher). The
128-byte NCCL unique id is made on rank 0 by the library and handed to the
other ranks out of band, without ``torch.distributed``:

* ``LGP_NCCL_ID`` (256 hex digits) in the environment, when the launcher made
  the id itself (``launch()`` below), else
* a rendezvous file: rank 0 writes the id atomically (temp file + rename) to
  ``LGP_RDZV_FILE`` (default: ``$TMPDIR/lgp-nccl-<MASTER_PORT>-<parent pid>``;
  the ranks of one launch share their parent process) and removes it once the
  communicator is up (ncclCommInitRank returns only after every rank joined,
  so every rank has read it by then); the other ranks poll for it.

The data path is the library's own NCCL all-gather / all-reduce over NVLink.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys
import tempfile
import time

from . import _lib


def env_rank_world():
    """(rank, world, local_rank) from the launcher's environment."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if not (world >= 1 and 0 <= rank < world):
        raise ValueError(f"bad RANK/WORLD_SIZE: {rank}/{world}")
    return rank, world, local


def new_id():
    """A fresh 128-byte NCCL unique id (rank 0 / the launcher)."""
    buf = C.create_string_buffer(128)
    _lib.check(_lib.lib().lgp_comm_unique_id(buf))
    return buf.raw


def rendezvous_path():
    if os.environ.get("LGP_RDZV_FILE"):
        return os.environ["LGP_RDZV_FILE"]
    port = os.environ.get("MASTER_PORT", "0")
    return os.path.join(tempfile.gettempdir(), f"lgp-nccl-{port}-{os.getppid()}")


def publish_id(path, ident):
    tmp = f"{path}.{os.getpid()}.tmp"
    with open(tmp, "wb") as f:
        f.write(ident)
    os.replace(tmp, path)


def wait_id(path, timeout=120.0):
    t_end = time.time() + timeout
    while time.time() < t_end:
        try:
            with open(path, "rb") as f:
                data = f.read()
            if len(data) == 128:
                return data
        except FileNotFoundError:
            pass
        time.sleep(0.01)
    raise TimeoutError(f"no NCCL id from rank 0 at {path} within {timeout:.0f} s")


def exchange_id(rank, world):
    """Rank 0 makes the id; every rank returns the same 128 bytes."""
    if os.environ.get("LGP_NCCL_ID"):
        ident = bytes.fromhex(os.environ["LGP_NCCL_ID"])
        if len(ident) != 128:
            raise ValueError("LGP_NCCL_ID must be 256 hex digits")
        return ident, None
    path = rendezvous_path()
    if rank == 0:
        ident = new_id()
        publish_id(path, ident)
        return ident, path
    return wait_id(path), None


def init(device=None, force_comm=False):
    """This rank's context; ``force_comm`` opens a one-rank NCCL communicator
    at world 1 so the row-sharded schedule runs on a single GPU."""
    rank, world, local = env_rank_world()
    if device is not None:
        local = int(device)
    if world == 1:
        ctx = _lib.Context(local, 0, 1, new_id()) if force_comm else _lib.Context(local)
    else:
        ident, owned = exchange_id(rank, world)
        try:
            ctx = _lib.Context(local, rank, world, ident)
        finally:
            if owned:
                try:
                    os.unlink(owned)
                except FileNotFoundError:
                    pass
    _lib.set_default_context(ctx)
    return ctx


def partition(n, world, rank):
    """[r0, r1) rows of an n-row operator owned by `rank` (lgp_partition)."""
    r0, r1 = C.c_int64(), C.c_int64()
    _lib.check(_lib.lib().lgp_partition(int(n), int(world), int(rank), C.byref(r0), C.byref(r1)))
    return r0.value, r1.value


def launch(argv, world, env=None, stdout_rank0=None):
    """Run ``argv`` as `world` ranks (one process per GPU, LOCAL_RANK = rank)
    with a shared NCCL id in LGP_NCCL_ID. Rank 0's stdout goes to
    ``stdout_rank0`` (default: ours); the other ranks' stdout is discarded and
    every rank's stderr is inherited. Returns the worst exit code."""
    base = dict(os.environ if env is None else env)
    base["LGP_NCCL_ID"] = new_id().hex()
    base.setdefault("MASTER_ADDR", "127.0.0.1")
    procs = []
    for r in range(world):
        e = dict(base, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(world),
                 LOCAL_WORLD_SIZE=str(world))
        out = (stdout_rank0 or sys.stdout) if r == 0 else subprocess.DEVNULL
        procs.append(subprocess.Popen(argv, env=e, stdout=out))
    codes = [p.wait() for p in procs]
    return max(codes, key=abs)
