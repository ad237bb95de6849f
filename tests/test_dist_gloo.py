"""World-size-2 (gloo, CPU) coverage of the multi-GPU path's host logic:
the library's row partition, the NCCL unique-id exchange used by
distributed.init() (rendezvous file, no torch.distributed), the sharded-CG schedule (local rows of K.p -> all-gather
-> redundant FP64 updates) and the multi-rank symmetric schedule (a share of
the block pairs over all rows -> all-reduce), both reproducing the unsharded
reference CG."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, rdzv):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import torch
        from oracle import gp_oracle as O
        from paper_2605_17898_b200 import distributed

        res = {}
        # 1. partition from the C ABI
        n = 1001
        r0, r1 = distributed.partition(n, world, rank)
        res["part"] = (r0, r1)
        # 2. NCCL id exchange of distributed.init (rendezvous file, no torch)
        os.environ["LGP_RDZV_FILE"] = os.path.join(rdzv, "nccl-id")
        os.environ["RANK"], os.environ["WORLD_SIZE"] = str(rank), str(world)
        try:
            ident, owned = distributed.exchange_id(rank, world)
        except Exception as exc:  # NCCL not loadable here
            ident, owned = f"ERR {exc}".encode(), None
        dist.barrier()  # (the library's ncclCommInitRank is this barrier on a GPU box)
        if owned:
            os.unlink(owned)
        res["id"] = ident
        # 3. sharded CG schedule on the oracle
        rng = np.random.default_rng(3)
        x = rng.random((n, 3))
        b = rng.standard_normal(n)
        nodes = O.parse_tree("(scale 1.2 (matern52 0.6))")
        S = -(-n // world)

        def sharded_apply(p):
            local = O.matvec(nodes, x, 0.1, p, block=64, row_range=(r0, r1))
            buf = torch.zeros(S, dtype=torch.float64)
            buf[: r1 - r0] = torch.from_numpy(local)
            parts = [torch.zeros(S, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, buf)
            full = torch.cat(parts).numpy()[:n]
            return full

        xs, it, rr = O.cg(sharded_apply, b, 1e-10)
        res["cg"] = (xs, it, rr)
        # 4. multi-rank symmetric schedule (engine.cpp cg_device, rank_split):
        #    each rank evaluates a contiguous share of the block pairs (I, J >= I)
        #    over ALL rows - K_IJ p_J into rows I and K_IJ^T p_I into rows J -
        #    and one all-reduce (sum) yields the full product on every rank
        B = 128
        nb = -(-n // B)
        pairs = [(I, J) for I in range(nb) for J in range(I, nb)]
        lo, hi = len(pairs) * rank // world, len(pairs) * (rank + 1) // world

        def split_apply(p):
            part = np.zeros(n)
            for I, J in pairs[lo:hi]:
                i0, i1, j0, j1 = I * B, min(n, (I + 1) * B), J * B, min(n, (J + 1) * B)
                k = O.gram(nodes, x[i0:i1], x[j0:j1])
                part[i0:i1] += k @ p[j0:j1]
                if J != I:
                    part[j0:j1] += k.T @ p[i0:i1]
            if rank == 0:
                part += 0.1 * p
            t = torch.from_numpy(part)
            dist.all_reduce(t)
            return t.numpy().copy()

        res["cg_split"] = O.cg(split_apply, b, 1e-10)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_world2_partition_id_and_sharded_cg(tmp_path):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # partition covers [0, n) without overlap
    assert out[0]["part"] == (0, 501) and out[1]["part"] == (501, 1001)
    # every rank received the same id bytes
    assert out[0]["id"] == out[1]["id"]
    if not out[0]["id"].startswith(b"ERR"):
        assert len(out[0]["id"]) == 128
    # both ranks hold identical CG state, equal to the unsharded reference CG
    from oracle import gp_oracle as O

    rng = np.random.default_rng(3)
    x = rng.random((1001, 3))
    b = rng.standard_normal(1001)
    nodes = O.parse_tree("(scale 1.2 (matern52 0.6))")
    ref = O.cg(lambda v: O.matvec(nodes, x, 0.1, v, block=64), b, 1e-10)
    x0, it0, r0 = out[0]["cg"]
    x1, it1, r1 = out[1]["cg"]
    np.testing.assert_array_equal(x0, x1)
    assert it0 == it1 == ref[1]
    np.testing.assert_allclose(x0, ref[0], rtol=0, atol=1e-9 * np.abs(ref[0]).max())
    # symmetric pair split + all-reduce: identical on both ranks, equal to the reference
    xs0, its0, _ = out[0]["cg_split"]
    xs1, its1, _ = out[1]["cg_split"]
    np.testing.assert_array_equal(xs0, xs1)
    assert its0 == its1 and abs(its0 - ref[1]) <= 1
    np.testing.assert_allclose(xs0, ref[0], rtol=0, atol=1e-8 * np.abs(ref[0]).max())
