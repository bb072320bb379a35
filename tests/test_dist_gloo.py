"""World-size-2 gloo test of the row-sharded multi-GPU host logic (on CPU).

The GPU multiply is replaced by the oracle (the checker) so the partition, the broadcast of
B's planes from rank 0 and the row gather are exercised without a GPU; on the B200 box the
same code runs with NCCL and m4rm_multiply (bench.py --gpus N)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_multiply(A, B):
    import oracle
    import paper_0901_1413_b200 as sg
    name = A.field.name
    C = oracle.m4rm(name, A.planes_numpy(), B.planes_numpy(), A.ncols, B.ncols, 8)
    return sg.BitslicedMatrix.from_planes(A.field, C, B.ncols, device="cpu")


def _oracle_add(X, Y):
    import oracle
    import paper_0901_1413_b200 as sg
    name = X.field.name
    q = oracle.ORDER[name]
    x, y = oracle.unpack(name, X.planes_numpy(), X.ncols), oracle.unpack(name, Y.planes_numpy(), Y.ncols)
    s = (x ^ y) if name in ("gf4", "gf8", "f2") else (x.astype(int) + y) % q
    return sg.BitslicedMatrix.from_planes(X.field, oracle.pack(name, s.astype(np.uint8)), X.ncols, device="cpu")


def _worker(rank, world, port, field_name, m, l, n, out_q, chunks=1):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_0901_1413_b200 as sg
        from paper_0901_1413_b200 import dist as sgdist
        field = sg.by_name(field_name)
        oname = field.name
        A_full = oracle.random_dense(oname, m, l, 0)
        r0, r1 = sgdist.row_partition(m, world)[rank]
        A_shard = sg.BitslicedMatrix.from_planes(field, oracle.pack(oname, A_full[r0:r1]), l, device="cpu")
        B = None
        if rank == 0:
            B = sg.BitslicedMatrix.from_planes(field, oracle.pack(oname, oracle.random_dense(oname, l, n, 1)), n,
                                               device="cpu")
        C_shard, B_local = sgdist.sharded_multiply(A_shard, B, field, l, n, src=0, multiply=_oracle_multiply,
                                                   chunks=chunks, add=_oracle_add if chunks > 1 else None)
        if rank == 1:
            want_b = oracle.pack(oname, oracle.random_dense(oname, l, n, 1))
            assert np.array_equal(B_local.planes_numpy(), want_b)
        C = sgdist.gather_rows(C_shard, m)
        if rank == 0:
            want = oracle.dense_multiply(oname, A_full, oracle.random_dense(oname, l, n, 1))
            got = oracle.unpack(oname, C.planes_numpy(), n)
            out_q.put(bool(np.array_equal(got, want)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("field_name,m,l,n,chunks", [("f3", 67, 90, 130, 1), ("f7", 10, 33, 65, 1),
                                                     ("gf4", 5, 17, 64, 1), ("f5", 9, 300, 70, 4),
                                                     ("f3", 33, 129, 65, 2), ("f7", 6, 200, 20, 3)])
def test_world2_sharded_multiply_matches_oracle(field_name, m, l, n, chunks):
    """chunks > 1: the broadcast of B in row blocks overlapped with the per-chunk products."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, field_name, m, l, n, q, chunks)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
