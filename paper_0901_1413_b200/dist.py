"""Row-sharded multi-GPU M4RM: A and C split by rows, B broadcast once from one rank.

C_i = A_i B depends only on row i of A, so rank r multiplies its contiguous
slab of A's rows by the whole of B; the inner dimension is never split, so every rank walks
the k-blocks in the same order and the output is bit-identical for any world size (the GPU
form of the reference's row-partition contract, and of the row0/row1 arguments
of every block driver, _core_py.py:205, 213, 274, 279).  The one exchange step is the
broadcast of B's packed planes (torch.distributed over NCCL, i.e. NVLink / NVSwitch on an
8xB200 node); with gloo the same host logic runs on CPU tensors for the tests.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .matrix import BitslicedMatrix


def row_partition(m: int, world: int) -> list:
    """Contiguous, balanced row slabs [(r0, r1)] for ranks 0..world-1."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    return [(m * r // world, m * (r + 1) // world) for r in range(world)]


def shard_rows(M: BitslicedMatrix, rank: int, world: int) -> BitslicedMatrix:
    r0, r1 = row_partition(M.nrows, world)[rank]
    return BitslicedMatrix(M.field, r1 - r0, M.ncols, M.planes[:, r0:r1].contiguous())


def broadcast_matrix(B: BitslicedMatrix, field, nrows: int, ncols: int, src: int = 0, group=None,
                     device=None) -> BitslicedMatrix:
    """Broadcast B's planes from rank `src`; other ranks pass B=None and get the matrix."""
    rank = dist.get_rank(group)
    shape = (field.bits, nrows, (ncols + 63) // 64)
    if rank == src:
        if B is None or (B.nrows, B.ncols) != (nrows, ncols) or B.field is not field:
            raise ValueError("source rank must pass B with the announced field and shape")
        t = B.planes if device is None else B.planes.to(device)
        t = t.contiguous()
    else:
        t = torch.empty(shape, dtype=torch.int64, device=device or "cpu")
    dist.broadcast(t, src=src, group=group)
    return BitslicedMatrix(field, nrows, ncols, t)


def sharded_multiply(A_shard: BitslicedMatrix, B: BitslicedMatrix, field, l: int, n: int, src: int = 0,
                     group=None, multiply=None, device=None):
    """C_shard = A_shard * B with B broadcast from `src`.  Returns (C_shard, B_local)."""
    if multiply is None:
        from .m4rm import m4rm_multiply as multiply
    if A_shard.ncols != l:
        raise ValueError(f"inner dimensions {A_shard.ncols} != {l}")
    B_local = broadcast_matrix(B, field, l, n, src=src, group=group, device=device)
    return multiply(A_shard, B_local), B_local


def gather_rows(C_shard: BitslicedMatrix, m: int, group=None) -> BitslicedMatrix:
    """All-gather row shards into the full C (verification only; not on the timed path)."""
    world = dist.get_world_size(group)
    parts = row_partition(m, world)
    R, W = C_shard.field.bits, C_shard.words_per_row
    bufs = [torch.empty((R, r1 - r0, W), dtype=torch.int64, device=C_shard.device) for r0, r1 in parts]
    maxrows = max(r1 - r0 for r0, r1 in parts)
    padded = torch.zeros((R, maxrows, W), dtype=torch.int64, device=C_shard.device)
    padded[:, : C_shard.nrows] = C_shard.planes
    gathered = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(gathered, padded, group=group)
    for i, (r0, r1) in enumerate(parts):
        bufs[i] = gathered[i][:, : r1 - r0]
    return BitslicedMatrix(C_shard.field, m, C_shard.ncols, torch.cat(bufs, dim=1).contiguous())
