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


SM_RESERVE = 8  # SMs left to the broadcast while later row blocks are in flight


def _default_multiply():
    from .m4rm import m4rm_multiply
    return m4rm_multiply


def _set_reserve(sms: int):
    from .m4rm import set_sm_reserve
    set_sm_reserve(sms)


def b_chunks(l: int, chunks: int, ratio: int = 1) -> list:
    """Word-aligned row ranges [(r0, r1)] of B (= k-chunks of the inner dimension).

    ratio 1: equal chunks; ratio r > 1: geometric, chunk j holds r^j parts of (1 + r + ... +
    r^(chunks-1)) -- a small first block so the first product starts early, the bulk last."""
    w = (l + 63) // 64
    chunks = max(1, min(chunks, w)) if l else 1
    weights = [ratio ** j for j in range(chunks)]
    tot, acc, cuts = sum(weights), 0, [0]
    for wt in weights[:-1]:
        acc += wt
        cuts.append(min(l, 64 * max(cuts[-1] // 64 + 1, (w * acc) // tot)))
    cuts.append(l)
    out = [(cuts[j], cuts[j + 1]) for j in range(chunks)]
    return [(a, b) for a, b in out if b > a] or [(0, l)]


def default_chunks(field, l: int, n: int) -> int:
    """Overlap the broadcast with the products when B is big enough for it to matter."""
    return 3 if field.bits * l * ((n + 63) // 64) * 8 >= (16 << 20) else 1


CHUNK_RATIO = 4  # geometric row blocks of B: 1/21, 4/21, 16/21 for three chunks


def sharded_multiply(A_shard: BitslicedMatrix, B: BitslicedMatrix, field, l: int, n: int, src: int = 0,
                     group=None, multiply=None, device=None, chunks: int = 1, add=None, return_b: bool = True):
    """C_shard = A_shard * B with B broadcast from `src`.  Returns (C_shard, B_local).

    chunks > 1 overlaps the broadcast with the products (SURVEY.md 8e "optional fusion"): B goes
    out as `chunks` word-aligned row blocks, all queued at once (async collectives), and the
    product of chunk j -- A's matching columns times B's rows -- starts as soon as chunk j has
    arrived, while chunk j+1 is still on the wire.  The chunk products are summed in the field
    (exact, then canonical), so the result is bit-identical to the single-broadcast path.
    B_local is None when return_b is False (saves re-assembling B from its chunks)."""
    if multiply is None:
        from .m4rm import m4rm_multiply as multiply
    if A_shard.ncols != l:
        raise ValueError(f"inner dimensions {A_shard.ncols} != {l}")
    parts = b_chunks(l, chunks, CHUNK_RATIO)
    if len(parts) == 1:
        B_local = broadcast_matrix(B, field, l, n, src=src, group=group, device=device)
        return multiply(A_shard, B_local), B_local
    canonical = add is None and field.name in ("f5", "f7")  # redundant encodings: canonical at the end
    if add is None:
        def add(X, Y):
            return X.add(Y)
    rank = dist.get_rank(group)
    W = (n + 63) // 64
    dev = device if device is not None else A_shard.device
    if rank == src:
        if B is None or (B.nrows, B.ncols) != (l, n) or B.field is not field:
            raise ValueError("source rank must pass B with the announced field and shape")
        src_planes = B.planes.to(dev)
        bufs = [src_planes[:, r0:r1].contiguous() for r0, r1 in parts]
    else:
        bufs = [torch.empty((field.bits, r1 - r0, W), dtype=torch.int64, device=dev) for r0, r1 in parts]
    works = [dist.broadcast(t, src=src, group=group, async_op=True) for t in bufs]
    # Product j runs while blocks j+1.. may still be on the wire: it is planned on all but
    # SM_RESERVE SMs so the collective's kernel always finds SMs (one product CTA fills an SM).
    # The last product starts only after every block has arrived (it waits for the last one),
    # so it gets every SM: the reserve is released exactly when the broadcast is complete.
    # With geometric blocks (CHUNK_RATIO) the reserved products cover ~1/4 of the work.
    reserve = SM_RESERVE if (multiply is _default_multiply() and dev.type == "cuda") else 0
    C = None
    try:
        for j, ((r0, r1), t, work) in enumerate(zip(parts, bufs, works)):
            w0, w1 = r0 // 64, (r1 + 63) // 64
            A_j = BitslicedMatrix(field, A_shard.nrows, r1 - r0, A_shard.planes[:, :, w0:w1].contiguous())
            work.wait()  # NCCL: the current stream waits for this chunk (the host does not block)
            if reserve:
                _set_reserve(reserve if j + 1 < len(parts) else 0)
            P = multiply(A_j, BitslicedMatrix(field, r1 - r0, n, t))
            C = P if C is None else add(C, P)
    finally:
        if reserve:
            _set_reserve(0)
    if canonical:
        C = C.reduce_canonical()
    B_local = BitslicedMatrix(field, l, n, torch.cat(bufs, dim=1)) if return_b else None
    return C, B_local


def multi_device_multiply(A: BitslicedMatrix, B: BitslicedMatrix, devices, params=None) -> BitslicedMatrix:
    """C = A B over several GPUs from ONE process (sg_m4rm_multi): rows of A / C sharded over
    `devices` (indices may repeat), B replicated by peer copies.  A and B are host matrices;
    C comes back on the host, bit-identical to the single-GPU product."""
    import ctypes

    from . import _lib
    from .m4rm import choose_k
    from .matrix import _vp
    if A.field is not B.field:
        raise ValueError("field mismatch")
    if A.ncols != B.nrows:
        raise ValueError(f"inner dimensions {A.ncols} != {B.nrows}")
    devices = [int(d) for d in devices]
    if not devices:
        raise ValueError("need at least one device")
    m, l, n = A.nrows, A.ncols, B.ncols
    k = (params.k if params is not None and params.k is not None else None) or choose_k(l)
    a = A.planes.cpu().contiguous()
    b = B.planes.cpu().contiguous()
    C = BitslicedMatrix.zero(A.field, m, n, device="cpu")
    devs = (ctypes.c_int * len(devices))(*devices)
    _lib.check(_lib.load().sg_m4rm_multi(A.field.code, _vp(a), _vp(b), _vp(C.planes), m, l, n, k, len(devices),
                                         devs))
    return C


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
