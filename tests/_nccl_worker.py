"""One rank of the multi-GPU NCCL parity check (tests/test_multi_gpu.py; launched by
torch.distributed.run, one process per GPU).

Every rank multiplies its row slab of A by B, which rank 0 broadcasts over NCCL -- whole, and
in geometric row blocks overlapped with the chunk products (dist.sharded_multiply) -- and the
gathered C must equal, bit for bit, the single-GPU product and the CPU oracle (SPEC.md:360:
a row partition gives identical output).  Rank 0 prints one line `RESULT <json>`."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402  (the checker)
import paper_0901_1413_b200 as sg  # noqa: E402
from paper_0901_1413_b200 import dist as sgdist  # noqa: E402

CASES = [  # (field, m, l, n, chunks)
    ("f3", 1000, 1100, 900, 1), ("f5", 777, 1030, 515, 1), ("f7", 1024, 640, 1024, 1), ("gf4", 513, 2048, 700, 1),
    ("f3", 4096, 8192, 8192, 3), ("f5", 2048, 4096, 4096, 3), ("f7", 2048, 4096, 6144, 3), ("gf4", 4096, 8192, 8192, 3),
]


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    results = []
    for field, m, l, n, chunks in CASES:
        f = sg.by_name(field)
        A = oracle.random_dense(field, m, l, 0)
        Bd = oracle.random_dense(field, l, n, 1)
        r0, r1 = sgdist.row_partition(m, world)[rank]
        A_shard = sg.BitslicedMatrix.from_dense(f, A[r0:r1], device=dev)
        B = sg.BitslicedMatrix.from_dense(f, Bd, device=dev) if rank == 0 else None
        C_shard, _ = sgdist.sharded_multiply(A_shard, B, f, l, n, src=0, chunks=chunks, return_b=False)
        C = sgdist.gather_rows(C_shard, m)
        if rank == 0:
            got = C.planes_numpy()
            one = sg.m4rm_multiply(sg.BitslicedMatrix.from_dense(f, A, device=dev), B).planes_numpy()
            want = oracle.m4rm(field, oracle.pack(field, A), oracle.pack(field, Bd), l, n, 8,
                               threads=os.cpu_count() or 1)
            results.append({"case": [field, m, l, n, chunks], "eq_1gpu": bool(np.array_equal(got, one)),
                            "eq_oracle": bool(np.array_equal(got, want))})
    # single-process multi-device path (peer copies) over every visible GPU
    if rank == 0:
        ndev = torch.cuda.device_count()
        for field, m, l, n, _ in CASES[:4]:
            f = sg.by_name(field)
            A = oracle.random_dense(field, m, l, 0)
            Bd = oracle.random_dense(field, l, n, 1)
            Ah = sg.BitslicedMatrix.from_planes(f, oracle.pack(field, A), l, device="cpu")
            Bh = sg.BitslicedMatrix.from_planes(f, oracle.pack(field, Bd), n, device="cpu")
            got = sgdist.multi_device_multiply(Ah, Bh, list(range(ndev))).planes_numpy()
            want = oracle.m4rm(field, oracle.pack(field, A), oracle.pack(field, Bd), l, n, 8)
            results.append({"case": ["sg_m4rm_multi", field, m, l, n, ndev], "eq_oracle": bool(np.array_equal(got, want))})
        print("RESULT " + json.dumps({"world": world, "backend": dist.get_backend(), "results": results}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
