"""bench.e2e_for vs a plain loop of sg_m4rm_host calls, alternating in ONE process."""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_0901_1413_b200 import _lib  # noqa: E402

L = _lib.load()
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)


class Args:
    steps, warmup = 10, 3


name, field, m, l, n = bench.CONFIGS[1]


def plain():
    f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
    Ah, Bh = A.planes.cpu().pin_memory(), B.planes.cpu().pin_memory()
    Ch = torch.empty((f.bits, m, (n + 63) // 64), dtype=torch.int64).pin_memory()
    vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    for _ in range(3):
        L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        _lib.check(L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0))
        ts.append(time.perf_counter() - t0)
    return 1e3 * sum(ts) / len(ts)


for r in range(4):
    a = plain()
    b = bench.e2e_for(bench.CONFIGS[1], Args, 1, 0, dev)["ms_per_step"]
    print("plain loop mean %.3f ms | bench.e2e_for %.3f ms" % (a, b), flush=True)
