"""Streamed host calls back to back vs alternating with B-first calls, in one process (means)."""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_0901_1413_b200 import _lib  # noqa: E402

L = _lib.load()
name, field, m, l, n = bench.CONFIGS[1]
f, A, B = bench.make_inputs(field, m, l, n, 0, torch.device("cuda", 0), True)
Ah, Bh = A.planes.cpu().pin_memory(), B.planes.cpu().pin_memory()
Ch = torch.empty((f.bits, m, (n + 63) // 64), dtype=torch.int64).pin_memory()
vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731


def call(mode):
    os.environ["SG_HOST_STREAM"] = mode
    t0 = time.perf_counter()
    _lib.check(L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0))
    return (time.perf_counter() - t0) * 1e3


for _ in range(3):
    call("1")
for rnd in range(3):
    s = [call("1") for _ in range(10)]
    alt = []
    for _ in range(10):
        call("0")
        alt.append(call("1"))
    print("streamed back to back: mean %.3f | streamed after a B-first call: mean %.3f" % (sum(s) / 10, sum(alt) / 10),
          flush=True)
