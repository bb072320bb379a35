"""Streamed vs B-first host pipeline alternating in ONE process (SG_HOST_STREAM read per call),
plus a plain torch H2D of the same pinned A, to separate process-level PCIe state from the path."""
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
d = torch.empty_like(Ah, device="cuda")


def call(mode):
    os.environ["SG_HOST_STREAM"] = mode
    t0 = time.perf_counter()
    _lib.check(L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0))
    return (time.perf_counter() - t0) * 1e3


def h2d():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.copy_(Ah, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


print("torch H2D before any call: %.3f ms" % min(h2d() for _ in range(5)), flush=True)
for _ in range(3):
    call("0")
print("torch H2D after B-first calls: %.3f ms" % min(h2d() for _ in range(5)), flush=True)
for _ in range(3):
    call("1")
print("torch H2D after streamed calls: %.3f ms" % min(h2d() for _ in range(5)), flush=True)
r0, r1 = [], []
for _ in range(8):
    r0.append(call("0"))
    r1.append(call("1"))
r0.sort(); r1.sort()
print("alternating: B-first min %.3f med %.3f | streamed min %.3f med %.3f" % (r0[0], r0[4], r1[0], r1[4]), flush=True)
print("torch H2D at the end: %.3f ms" % min(h2d() for _ in range(5)), flush=True)
