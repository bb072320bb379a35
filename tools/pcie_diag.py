"""Diagnose e2e variance of sg_m4rm_host (headline shape): back-to-back calls, calls separated by
a torch H2D copy, calls after a short host sleep; PCIe copy speed next to them."""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_0901_1413_b200 import _lib  # noqa: E402

L = _lib.load()
dev = torch.device('cuda', 0)
name, field, m, l, n = bench.CONFIGS[1]
f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
Ah, Bh = A.planes.cpu().pin_memory(), B.planes.cpu().pin_memory()
Ch = torch.empty((f.bits, m, (n + 63) // 64), dtype=torch.int64).pin_memory()
vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
d = torch.empty_like(Ah, device=dev)


def h2d():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.copy_(Ah, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


def call():
    t0 = time.perf_counter()
    _lib.check(L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0))
    return (time.perf_counter() - t0) * 1e3


for _ in range(3):
    call()
r = sorted(call() for _ in range(10))
print('back-to-back: min %.3f med %.3f ms' % (r[0], r[5]), flush=True)
r = []
for _ in range(10):
    h2d()
    r.append(call())
r.sort()
print('after a torch H2D: min %.3f med %.3f ms' % (r[0], r[5]), flush=True)
r = []
for _ in range(10):
    time.sleep(0.01)
    r.append(call())
r.sort()
print('after 10 ms sleep: min %.3f med %.3f ms' % (r[0], r[5]), flush=True)
print('torch H2D 6.3 MB: %.3f ms' % min(h2d() for _ in range(5)), flush=True)
