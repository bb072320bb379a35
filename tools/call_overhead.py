"""Host cost per m4rm_multiply call on tiny device-resident operands (wall clock per call).

python tools/call_overhead.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes  # noqa: E402

import torch  # noqa: E402

import paper_0901_1413_b200 as sg  # noqa: E402
from paper_0901_1413_b200 import _lib  # noqa: E402
from paper_0901_1413_b200.matrix import _vp  # noqa: E402

A = sg.BitslicedMatrix.random(sg.F3, 64, 64, seed=0)
B = sg.BitslicedMatrix.random(sg.F3, 64, 64, seed=1)
C = sg.BitslicedMatrix.zero(sg.F3, 64, 64)
P = sg.M4rmParams(8)
for _ in range(100):
    sg.m4rm_multiply(A, B, P, out=C)
torch.cuda.synchronize()
N = 2000
t0 = time.perf_counter()
for _ in range(N):
    sg.m4rm_multiply(A, B, P, out=C)
torch.cuda.synchronize()
py = (time.perf_counter() - t0) / N
L = _lib.load()
st = _lib.current_stream_handle(A.device)
a, b, c = _vp(A.planes), _vp(B.planes), _vp(C.planes)
t0 = time.perf_counter()
for _ in range(N):
    L.sg_m4rm(1, a, b, c, 64, 64, 64, 8, None, 0, st)
torch.cuda.synchronize()
cab = (time.perf_counter() - t0) / N
print(f"m4rm_multiply (Python API) {py * 1e6:.1f} us/call, sg_m4rm (C ABI via ctypes) {cab * 1e6:.1f} us/call")
