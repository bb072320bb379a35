"""Copies of the host pipeline's shapes from torch-pinned buffers inside a torch process (cuda-python
runtime calls on a private stream): A's row piece as one 2-D copy vs contiguous, B's chunks."""
import time

import torch
from cuda.bindings import runtime as rt

R, rows, rowb = 3, 4096, 512
plane = rows * rowb
hA = torch.empty(R * plane, dtype=torch.uint8).pin_memory()
hB = torch.empty(R * plane, dtype=torch.uint8).pin_memory()
hA.fill_(1); hB.fill_(2)
dA = torch.empty(R * plane, dtype=torch.uint8, device="cuda")
dB = torch.empty(R * plane, dtype=torch.uint8, device="cuda")
err, s = rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking)
H2D = rt.cudaMemcpyKind.cudaMemcpyHostToDevice
half = plane // 2


def timed(fn, reps=10):
    best = 1e9
    for _ in range(reps):
        rt.cudaStreamSynchronize(s)
        t0 = time.perf_counter()
        fn()
        rt.cudaStreamSynchronize(s)
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


a2d = timed(lambda: rt.cudaMemcpy2DAsync(dA.data_ptr(), half, hA.data_ptr(), plane, half, R, H2D, s))
a1d = timed(lambda: [rt.cudaMemcpyAsync(dA.data_ptr() + p * half, hA.data_ptr() + p * plane, half, H2D, s) for p in range(R)])
acont = timed(lambda: rt.cudaMemcpyAsync(dA.data_ptr(), hA.data_ptr(), R * half, H2D, s))
g0 = 4 * 32 * rowb
lo = lambda j: min(plane, g0 * ((1 << j) - 1))  # noqa: E731


def bchunks():
    j = 0
    while lo(j) < plane:
        rt.cudaMemcpy2DAsync(dB.data_ptr() + lo(j), plane, hB.data_ptr() + lo(j), plane, lo(j + 1) - lo(j), R, H2D, s)
        j += 1


b2d = timed(bchunks)
bcont = timed(lambda: rt.cudaMemcpyAsync(dB.data_ptr(), hB.data_ptr(), R * plane, H2D, s))
print("A piece (3.1 MB): 2-D %.3f ms | 3 per-plane %.3f | contiguous %.3f ;  B (6.3 MB): 6 geometric 2-D chunks %.3f | "
      "contiguous %.3f" % (a2d, a1d, acont, b2d, bcont), flush=True)
