"""Host pipeline timing with torch-pinned buffers vs 2 MB-aligned, transparent-huge-page-backed
buffers registered with cudaHostRegister, in one process (does the pinned pages' size matter?)."""
import ctypes
import mmap
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_0901_1413_b200 import _lib  # noqa: E402

print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(), flush=True)
L = _lib.load()
name, field, m, l, n = bench.CONFIGS[1]
f, A, B = bench.make_inputs(field, m, l, n, 0, torch.device("cuda", 0), True)
vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
libc = ctypes.CDLL("libc.so.6")
MADV_HUGEPAGE = 14


def huge_pinned_like(t):
    nbytes = t.numel() * t.element_size()
    size = (nbytes + (2 << 20) - 1) // (2 << 20) * (2 << 20)
    buf = mmap.mmap(-1, size + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = ctypes.addressof(ctypes.c_char.from_buffer(buf))
    off = (-base) % (2 << 20)
    addr = base + off
    libc.madvise(ctypes.c_void_p(addr), ctypes.c_size_t(size), MADV_HUGEPAGE)
    arr = np.frombuffer(buf, dtype=np.uint8, count=size, offset=off)
    arr[:] = 0  # touch
    torch.cuda.cudart().cudaHostRegister(addr, size, 0)
    out = torch.from_numpy(arr[:nbytes].view(np.int64)).view(t.shape)
    out._keep = buf
    return out


def timed(Ah, Bh, Ch, k=10):
    for _ in range(3):
        L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0)
    r = []
    for _ in range(k):
        t0 = time.perf_counter()
        _lib.check(L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0))
        r.append((time.perf_counter() - t0) * 1e3)
    r.sort()
    return "min %.3f med %.3f" % (r[0], r[k // 2])


Cshape = (f.bits, m, (n + 63) // 64)
T = (A.planes.cpu().pin_memory(), B.planes.cpu().pin_memory(), torch.empty(Cshape, dtype=torch.int64).pin_memory())
Hh = [huge_pinned_like(x) for x in (A.planes.cpu(), B.planes.cpu(), torch.empty(Cshape, dtype=torch.int64))]
Hh[0].copy_(A.planes.cpu()); Hh[1].copy_(B.planes.cpu())
for rnd in range(2):
    print("torch-pinned: %s | huge-page registered: %s" % (timed(*T), timed(*Hh)), flush=True)
print("results equal:", bool(torch.equal(T[2], Hh[2])), flush=True)
