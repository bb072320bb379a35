"""In-process A/B of host-pipeline variants (environment switches read per call, e.g.
SG_HOST_PIECES / SG_HOST_CHUNKS): the calls alternate variant by variant, so the shared host's
per-process PCIe state is the same for all of them.
python tools/e2e_ab.py CONFIG 'SG_HOST_PIECES=1,1' 'SG_HOST_PIECES=1,1,1,1' ..."""
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_0901_1413_b200 import _lib  # noqa: E402

ci = int(sys.argv[1])
variants = sys.argv[2:]
L = _lib.load()
dev = torch.device("cuda", 0)
name, field, m, l, n = bench.CONFIGS[ci]
f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
Ah, Bh = A.pin_memory().planes, B.pin_memory().planes  # written by one thread on one CPU
Ch = A.pinned_zero(f, m, n).planes
vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731


def setv(v):
    for kv in variants:
        os.environ.pop(kv.split("=")[0], None)
    if "=" in v:
        k, val = v.split("=", 1)
        os.environ[k] = val


times = {v: [] for v in variants}
for rnd in range(12):
    for v in variants:
        setv(v)
        _lib.check(L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0))
        t0 = time.perf_counter()
        _lib.check(L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0))
        if rnd >= 2:
            times[v].append(1e3 * (time.perf_counter() - t0))
ref = A.planes.new_empty(Ch.shape)
import paper_0901_1413_b200 as sg  # noqa: E402
ok = torch.equal(sg.m4rm_multiply(A, B).planes.cpu(), Ch)
for v in variants:
    print(f"{name} {v:34s} e2e min {min(times[v]):.3f} median {statistics.median(times[v]):.3f} ms"
          + ("" if ok else "  (LAST RESULT WRONG)"), flush=True)
