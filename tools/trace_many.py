"""Several traced streamed host calls in one process (SG_HOST_TRACE=1 output parsed): per call,
A's piece 0 upload time, B's upload span, product 0 span, total."""
import ctypes
import os
import subprocess
import sys

code = r'''
import sys, ctypes, torch
sys.path.insert(0, '.')
import bench
from paper_0901_1413_b200 import _lib
L = _lib.load()
name, field, m, l, n = bench.CONFIGS[1]
f, A, B = bench.make_inputs(field, m, l, n, 0, torch.device('cuda', 0), True)
Ah, Bh = A.planes.cpu().pin_memory(), B.planes.cpu().pin_memory()
Ch = torch.empty((f.bits, m, (n + 63) // 64), dtype=torch.int64).pin_memory()
vp = lambda t: ctypes.c_void_p(t.data_ptr())
for _ in range(12): L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0)
'''
out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                     env=dict(os.environ, SG_HOST_TRACE="1")).stderr
calls, cur = [], None
for line in out.splitlines():
    if line.startswith("host_streamed trace"):
        cur = {}
        calls.append(cur)
    elif cur is not None and "ms" in line:
        t, what = line.split("ms", 1)
        cur[what.strip()] = float(t)
for c in calls[2:]:
    b = [v for k, v in c.items() if k.startswith("in: B chunk")]
    print("A0 %.3f | B done %.3f | A1 %.3f | p0 %.3f-%.3f | p1 done %.3f | end %.3f" % (
        c.get("in: A piece 0 up", -1), max(b) if b else -1, c.get("in: A piece 1 up", -1),
        c.get("comp: product 0 queued (inputs up)", -1), c.get("comp: product 0 done", -1),
        c.get("comp: product 1 done", -1), c.get("out: piece 1 down", -1)))
