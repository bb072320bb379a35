"""Is the host pipeline slower after bench.py's device-path loop in the same process?
Runs: host calls (fresh process), then bench.run_config (device loop + its e2e), then host calls."""
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
name, field, m, l, n = bench.CONFIGS[1]
f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
Ah, Bh = A.planes.cpu().pin_memory(), B.planes.cpu().pin_memory()
Ch = torch.empty((f.bits, m, (n + 63) // 64), dtype=torch.int64).pin_memory()
vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731


def clocks():
    import subprocess
    q = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.mem,pstate,power.draw",
                        "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    return q


def calls(k=10):
    print("   [clocks before: %s]" % clocks(), flush=True)
    r = []
    for _ in range(k):
        t0 = time.perf_counter()
        _lib.check(L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0))
        r.append((time.perf_counter() - t0) * 1e3)
    r.sort()
    return "min %.3f med %.3f [after: %s]" % (r[0], r[len(r) // 2], clocks())


calls(3)
print("fresh:", calls(), flush=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for i in range(5):
    flush.fill_(i)
print("after 256 MB flush buffer + fills:", calls(), flush=True)
import paper_0901_1413_b200 as sg  # noqa: E402
C = sg.BitslicedMatrix.zero(f, m, n, device=dev)
for i in range(10):
    flush.fill_(i)
    sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
torch.cuda.synchronize()
print("after device products:", calls(), flush=True)
with bench.ClockSampler(0):
    for i in range(10):
        flush.fill_(i)
        sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
    torch.cuda.synchronize()
print("after device products under the nvidia-smi sampler:", calls(), flush=True)
sg.m4rm.set_timing(True)
for i in range(5):
    flush.fill_(i)
    sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
sg.m4rm.set_timing(False)
print("after set_timing products:", calls(), flush=True)
peaks = sg.m4rm.probe_peaks(0)
print("after probe_peaks:", calls(), flush=True)
time.sleep(2)
print("after 2 s idle:", calls(), flush=True)
