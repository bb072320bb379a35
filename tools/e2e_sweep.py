"""e2e sweep of the streamed host pipeline: row pieces x first B chunk in 32-row groups (SG_HOST_CHUNKS, SG_HOST_BFIRST).

python tools/e2e_sweep.py [--config 1] [--pieces 1,2,3,4] [--bfirst 2,4,8,16] [--stream 0,1]"""
import argparse
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="1")
ap.add_argument("--pieces", default="1,2,3,4")
ap.add_argument("--bfirst", default="2,4,8,16")
ap.add_argument("--stream", default="1")
a = ap.parse_args()
code = f"""
import sys, time, ctypes, torch
sys.path.insert(0, '.')
import bench
from paper_0901_1413_b200 import _lib
L = _lib.load()
dev = torch.device('cuda', 0)
name, field, m, l, n = bench.CONFIGS[{a.config}]
f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
Ah, Bh = A.planes.cpu().pin_memory(), B.planes.cpu().pin_memory()
Ch = torch.empty((f.bits, m, (n + 63) // 64), dtype=torch.int64).pin_memory()
vp = lambda t: ctypes.c_void_p(t.data_ptr())
for _ in range(3): L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0)
ts = []
for _ in range(20):
    t0 = time.perf_counter(); _lib.check(L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0)); ts.append(time.perf_counter() - t0)
ts.sort()
print(name, 'min %.3f med %.3f ms' % (1e3 * ts[0], 1e3 * ts[len(ts) // 2]), flush=True)
"""
for st in a.stream.split(","):
    for pr in a.pieces.split(","):
        for bc in a.bfirst.split(","):
            env = dict(os.environ, SG_HOST_STREAM=st, SG_HOST_CHUNKS=pr, SG_HOST_BFIRST=bc)
            out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
            print(f"stream={st} pieces={pr} bfirst={bc} |", out.stdout.strip(), out.stderr.strip()[-300:], flush=True)
