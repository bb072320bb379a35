"""Print sg_m4rm_host's pipeline timeline (SG_HOST_TRACE) for one config and chunkings.

python tools/e2e_trace.py [--config 1] [--chunks 1:2,4:2]"""
import argparse
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--chunks", default="1:2,4:2,4:4")
a = ap.parse_args()
for P in a.chunks.split(","):
    PK, PR = P.split(":")
    env = dict(os.environ, SG_HOST_KCHUNKS=PK, SG_HOST_CHUNKS=PR)
    code = f"""
import os, sys, time, ctypes, torch
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
t0 = time.perf_counter(); L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0)
print(name, 'wall %.3f ms' % (1e3 * (time.perf_counter() - t0)), flush=True)
"""
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=dict(env, SG_HOST_TRACE="1"))
    err = out.stderr.strip().split("sg_m4rm_host trace")
    print(out.stdout.strip(), "sg_m4rm_host trace" + err[-1] if len(err) > 1 else out.stderr[-500:], flush=True)
