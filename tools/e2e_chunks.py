"""e2e experiments for sg_m4rm_host: chunk count sweep, copy-only bandwidth, per-chunk compute.

python tools/e2e_chunks.py [--configs 1,2,3] [--chunks 1:1,2:2,4:4]   (k-chunks:row pieces[:column pieces])"""
import argparse
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3")
ap.add_argument("--chunks", default="1:1,1:2,1:4,2:2,2:4,4:2,4:4,3:4")
a = ap.parse_args()
for P in a.chunks.split(","):
    parts = P.split(":")
    PK, PR = parts[0], parts[1]
    PC = parts[2] if len(parts) > 2 else "1"
    out = subprocess.run([sys.executable, "-c", f"""
import os, sys, time, ctypes, torch
os.environ['SG_HOST_KCHUNKS'] = '{PK}'
os.environ['SG_HOST_CCHUNKS'] = '{PC}'
os.environ['SG_HOST_CHUNKS'] = '{PR}'
sys.path.insert(0, '.')
import bench
import paper_0901_1413_b200 as sg
from paper_0901_1413_b200 import _lib
L = _lib.load()
dev = torch.device('cuda', 0)
for ci in ({a.configs},):
    name, field, m, l, n = bench.CONFIGS[ci]
    f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
    Ah, Bh = A.planes.cpu().pin_memory(), B.planes.cpu().pin_memory()
    Ch = torch.empty((f.bits, m, (n + 63) // 64), dtype=torch.int64).pin_memory()
    vp = lambda t: ctypes.c_void_p(t.data_ptr())
    for _ in range(3): L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0); ts.append(time.perf_counter() - t0)
    extra = ''
    if '{P}' == '1:1':
        d = torch.empty_like(Ah, device=dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5): d.copy_(Ah, non_blocking=True)
        torch.cuda.synchronize(); h2d = (time.perf_counter() - t0) / 5
        t0 = time.perf_counter()
        for _ in range(5): Ah.copy_(d, non_blocking=True)
        torch.cuda.synchronize(); d2h = (time.perf_counter() - t0) / 5
        extra = ' h2d %.1f GB/s d2h %.1f GB/s (%.1f MB)' % (Ah.numel() * 8 / h2d / 1e9, Ah.numel() * 8 / d2h / 1e9, Ah.numel() * 8 / 1e6)
        for parts in (1, 2, 4, 8):
            mm = m // parts
            sub = sg.BitslicedMatrix(f, mm, l, A.planes[:, :mm].contiguous())
            C = sg.m4rm_multiply(sub, B, sg.M4rmParams(8))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(parts): sg.m4rm_multiply(sub, B, sg.M4rmParams(8), out=C)
            e1.record(); torch.cuda.synchronize()
            extra += ' | %d x %d rows: %.3f ms' % (parts, mm, e0.elapsed_time(e1))
    print('P={P}', name, '%.3f ms' % (1e3 * min(ts)) + extra, flush=True)
"""], capture_output=True, text=True)
    print(out.stdout.strip(), out.stderr.strip()[-300:], flush=True)
