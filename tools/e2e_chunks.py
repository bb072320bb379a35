import ctypes, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for P in ("1", "2", "3", "4"):
    out = subprocess.run([sys.executable, "-c", f"""
import os, sys, time, ctypes, torch
os.environ['SG_HOST_CHUNKS'] = '{P}'
sys.path.insert(0, '.')
import bench
from paper_0901_1413_b200 import _lib
L = _lib.load()
dev = torch.device('cuda', 0)
for ci in (1, 2, 3):
    name, field, m, l, n = bench.CONFIGS[ci]
    f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
    Ah, Bh = A.planes.cpu().pin_memory(), B.planes.cpu().pin_memory()
    Ch = torch.empty((f.bits, m, (n + 63) // 64), dtype=torch.int64).pin_memory()
    vp = lambda t: ctypes.c_void_p(t.data_ptr())
    for _ in range(3): L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0); ts.append(time.perf_counter() - t0)
    print('P={P}', name, '%.3f ms' % (1e3 * min(ts)), flush=True)
"""], capture_output=True, text=True)
    print(out.stdout.strip(), out.stderr.strip()[-300:])
