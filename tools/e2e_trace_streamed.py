import sys, time, ctypes, torch, os
sys.path.insert(0, '.')
import bench
from paper_0901_1413_b200 import _lib
L = _lib.load()
dev = torch.device('cuda', 0)
name, field, m, l, n = bench.CONFIGS[1]
f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
Ah, Bh = A.planes.cpu().pin_memory(), B.planes.cpu().pin_memory()
Ch = torch.empty((f.bits, m, (n + 63) // 64), dtype=torch.int64).pin_memory()
vp = lambda t: ctypes.c_void_p(t.data_ptr())
for _ in range(5): L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0)
t0 = time.perf_counter(); L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0); print('wall %.3f ms' % (1e3*(time.perf_counter()-t0)), file=sys.stderr)
