"""Small products through every schedule and a few fields, for compute-sanitizer runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_0901_1413_b200 as sg  # noqa: E402
from paper_0901_1413_b200 import m4rm as M  # noqa: E402

fields = {"f3": sg.F3, "f5": sg.F5, "f7": sg.F7, "gf4": sg.GF4}
bad = 0
for name, f in fields.items():
    A = oracle.random_dense(name, 300, 200, 1)
    B = oracle.random_dense(name, 200, 300, 2)
    want = oracle.pack(name, oracle.dense_multiply(name, A, B))
    Ag, Bg = sg.BitslicedMatrix.from_dense(f, A), sg.BitslicedMatrix.from_dense(f, B)
    for rt, nt, sched, splits in ((1, 256, 0, 2), (2, 256, 1, 1), (4, 256, 2, 3), (2, 512, 1, 2)):
        M.set_plan_override(rt, splits, sched, nt)
        try:
            C = sg.m4rm_multiply(Ag, Bg)
        except RuntimeError:
            continue
        ok = np.array_equal(C.planes_numpy(), want)
        bad += not ok
        print(name, rt, nt, sched, splits, "ok" if ok else "MISMATCH", flush=True)
# streamed B through the host pipeline (pinned buffers, forced stream-K warp-specialized plans)
from paper_0901_1413_b200 import _lib  # noqa: E402
L = _lib.load()
for name, f in fields.items():
    A = oracle.random_dense(name, 1500, 1024, 5)
    B = oracle.random_dense(name, 1024, 256, 6)
    want = oracle.pack(name, oracle.dense_multiply(name, A, B))
    Ah = sg.BitslicedMatrix(f, 1500, 1024, sg.BitslicedMatrix.from_planes(f, oracle.pack(name, A), 1024,
                                                                           device="cpu").planes.pin_memory())
    Bh = sg.BitslicedMatrix(f, 1024, 256, sg.BitslicedMatrix.from_planes(f, oracle.pack(name, B), 256,
                                                                          device="cpu").planes.pin_memory())
    M.set_plan_override(4 if f.bits == 3 else 8, -1, 2, 256)
    c0 = L.sg_host_streamed_count()
    C = sg.m4rm_multiply(Ah, Bh, sg.M4rmParams(8))
    ok = np.array_equal(C.planes_numpy(), want) and L.sg_host_streamed_count() == c0 + 1
    bad += not ok
    print(name, "streamed host", "ok" if ok else "MISMATCH", flush=True)
M.set_plan_override(0, 0, -1, 0)
C = sg.m4rm_multiply(sg.BitslicedMatrix.from_dense(sg.F3, oracle.random_dense("f3", 64, 77, 3)),
                     sg.BitslicedMatrix.from_dense(sg.F3, oracle.random_dense("f3", 77, 65, 4)), sg.M4rmParams(5))
print("done, mismatches:", bad)
sys.exit(1 if bad else 0)
