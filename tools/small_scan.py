"""Small-product cost model on the GPU: step time (flushed L2, events around one call, as in
bench.py) and back-to-back time for F3 1024 x l x 1024 over l, under the planner's choice and a
few forced plans -- intercept = fixed per-call cost, slope = per-k-block cost.
python tools/small_scan.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0901_1413_b200 as sg  # noqa: E402
from paper_0901_1413_b200 import m4rm as M  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for ov in [(0, 0, -1, 0), (4, 16, 1, 256), (2, 16, 0, 512), (4, 32, 0, 256), (2, 32, 0, 256), (1, 32, 0, 256)]:
    M.set_plan_override(*ov)
    for l in (64, 128, 256, 512, 1024, 2048):
        f, A, B = bench.make_inputs("f3", 1024, l, 1024, 0, dev, True)
        C = sg.BitslicedMatrix.zero(f, 1024, 1024, device=dev)
        try:
            p = sg.plan(f, 1024, l, 1024, 8)
        except Exception as e:  # noqa: BLE001
            print(ov, l, "no plan", e)
            continue
        for _ in range(5):
            sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
        ts = []
        for i in range(20):
            flush.fill_(i & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
        e1.record()
        torch.cuda.synchronize()
        print(ov, "l=%d" % l, "plan rows/cta %d splits %d ctas %d sched %s" % (p["rows_per_cta"], p["splits"], p["ctas"],
              p["schedule"][:4]), "step median %.1f us, back-to-back %.1f us" % (
              sorted(ts)[len(ts) // 2], e0.elapsed_time(e1) * 1e3 / 50), flush=True)
M.set_plan_override(0, 0, -1, 0)
