"""Per-launch breakdown (serialised events, sg_set_timing) of small products under forced plans.

python tools/small_breakdown.py [--shape f3:1024:1024:1024]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0901_1413_b200 as sg  # noqa: E402
from paper_0901_1413_b200 import m4rm as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="f3:1024:1024:1024")
ap.add_argument("--fused-only", action="store_true")
a = ap.parse_args()
fld, m, l, n = a.shape.split(":")
m, l, n = int(m), int(l), int(n)
dev = torch.device("cuda", 0)
f, A, B = bench.make_inputs(fld, m, l, n, 0, dev, True)
C = sg.BitslicedMatrix.zero(f, m, n, device=dev)
pipes = (10, 11) if a.fused_only else (0, 1, 2, 10, 11)
plans = [(0, 0, -1, 0)] + [(rt, sp, pipe, nt) for rt in (1, 2, 4, 8) for nt in (256,) for pipe in pipes
                           for sp in (4, 8, 16, 18, 32, 37, -1)]
for ov in plans:
    M.set_plan_override(*ov)
    try:
        p = sg.plan(f, m, l, n, 8)
    except Exception:
        continue
    if ov[1] and p["splits"] != ov[1]:
        continue
    for _ in range(3):
        sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
    e1.record()
    torch.cuda.synchronize()
    pipelined = e0.elapsed_time(e1) / 20
    M.set_timing(True)
    best = None
    for _ in range(5):
        sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
        t = M.last_timing()
        if best is None or t["m4rm_ms"] < best["m4rm_ms"]:
            best = t
    M.set_timing(False)
    print(ov, p["rows_per_cta"], p["splits"], p["ctas"], "back-to-back %.1f us | pre %.1f kern %.1f red %.1f us" % (
        1e3 * pipelined, 1e3 * best["transpose_ms"], 1e3 * best["m4rm_ms"], 1e3 * best["reduce_ms"]), flush=True)
M.set_plan_override(0, 0, -1, 0)
