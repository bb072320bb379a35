"""Time every compiled k=8 variant x split count for the BASELINE configs (device events).

python tools/tune.py [--configs 0,1,2,3,4] [--reps 3]  -> prints one JSON line per measurement"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0901_1413_b200 as sg  # noqa: E402
from paper_0901_1413_b200 import _lib, m4rm as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="0,1,2,3,4")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--shapes", default="", help="extra field:m:l:n shapes")
ap.add_argument("--rts", default="1,2,4,8,16")
ap.add_argument("--splits", default="-1,1,2,4,8,16")  # -1 = stream-K
ap.add_argument("--pipes", default="0,1,2")  # schedules; 10 / 11 = fused serial / pipelined
a = ap.parse_args()
dev = torch.device("cuda", 0)
KINFO = M.kernel_info(0)
L = _lib.load()
variants = set()
import ctypes  # noqa: E402
jobs = [bench.CONFIGS[int(x)] for x in a.configs.split(",") if x]
for sh in a.shapes.split(","):  # field:m:l:n, e.g. the per-rank shapes of a sharded run
    if sh:
        fld, m, l, n = sh.split(":")
        jobs.append((f"{fld.upper()} {m}x{l}x{n} k=8", fld, int(m), int(l), int(n)))
for name, field, m, l, n in jobs:
    f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
    C = sg.BitslicedMatrix.zero(f, m, n, device=dev)
    M.set_plan_override(0, 0, -1, 0)
    auto = sg.plan(f, m, l, n, 8)
    best = None
    for rt in [int(x) for x in a.rts.split(",")]:
        for nt in (256, 512):
            for pipe in [int(x) for x in a.pipes.split(",")]:
                for sp in [int(x) for x in a.splits.split(",")]:
                    M.set_plan_override(rt, sp, pipe, nt)
                    try:
                        p = sg.plan(f, m, l, n, 8)
                    except Exception:
                        continue
                    if p["splits"] != sp:
                        continue
                    sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
                    torch.cuda.synchronize()
                    ts = []
                    for _ in range(a.reps):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
                        e1.record()
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1))
                    ms = min(ts)
                    ki = KINFO[p["kernel"]]
                    rec = {"config": name, "field": field, "m": m, "l": l, "n": n, "rt": rt, "threads": nt,
                           "pipe": pipe, "splits": sp, "ms": ms, "muladds_per_s": m * l * n / ms * 1e3,
                           "ctas": p["ctas"], "occ": ki["occupancy"], "regs": ki["regs"]}
                    print(json.dumps(rec), flush=True)
                    if best is None or ms < best["ms"]:
                        best = rec
    M.set_plan_override(0, 0, -1, 0)
    sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    auto["ms"] = min(ts)
    print(json.dumps({"config": name, "BEST": best, "auto_plan": auto}), flush=True)
    del A, B, C
    torch.cuda.empty_cache()
