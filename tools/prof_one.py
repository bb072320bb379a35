"""Run one BASELINE config's multiply a few times (for ncu / compute-sanitizer).

python tools/prof_one.py --config 1 --reps 3 [--rt R --splits S]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0901_1413_b200 as sg  # noqa: E402
from paper_0901_1413_b200 import m4rm as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--rt", type=int, default=0)
ap.add_argument("--splits", type=int, default=0)
ap.add_argument("--m", type=int, default=0)
ap.add_argument("--pipe", type=int, default=-1)
ap.add_argument("--threads", type=int, default=0)
a = ap.parse_args()
name, field, m, l, n = bench.CONFIGS[a.config]
if a.m:
    m = a.m
dev = torch.device("cuda", 0)
f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
M.set_plan_override(a.rt, a.splits, a.pipe, a.threads)
print(name, sg.plan(f, m, l, n, 8))
for _ in range(a.reps):
    C = sg.m4rm_multiply(A, B, sg.M4rmParams(8))
torch.cuda.synchronize()
M.set_timing(True)
C = sg.m4rm_multiply(A, B, sg.M4rmParams(8))
print(M.last_timing())
print("peaks", M.probe_peaks(0))
