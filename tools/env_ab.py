"""Time configs under several values of one environment switch (SG_TMA, SG_PDL, ...).

python tools/env_ab.py --var SG_TMA --values 0,1 [--configs 0,1,2]"""
import argparse
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--var", required=True)
ap.add_argument("--values", default="0,1")
ap.add_argument("--configs", default="0,1,2,3")
ap.add_argument("--shapes", default="", help="extra field:m:l:n shapes")
a = ap.parse_args()
code = f"""
import sys, torch
sys.path.insert(0, '.')
import bench
import paper_0901_1413_b200 as sg
dev = torch.device('cuda', 0)
jobs = [bench.CONFIGS[int(x)] for x in '{a.configs}'.split(',') if x]
for sh in '{a.shapes}'.split(','):
    if sh:
        f_, m_, l_, n_ = sh.split(':')
        jobs.append((sh, f_, int(m_), int(l_), int(n_)))
for name, field, m, l, n in jobs:
    f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
    C = sg.BitslicedMatrix.zero(f, m, n, device=dev)
    reps = 20 if m * l * n < 1e12 else 3
    for _ in range(3): sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps): sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    print(name, '%.4f ms' % best, flush=True)
    del A, B, C
    torch.cuda.empty_cache()
"""
for v in a.values.split(","):
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=dict(os.environ, **{a.var: v}))
    print(f"{a.var}={v} |", out.stdout.strip().replace("\n", " | "), out.stderr.strip()[-400:], flush=True)
