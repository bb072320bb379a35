"""Time configs under SG_PDL=0/1/2 (plain launches / PDL / PDL with early trigger).

python tools/pdl_check.py [--configs 0,1]"""
import argparse
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="0,1,2")
a = ap.parse_args()
code = f"""
import sys, torch
sys.path.insert(0, '.')
import bench
import paper_0901_1413_b200 as sg
dev = torch.device('cuda', 0)
for ci in ({a.configs},):
    name, field, m, l, n = bench.CONFIGS[ci]
    f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
    C = sg.BitslicedMatrix.zero(f, m, n, device=dev)
    for _ in range(5): sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 20)
    print(name, 'back-to-back %.4f ms' % best, flush=True)
"""
for mode in ("0", "1", "2"):
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=dict(os.environ, SG_PDL=mode))
    print("SG_PDL=" + mode, out.stdout.strip().replace("\n", " | "), out.stderr.strip()[-300:], flush=True)
