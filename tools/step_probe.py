"""Bench-style step time of one product under forced plans: every step = L2 flush (256 MiB
write, untimed) then CUDA events around one m4rm_multiply, all steps queued back to back as in
bench.py's timed loop.   python tools/step_probe.py --shape f3:1024:1024:1024 [--plans rt,sp,pipe,nt;...]"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0901_1413_b200 as sg  # noqa: E402
from paper_0901_1413_b200 import m4rm as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="f3:1024:1024:1024")
ap.add_argument("--plans", default="")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--json", action="store_true", help="tools/tune.py-style JSON lines (for tools/fit_calib.py)")
ap.add_argument("--grid", action="store_true", help="fused and unfused variants x split counts")
a = ap.parse_args()
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
KINFO = M.kernel_info(0)


def run_shape(shape):
  fld, m, l, n = shape.split(":")
  m, l, n = int(m), int(l), int(n)
  f, A, B = bench.make_inputs(fld, m, l, n, 0, dev, True)
  C = sg.BitslicedMatrix.zero(f, m, n, device=dev)
  plans = [(0, 0, -1, 0)]
  if a.plans:
    plans += [tuple(int(x) for x in p.split(",")) for p in a.plans.split(";")]
  elif a.grid:
    plans += [(rt, sp, pipe, 256) for rt in (1, 2, 4) for pipe in (10, 11) for sp in (1, 2, 4, 8, 12, 16, 24, 32)]
    plans += [(rt, sp, pipe, nt) for rt in (2, 4, 8, 16) for pipe in (0, 1, 2) for nt in (256, 512)
              for sp in (1, 2, 4, 8, 16, -1)]
  else:
    plans += [(rt, sp, pipe, 256) for rt in (1, 2, 4) for pipe in (10, 11) for sp in (8, 9, 12, 16, 18, 24, 32, 36)]
    plans += [(rt, sp, pipe, 256) for rt in (1, 2, 4) for pipe in (0, 1) for sp in (8, 9, 16)]
  ref = None
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
    if ref is None:
        ref = C.planes.clone()
    assert torch.equal(C.planes, ref), ov
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    for i in range(a.steps):
        flush.fill_(i & 0xFF)
        ev[i][0].record()
        sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
        ev[i][1].record()
    torch.cuda.synchronize()
    ts = [1e3 * x.elapsed_time(y) for x, y in ev]
    if a.json:
      ki = KINFO[p["kernel"]]
      print(json.dumps({"config": shape, "field": fld, "m": m, "l": l, "n": n, "rt": ki["rt"], "threads": ki["threads"],
                        "pipe": ki["schedule"], "splits": p["splits"], "ms": statistics.median(ts) * 1e-3,
                        "ctas": p["ctas"], "occ": ki["occupancy"], "regs": ki["regs"], "auto": ov[0] == 0}), flush=True)
    else:
      print(f"{str(ov):22s} rows {p['rows_per_cta']:5d} splits {p['splits']:3d} ctas {p['ctas']:4d} "
            f"{p['schedule'][:22]:22s} step median {statistics.median(ts):6.1f} min {min(ts):6.1f} us", flush=True)
  M.set_plan_override(0, 0, -1, 0)
  del A, B, C
  torch.cuda.empty_cache()


for sh in a.shape.split(","):
  run_shape(sh)
