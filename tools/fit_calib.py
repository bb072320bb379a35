"""Fit the planner's per-variant cost constants (g_calib in csrc/sg_plan.cu) from tools/tune.py output.

python tools/fit_calib.py tune1.jsonl [tune2.jsonl ...]   -> C++ table rows on stdout

Model (the planner's, make_plan_uncached): with slabs = ceil(wc32 / 4), rows = rt * threads,
row groups = ceil(m / rows), k-blocks nb = ceil(l / 8), and SMs = 148,
  split-K:  T = waves * occ' * (bps * blk + cta) + reduce,   waves = ceil(ctas / (SMs * occ)),
            occ' = occ if ctas > SMs else 1, reduce = (splits + 1) R m wc32 4 / 3000 + 8000 (splits > 1)
  stream-K: T = occ * (ceil(U / G) * blk + nseg cta) + (G 2 R rows 16 + R m wc32 4) / 3000 + 8000,
            nseg = min(2, per) + floor(per / nb) segments per CTA,
            G = SMs * occ, U = slabs * row groups * nb
plus FIX = 20000 clocks per product (pre-pass, launches; the same for every variant, so it does not
steer the planner).  Fused variants (pipe 10 / 11, one launch): no pre-pass (FIX - 6000) and the
split-K meeting inside the kernel (1500 instead of a reduction launch's 8000).  T in SM clocks at 1965 MHz; (blk, cta) by least squares on the relative error."""
FIX = 20000.0
FUSED_CREDIT = 6000.0  # fused variants (pipe 10 / 11): one launch instead of pre-pass + product (+ reduce)
import json
import math
import sys
from collections import defaultdict

import numpy as np

SMS, CLK = 148, 1.965e9
R = {"f2": 1, "f3": 2, "gf4": 2, "z4": 2, "f5": 3, "f7": 3, "gf8": 3, "z8": 3}
CODE = {"f2": 0, "f3": 1, "f5": 2, "f7": 3, "gf4": 4, "gf8": 5, "z4": 6, "z8": 7}

recs = []
for path in sys.argv[1:]:
    for line in open(path):
        r = json.loads(line)
        if "BEST" in r or "m" not in r:
            continue
        recs.append(r)
groups = defaultdict(list)
for r in recs:
    groups[(r["field"], r["rt"], r["threads"], r["pipe"])].append(r)

for key in sorted(groups, key=lambda k: (CODE[k[0]], k[1], k[2], k[3])):
    field, rt, nt, pipe = key
    rows_x, rhs, ts = [], [], []
    for r in groups[key]:
        m, l, n, occ, sp = r["m"], r["l"], r["n"], max(1, r["occ"]), r["splits"]
        wc32 = 2 * ((n + 63) // 64)
        slabs, rows = (wc32 + 3) // 4, rt * nt
        rg, nb = (m + rows - 1) // rows, (l + 7) // 8
        T = r["ms"] * 1e-3 * CLK
        if sp == -1:
            G = SMS * occ
            U = slabs * rg * nb
            per = math.ceil(U / G)
            x, y = occ * per, occ * (min(2.0, per) + per // nb)  # segments per CTA, as the planner
            red = (G * 2 * R[field] * rows * 16 + R[field] * m * wc32 * 4) / 3000 + 8000
        else:
            bps = (nb + sp - 1) // sp
            spl = (nb + bps - 1) // bps
            ctas = slabs * rg * spl
            waves = math.ceil(ctas / (SMS * occ))
            mult = occ if ctas / SMS > 1 else 1
            x, y = waves * mult * bps, waves * mult
            if pipe >= 10:  # fused: the split-K meeting inside the kernel, no pre-pass launch
                red = ((spl + 1) * R[field] * m * wc32 * 4 / 3000 + 1500) if spl > 1 else 0.0
                red -= FUSED_CREDIT
            else:
                red = ((spl + 1) * R[field] * m * wc32 * 4 / 3000 + 8000) if spl > 1 else 0.0
        red += FIX
        rows_x.append([x / T, y / T])
        rhs.append((T - red) / T)
        ts.append((x, y, red, T))
    if len(rows_x) < 2:
        continue
    X, b = np.array(rows_x), np.array(rhs)
    (blk, cta), *_ = np.linalg.lstsq(X, b, rcond=None)
    if cta < 0:
        (blk,), *_ = np.linalg.lstsq(X[:, :1], b, rcond=None)
        cta = 0.0
    blk = max(blk, 1.0)
    err = max(abs((x * blk + y * cta + red) - T) / T for x, y, red, T in ts)
    print(f"    {{{CODE[field]}, {rt}, {nt}, {pipe}, {blk:.0f}, {cta:.0f}}},  "
          f"// max err {100 * err:.0f}%, {len(ts)} runs")
