"""Ablation timing of the M4RM kernel (results are wrong while ablating; timing only).

Needs the experiments build: `make -C paper_0901_1413_b200/csrc clean all EXTRA=-DSG_EXPERIMENTS`
(sg_debug_ablation and the ablated kernel variants are not in the production library)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0901_1413_b200 as sg  # noqa: E402
from paper_0901_1413_b200 import _lib, m4rm as M  # noqa: E402

L = _lib.load()
dev = torch.device("cuda", 0)
for ci, rt, pipes, masks in ((4, 16, (0, 2), (0, 1, 2, 4)), (3, 8, (2,), (0, 2, 4))):
    name, field, m, l, n = bench.CONFIGS[ci]
    if ci == 4:
        m = 8192
    f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
    C = sg.BitslicedMatrix.zero(f, m, n, device=dev)
    for pipe in pipes:
        for mask in masks:
            if mask == 3 and pipe:
                continue
            L.sg_debug_ablation(mask)
            M.set_plan_override(rt, 1, pipe, 256)
            M.set_timing(True)
            ts = []
            for _ in range(3):
                sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=C)
                ts.append(M.last_timing()["m4rm_ms"])
            M.set_timing(False)
            print(f"{name} m={m} rt={rt} pipe={pipe} ablate={mask}: kernel {min(ts):.3f} ms", flush=True)
    L.sg_debug_ablation(0)
    M.set_plan_override(0, 0, -1, 0)
