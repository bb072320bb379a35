import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_0901_1413_b200 as sg
from paper_0901_1413_b200 import _lib, m4rm as M
L = _lib.load()
dev = torch.device("cuda", 0)
for ci, splits_list in ((1, (2, 9)), (3, (1,))):
    name, field, m, l, n = bench.CONFIGS[ci]
    f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
    ref = None
    for sched in (1, 2):
        for abl in (0, 8):
            for sp in splits_list:
                L.sg_debug_ablation(abl)
                M.set_plan_override(8, sp, sched, 256)
                try:
                    C = sg.m4rm_multiply(A, B, sg.M4rmParams(8))
                except Exception as e:
                    print(name, sched, abl, sp, "ERR", e); continue
                if ref is None:
                    ref = C.planes.clone()
                ok = torch.equal(C.planes, ref)
                ts = []
                for _ in range(5):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(); sg.m4rm_multiply(A, B, sg.M4rmParams(8)); e1.record(); torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                print(name, "sched", sched, "abl", abl, "splits", sp, "%.3f ms" % min(ts), "exact" if ok else "MISMATCH", flush=True)
    L.sg_debug_ablation(0)
    M.set_plan_override(0, 0, -1, 0)
