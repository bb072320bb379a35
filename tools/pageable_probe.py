"""Host-buffer product on pageable (numpy) operands through the public API, per-call wall times;
run under SG_HOST_STREAM / SG_HOST_CHUNKS settings to compare pipelines.
python tools/pageable_probe.py [config_index]"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0901_1413_b200 as sg  # noqa: E402

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 1
name, field, m, l, n = bench.CONFIGS[ci]
dev = torch.device("cuda", 0)
f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
An = np.ascontiguousarray(A.planes.cpu().numpy().view(np.uint64))
Bn = np.ascontiguousarray(B.planes.cpu().numpy().view(np.uint64))
Ah = sg.BitslicedMatrix.from_planes(f, An, l, device="cpu")
Bh = sg.BitslicedMatrix.from_planes(f, Bn, n, device="cpu")
if os.environ.get("PINNED"):  # page-locked operands through the same public call
    Ah, Bh = Ah.pin_memory(), Bh.pin_memory()
want = sg.m4rm_multiply(A, B, sg.M4rmParams(8)).planes_numpy()
for _ in range(3):
    C = sg.m4rm_multiply(Ah, Bh, sg.M4rmParams(8))
ts = []
for _ in range(30):
    t0 = time.perf_counter()
    C = sg.m4rm_multiply(Ah, Bh, sg.M4rmParams(8)).planes_numpy()
    ts.append(1e3 * (time.perf_counter() - t0))
ok = bool(np.array_equal(C, want))
print(f"{name} PINNED={os.environ.get('PINNED', '-')} STREAM={os.environ.get('SG_HOST_STREAM', '-')} CHUNKS={os.environ.get('SG_HOST_CHUNKS', '-')}: "
      f"mean {statistics.mean(ts):.3f} median {statistics.median(ts):.3f} min {min(ts):.3f} max {max(ts):.3f} ms ok={ok}")
