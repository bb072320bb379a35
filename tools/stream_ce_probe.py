"""H2D / D2H speed of the same pinned copy issued on several CUDA streams of one process: do streams
land on copy engines of different speed?"""
import time

import torch

h = torch.empty(6 << 20, dtype=torch.uint8).pin_memory()
h.fill_(1)
d = torch.empty(6 << 20, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(11)]
res = []
for i, s in enumerate(streams):
    best_h = best_d = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        best_h = min(best_h, time.perf_counter() - t0)
        t0 = time.perf_counter()
        with torch.cuda.stream(s):
            h.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        best_d = min(best_d, time.perf_counter() - t0)
    res.append("s%d %.0f/%.0f" % (i, 6.29e6 / best_h / 1e9, 6.29e6 / best_d / 1e9))
print("GB/s H2D/D2H per stream:", " ".join(res), flush=True)
