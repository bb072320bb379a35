"""H2D / D2H bandwidth of pinned buffers allocated with the process bound to each CPU set
(GPU-local CPUs from NVML vs the others): does the pinned buffers' NUMA placement matter?"""
import os
import time

import torch

import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
ncpu = os.cpu_count()
mask = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
local = [c for c in range(ncpu) if (mask[c // 64] >> (c % 64)) & 1]
allc = sorted(os.sched_getaffinity(0))
other = [c for c in allc if c not in local]
print("cpus", ncpu, "local", local[:8], "...", len(local), "other", len(other), flush=True)
os.system("nvidia-smi topo -m 2>/dev/null | head -5; numactl -H 2>/dev/null | head -4; lscpu | grep -i numa")
d = torch.empty(12 << 20, dtype=torch.uint8, device="cuda")
for name, cpus in (("local", local), ("other", other), ("all", allc)):
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    hbuf = torch.empty(12 << 20, dtype=torch.uint8).pin_memory()
    hbuf.fill_(1)
    for _ in range(3):
        d.copy_(hbuf, non_blocking=True)
    torch.cuda.synchronize()
    best_h2d = best_d2h = 1e9
    for _ in range(10):
        t0 = time.perf_counter(); d.copy_(hbuf, non_blocking=True); torch.cuda.synchronize(); best_h2d = min(best_h2d, time.perf_counter() - t0)
        t0 = time.perf_counter(); hbuf.copy_(d, non_blocking=True); torch.cuda.synchronize(); best_d2h = min(best_d2h, time.perf_counter() - t0)
    print(f"{name:6s} cpus={len(cpus)}: H2D {12.58e6 / best_h2d / 1e9:.1f} GB/s  D2H {12.58e6 / best_d2h / 1e9:.1f} GB/s", flush=True)
    del hbuf
