"""Per-process H2D variance vs CPU affinity: the CPU / NUMA node the process is on when it
allocates its pinned buffers and the headline host-buffer e2e of that process.
python tools/affinity_probe.py [pin | late | lateN | allocpin | callpin]   (pin: whole process on
CPU 0 from the start; late: only the calling thread, after CUDA init, on its current CPU or CPU N;
allocpin: pinned only while the host buffers are allocated; callpin: pinned only for the calls)"""
import ctypes
import os
import statistics
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def cpu_now():
    with open("/proc/self/stat") as f:
        return int(f.read().split(")")[1].split()[36])


def node_of(cpu):
    for d in os.listdir("/sys/devices/system/node"):
        if d.startswith("node") and os.path.exists(f"/sys/devices/system/node/{d}/cpu{cpu}"):
            return int(d[4:])
    return -1


def gpu_cpus():
    """CPU list the driver reports as local to GPU 0 (nvidia-smi topo -m 'CPU Affinity')."""
    try:
        out = subprocess.run(["nvidia-smi", "topo", "-C", "-i", "0"], capture_output=True, text=True).stdout
        lst = out.strip().split(":")[-1].strip()
        cpus = set()
        for part in lst.split(","):
            if "-" in part:
                a, b = part.split("-")
                cpus.update(range(int(a), int(b) + 1))
            elif part.strip():
                cpus.add(int(part))
        return cpus
    except Exception:  # noqa: BLE001
        return set()


MODE = sys.argv[1] if len(sys.argv) > 1 else ""
if MODE == "pin":  # the whole process (every thread created later inherits it) on CPU 0
    os.sched_setaffinity(0, {0})
import torch  # noqa: E402

import bench  # noqa: E402
from paper_0901_1413_b200 import _lib  # noqa: E402

L = _lib.load()
dev = torch.device("cuda", 0)
name, field, m, l, n = bench.CONFIGS[1]
f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
FULL = os.sched_getaffinity(0)
if MODE in ("warm", "allocpin1"):  # create torch's CPU thread pool first, on every CPU
    torch.ones(1 << 22).add_(1)
NT0 = torch.get_num_threads()
if MODE == "allocpin1":  # pinned, single-threaded host copies while the buffers are filled
    torch.set_num_threads(1)
if MODE.startswith("late") or MODE in ("allocpin", "allocpin1"):  # the calling thread on one CPU
    os.sched_setaffinity(0, {int(MODE[4:]) if MODE.startswith("late") and MODE[4:] else cpu_now()})
c0 = cpu_now()
Ah, Bh = A.planes.cpu().pin_memory(), B.planes.cpu().pin_memory()
Ch = torch.empty((f.bits, m, (n + 63) // 64), dtype=torch.int64).pin_memory()
if MODE in ("allocpin", "allocpin1"):  # pinned only while the host buffers are allocated and filled
    os.sched_setaffinity(0, FULL)
    torch.set_num_threads(NT0)
if MODE == "callpin":  # buffers allocated unpinned, the calls pinned
    os.sched_setaffinity(0, {cpu_now()})
vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
ts = []
for i in range(25):
    t0 = time.perf_counter()
    _lib.check(L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0))
    ts.append(1e3 * (time.perf_counter() - t0))
nodes = sorted({node_of(c) for c in os.sched_getaffinity(0)})
print(f"alloc on cpu {c0} (node {node_of(c0)}), now cpu {cpu_now()} (node {node_of(cpu_now())}); affinity nodes "
      f"{nodes}; gpu-local cpus {min(gpu_cpus(), default=-1)}..{max(gpu_cpus(), default=-1)}; "
      f"e2e median {statistics.median(ts[5:]):.3f} ms", flush=True)
