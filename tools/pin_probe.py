"""H2D bandwidth from page-locked buffers in ONE python process, step by step: a cudaHostAlloc
buffer (ctypes), torch pinned buffers, and what happens after torch CPU ops touch host memory --
is the slow-process H2D variance tied to the torch pinned allocator or to CPU-side activity?
python tools/pin_probe.py"""
import ctypes
import glob
import os
import time

import torch

lib = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
rt = ctypes.CDLL(lib[0])
N = 6291456
dev = torch.empty(N, dtype=torch.uint8, device="cuda")
T0 = time.perf_counter()


def bw(name, ptr):
    s = torch.cuda.current_stream().cuda_stream
    ts = []
    for i in range(25):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rt.cudaMemcpyAsync(ctypes.c_void_p(dev.data_ptr()), ctypes.c_void_p(ptr), ctypes.c_size_t(N), 1, ctypes.c_void_p(s))
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"t={time.perf_counter() - T0:6.2f}s {name:44s} H2D best {N / ts[0] / 1e9:5.1f} median {N / ts[len(ts) // 2] / 1e9:5.1f} GB/s",
          flush=True)


p = ctypes.c_void_p()
assert rt.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(N), 0) == 0
ctypes.memset(p, 3, N)
bw("cudaHostAlloc, memset", p.value)
tp = torch.empty(N, dtype=torch.uint8, pin_memory=True)
bw("torch empty(pin_memory=True), untouched", tp.data_ptr())
ctypes.memset(tp.data_ptr(), 3, N)
bw("  ... after ctypes memset", tp.data_ptr())
bw("cudaHostAlloc again", p.value)
tp.fill_(5)
bw("torch pinned after torch fill_ (CPU threads)", tp.data_ptr())
bw("cudaHostAlloc after torch fill_", p.value)
time.sleep(1.0)
bw("cudaHostAlloc 1 s later", p.value)
bw("torch pinned 1 s later", tp.data_ptr())
x = torch.empty(N, dtype=torch.uint8, device="cuda").cpu().pin_memory()
bw("bench-style .cpu().pin_memory()", x.data_ptr())
bw("cudaHostAlloc after that", p.value)
