"""Headline end-to-end path (sg_m4rm_host, host planes in / C out) on the GPU box: per-step wall
times for pipeline variants, an event trace of one call, and the plain pinned copy bandwidth
beside it.   python tools/e2e_probe.py [config_index]"""
import ctypes
import os
import statistics
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_0901_1413_b200 as sg  # noqa: E402
from paper_0901_1413_b200 import _lib  # noqa: E402


def main():
    ci = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    variant = os.environ.get("VARIANT", "")
    L = _lib.load()
    dev = torch.device("cuda", 0)
    name, field, m, l, n = bench.CONFIGS[ci]
    f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
    Ah, Bh = A.pin_memory().planes, B.pin_memory().planes
    Ch = sg.BitslicedMatrix.pinned_zero(f, m, n).planes
    vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    for _ in range(5):
        _lib.check(L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0))
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        _lib.check(L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0))
        ts.append(1e3 * (time.perf_counter() - t0))
    # plain copies of the same bytes
    Ad, Bd, Cd = A.planes, B.planes, torch.empty_like(Ch, device=dev)

    def t(fn):
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return 1e3 * best
    up = t(lambda: (Ad.copy_(Ah, non_blocking=True), Bd.copy_(Bh, non_blocking=True)))
    down = t(lambda: Ch.copy_(Cd, non_blocking=True))
    print(f"{name} variant={variant or 'default'}: e2e min {min(ts):.3f} median {statistics.median(ts):.3f} "
          f"max {max(ts):.3f} ms | plain H2D A+B {up:.3f} ms ({(Ah.numel() + Bh.numel()) * 8 / up / 1e6:.1f} GB/s), "
          f"D2H C {down:.3f} ms ({Ch.numel() * 8 / down / 1e6:.1f} GB/s)", flush=True)
    if os.environ.get("TRACE"):
        env = dict(os.environ, SG_HOST_TRACE="1")
        env.pop("TRACE")
        subprocess.run([sys.executable, __file__, str(ci)], env=env)


if __name__ == "__main__":
    if os.environ.get("SG_HOST_TRACE"):
        # child: one traced call after warm-up
        L = _lib.load()
        dev = torch.device("cuda", 0)
        name, field, m, l, n = bench.CONFIGS[int(sys.argv[1])]
        f, A, B = bench.make_inputs(field, m, l, n, 0, dev, True)
        Ah, Bh = A.pin_memory().planes, B.pin_memory().planes
        Ch = sg.BitslicedMatrix.pinned_zero(f, m, n).planes
        vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        os.environ.pop("SG_HOST_TRACE")
        for _ in range(5):
            L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0)
        os.environ["SG_HOST_TRACE"] = "1"
        L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, 0)
    else:
        main()
