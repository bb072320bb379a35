#!/usr/bin/env python
"""bench.py -- field multiply-adds per second of the B200 bitsliced M4RM product.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` prints ONE JSON line on
rank 0.  N > 1 runs under torch.distributed.run (one rank per GPU, NCCL).

Metric (BASELINE.json): field mul-adds/s = m*l*n / t for C = A B, with the fraction of the
binding roofline (LOP3 integer-logic issue or shared-memory bandwidth).
Workload (N=1): BASELINE.json configs[1], F5 4096x4096x4096, k=8; the other configs are
reported under "per_config".  A step is one C = A B of the workload on inputs resident in
HBM; with N GPUs every rank multiplies its own 4096-row (configs' m-row) slab of A by B,
which rank 0 broadcasts over NCCL inside the step (weak scaling: per-GPU work fixed).
L2 is flushed (256 MiB write) before every timed step; device time with CUDA events, summed
over K steps, max over ranks.

`--impl reference` times the reference's CPU path -- the oracle port of it (oracle/, C with
pthreads on all host cores; the reference itself is Python and does not travel to the box)
-- on a bounded row sample of the same workload, extrapolated to the full product.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# (name, field, m, l, n): BASELINE.json configs 0..4
CONFIGS = [
    ("F3 1024x1024x1024 k=8", "f3", 1024, 1024, 1024),
    ("F5 4096x4096x4096 k=8", "f5", 4096, 4096, 4096),
    ("GF(4) 8192x8192x8192 k=8", "gf4", 8192, 8192, 8192),
    ("F7 16384x8192x16384 k=8", "f7", 16384, 8192, 16384),
    ("F3 32768x32768x32768 k=8", "f3", 32768, 32768, 32768),
]
HEADLINE = 1
# configs whose BASELINE text shards a fixed problem over the GPUs ("row-sharded over 1/2/4/8
# GPUs"): strong scaling; the others run the same per-GPU problem on every rank (weak scaling)
STRONG = {"F7 16384x8192x16384 k=8", "F3 32768x32768x32768 k=8"}
# dram__bytes_read.sum + dram__bytes_write.sum of the M4RM kernel per launch, from the committed
# `ncu --set full` captures (profiles/*_traffic.json, written by tools/traffic_from_ncu.py)
TRAFFIC = {}
for _f in sorted(os.listdir(os.path.join(ROOT, "profiles"))) if os.path.isdir(os.path.join(ROOT, "profiles")) else []:
    if _f.endswith("_traffic.json"):
        with open(os.path.join(ROOT, "profiles", _f)) as _fh:
            TRAFFIC.update(json.load(_fh))
# ALU-pipe and shared-memory-wavefront utilization of the M4RM kernel from the same captures
# (profiles/*_pipes.json, tools/pipes_from_ncu.py): what the kernel is actually bound by
PIPES = {}
for _f in sorted(os.listdir(os.path.join(ROOT, "profiles"))) if os.path.isdir(os.path.join(ROOT, "profiles")) else []:
    if _f.endswith("_pipes.json"):
        with open(os.path.join(ROOT, "profiles", _f)) as _fh:
            PIPES.update(json.load(_fh))
MEASURED = {}
if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")):
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as _fh:
        MEASURED = json.load(_fh)
METRIC = "field mul-adds/sec (m*l*n/t) for C=A*B over F3/F5/F7/GF(4), % of roofline"
UNIT = "mul-adds/s"

# Algorithmic work per field mul-add for the accumulate phase: LOP3 count of
# the reference formulas and shared-memory table bytes; plus the table build once per GPU.
LOP3_PER_MULADD = {"f2": 1 / 256, "f3": 9 / 256, "f5": 42 / 256, "f7": 32 / 256, "gf4": 3 / 256}
# ... and the LOP3 count of this kernel's own networks (csrc/sg_field.cuh)
OWN_LOP3_PER_MULADD = {"f2": 1 / 256, "f3": 6 / 256, "f5": 20 / 256, "f7": 18 / 256, "gf4": 3 / 256}
SMEM_PER_MULADD = {"f2": 4 / 256, "f3": 16 / 256, "f5": 36 / 256, "f7": 36 / 256, "gf4": 16 / 256}
TABLE_LOP3_PER_WORD = {"f2": 1, "f3": 5, "f5": 12, "f7": 10, "gf4": 2}  # one field add, 32-bit word
PLANES = {"f2": 1, "f3": 2, "f5": 3, "f7": 3, "gf4": 2}
ORDER = {"f2": 2, "f3": 3, "f5": 5, "f7": 7, "gf4": 4, "gf8": 8, "z4": 4, "z8": 8}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- our arm
def make_inputs(field, m, l, n, rank, device, with_b):
    import torch
    import paper_0901_1413_b200 as sg
    f = sg.by_name(field)
    g = torch.Generator(device=device)
    g.manual_seed(1000 + rank)
    A = torch.randint(0, ORDER[field], (m, l), dtype=torch.uint8, device=device, generator=g)
    Am = sg.BitslicedMatrix.from_dense(f, A, device=device)
    del A
    if with_b:
        g.manual_seed(1)
        B = torch.randint(0, ORDER[field], (l, n), dtype=torch.uint8, device=device, generator=g)
        Bm = sg.BitslicedMatrix.from_dense(f, B, device=device)
        del B
    else:
        Bm = sg.BitslicedMatrix.zero(f, l, n, device=device)
    return f, Am, Bm


def run_config(cfg, args, world, rank, device, peaks, e2e=False):
    import torch
    import torch.distributed as dist
    import paper_0901_1413_b200 as sg
    from paper_0901_1413_b200 import m4rm as M

    name, field, m, l, n = cfg
    strong = name in STRONG and world > 1
    if strong:  # BASELINE.json configs 3-4: A/C rows sharded over the GPUs (fixed total work)
        from paper_0901_1413_b200.dist import row_partition
        r0, r1 = row_partition(m, world)[rank]
        m_total, m = m, r1 - r0
    f, A, B = make_inputs(field, m, l, n, rank, device, with_b=(rank == 0))
    C = sg.BitslicedMatrix.zero(f, m, n, device=device)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    params = sg.M4rmParams(8)

    from paper_0901_1413_b200 import dist as sgdist
    chunks = sgdist.default_chunks(f, l, n)

    def step():
        if world > 1:  # B broadcast from rank 0 in row blocks, overlapped with the chunk products
            sgdist.sharded_multiply(A, B if rank == 0 else None, f, l, n, src=0, chunks=chunks, return_b=False)
        else:
            sg.m4rm_multiply(A, B, params, out=C)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = M.launch_count()
    with ClockSampler(device.index or 0) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # evict L2 (126 MB) between timed steps; untimed
            ev[i][0].record()
            step()
            ev[i][1].record()
        torch.cuda.synchronize()
    launches = M.launch_count() - launches0
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([total_ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    work = float(m) * l * n
    value = (float(m_total) * l * n if strong else world * work) / (ms_per_step * 1e-3)

    # dominant-kernel duration (events around each internal launch, on the launching stream)
    M.set_timing(True)
    kern, tr, red = [], [], []
    for i in range(max(3, min(args.steps, 10))):
        flush.fill_(i & 0xFF)
        sg.m4rm_multiply(A, B, params, out=C)
        lt = M.last_timing()
        kern.append(lt["m4rm_ms"]); tr.append(lt["transpose_ms"]); red.append(lt["reduce_ms"])
    M.set_timing(False)
    k_ms = statistics.median(kern)
    plan = sg.plan(f, m, l, n, 8)

    # roofline of the M4RM kernel: min over the LOP3 and LDS rooflines
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    clk_hz = peaks["clock_mhz_for_peak"] * 1e6
    p_lop3 = peaks["lop3_per_clk_per_sm"] * sms * clk_hz
    p_smem = peaks["lds_bytes_per_clk_per_sm"] * sms * clk_hz
    words32 = 2 * ((n + 63) // 64)
    table_lop3 = (l / 8.0) * 255 * words32 * TABLE_LOP3_PER_WORD[field]

    def roofline(c_lop3):
        lop3 = work * c_lop3 + table_lop3
        smem = work * SMEM_PER_MULADD[field]
        lop3_t, smem_t = lop3 / p_lop3, smem / p_smem
        if lop3_t >= smem_t:
            r = {"bound": "lop3 (integer-logic pipe)", "achieved": lop3 / (k_ms * 1e-3) / 1e12, "peak": p_lop3 / 1e12,
                 "unit": "TLOP3/s"}
        else:
            r = {"bound": "smem (LDS bandwidth)", "achieved": smem / (k_ms * 1e-3) / 1e12, "peak": p_smem / 1e12,
                 "unit": "TB/s"}
        r["frac"] = r["achieved"] / r["peak"]
        r["roofline_muladds_per_s"] = work / max(lop3_t, smem_t)
        return r

    roof = roofline(LOP3_PER_MULADD[field])
    own = roofline(OWN_LOP3_PER_MULADD[field])
    roof["definition"] = ("SURVEY.md 8d: algorithmic LOP3 = the reference formulas' SASS count per mul-add "
                          "(+ one table build per GPU), LDS bytes = table lookups; binding = the slower of the two")
    roof["own_ops"] = {"bound": own["bound"], "frac": own["frac"], "roofline_muladds_per_s": own["roofline_muladds_per_s"],
                       "definition": "same, with this kernel's own LOP3 networks (fewer ops than the reference's)"}
    roof["traffic"] = TRAFFIC.get(name)
    roof["traffic_source"] = TRAFFIC.get("_source") if name in TRAFFIC else None
    roof["measured_pipes"] = PIPES.get(name)
    roof["measured_pipes_source"] = PIPES.get("_source") if name in PIPES else None
    roof["kernel_ms"] = k_ms
    roof["kernel_share_of_step"] = k_ms / ms_per_step if world == 1 else None
    roof["achieved_muladds_per_s"] = work / (k_ms * 1e-3)
    roof["peak_source"] = ("sg_probe_peaks on this GPU: %.1f LOP3/clk/SM, %.1f LDS B/clk/SM, x %d SMs x %.0f MHz (%s)"
                           % (peaks["lop3_per_clk_per_sm"], peaks["lds_bytes_per_clk_per_sm"], sms,
                              peaks["clock_mhz_for_peak"], peaks["clock_note"]))
    out = {"value": value, "ms_per_step": ms_per_step, "gpu_launches": launches, "clocks": clk.summary(),
           "scaling": "strong" if name in STRONG else "weak", "m_per_gpu": m,
           "roofline": roof, "plan": plan, "transpose_ms": statistics.median(tr), "reduce_ms": statistics.median(red)}

    if e2e:
        out["e2e"] = run_e2e(f, A, B, m, l, n, args, world, device)
    del A, B, C, flush
    torch.cuda.empty_cache()
    return out


def run_pack_unpack(device, field="f3", m=16384, n=32768, reps=5):
    """HBM roofline of the pack / unpack kernels (dense uint8 residues <-> bit planes) on a matrix
    larger than L2: algorithmic bytes = m n (1 + R/8) per call, against MEASURED_PEAKS.json."""
    import ctypes

    import torch
    import paper_0901_1413_b200 as sg
    from paper_0901_1413_b200 import _lib

    L = _lib.load()
    f = sg.by_name(field)
    dense = torch.randint(0, ORDER[field], (m, n), dtype=torch.uint8, device=device)
    planes = torch.empty((f.bits, m, (n + 63) // 64), dtype=torch.int64, device=device)
    out = torch.empty_like(dense)
    st = _lib.current_stream_handle(device)
    vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    pack = lambda: _lib.check(L.sg_pack(f.code, vp(dense), m, n, n, vp(planes), st))  # noqa: E731
    unpack = lambda: _lib.check(L.sg_unpack(f.code, vp(planes), m, n, vp(out), n, st))  # noqa: E731
    res = {}
    for name, fn in (("pack", pack), ("unpack", unpack)):
        fn()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[name + "_ms"] = min(ts)
    assert torch.equal(out, dense), "pack/unpack round trip"
    nbytes = m * n * (1 + f.bits / 8.0)
    peak = MEASURED.get("hbm_gbs")
    for name in ("pack", "unpack"):
        res[name + "_gbps"] = nbytes / (res[name + "_ms"] * 1e-3) / 1e9
        res[name + "_frac"] = res[name + "_gbps"] / peak if peak else None
    res.update({"workload": f"{field.upper()} {m}x{n} dense uint8 <-> {f.bits} planes",
                "bytes_per_call": nbytes, "peak_gbps": peak,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)",
                "note": "each call includes the range-check flag read-back (a few us)"})
    del dense, planes, out
    torch.cuda.empty_cache()
    return res


def e2e_for(cfg, args, world, rank, device):
    """run_e2e on fresh inputs of `cfg` (rows sharded as in run_config for the strong configs)."""
    import torch
    name, field, m, l, n = cfg
    if name in STRONG and world > 1:
        from paper_0901_1413_b200.dist import row_partition
        r0, r1 = row_partition(m, world)[rank]
        m = r1 - r0
    f, A, B = make_inputs(field, m, l, n, rank, device, with_b=(rank == 0))
    out = run_e2e(f, A, B, m, l, n, args, world, device)
    del A, B
    torch.cuda.empty_cache()
    return out


def run_e2e(f, A, B, m, l, n, args, world, device):
    """Same metric end to end through the public API with host buffers (pinned memory).

    N = 1: the C-ABI host entry point sg_m4rm_host (H2D of A and B, multiply, D2H of C, copies
    pipelined by row chunks).  N > 1: the multi-GPU public path -- rank 0 uploads B and
    broadcasts it (NCCL), every rank uploads its A rows, multiplies (m4rm_multiply) and
    downloads its C rows.
    """
    import ctypes

    import torch
    import torch.distributed as dist
    import paper_0901_1413_b200 as sg
    from paper_0901_1413_b200 import _lib

    L = _lib.load()
    rank = dist.get_rank() if world > 1 else 0
    Ah = A.planes.cpu().pin_memory()
    Bh = B.planes.cpu().pin_memory()
    Ch = torch.empty((f.bits, m, (n + 63) // 64), dtype=torch.int64).pin_memory()
    vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    dev = device.index or 0
    Bd = torch.empty_like(B.planes)

    def one():
        if world == 1:
            _lib.check(L.sg_m4rm_host(f.code, vp(Ah), vp(Bh), vp(Ch), m, l, n, 8, dev))
            return
        from paper_0901_1413_b200 import dist as sgdist
        Bm = None
        if rank == 0:
            Bd.copy_(Bh, non_blocking=True)
            Bm = sg.BitslicedMatrix(f, l, n, Bd)
        Ad = Ah.to(device, non_blocking=True)
        C, _ = sgdist.sharded_multiply(sg.BitslicedMatrix(f, m, l, Ad), Bm, f, l, n, src=0,
                                       chunks=sgdist.default_chunks(f, l, n), return_b=False)
        Ch.copy_(C.planes, non_blocking=True)
        torch.cuda.synchronize()

    s0 = L.sg_host_streamed_count()
    for _ in range(max(1, args.warmup)):
        one()
    if world > 1:
        dist.barrier()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        one()
        times.append(time.perf_counter() - t0)
    total = torch.tensor([sum(times)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(total, op=dist.ReduceOp.MAX)
    per = float(total.item()) / args.steps
    if os.environ.get("SG_BENCH_E2E_TIMES"):  # experiments: every step's wall time
        log("e2e step ms: " + " ".join("%.3f" % (1e3 * t) for t in times))
    h2d = Ah.numel() * 8 + (Bh.numel() * 8 if rank == 0 else 0)
    extra = {}
    if world == 1:
        # the host-path result must equal the device path's (outside the timed region)
        extra["verified_vs_device_path"] = bool(torch.equal(sg.m4rm_multiply(A, B).planes.cpu(), Ch))
        extra["streamed_b_calls"] = int(L.sg_host_streamed_count() - s0)
        # context: this process's plain pinned copy bandwidth right now (PCIe on a shared host varies)
        Ad = torch.empty_like(Ah, device=device)

        def copy_ms(dst, src):
            best = 1e9
            for _ in range(5):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                dst.copy_(src, non_blocking=True)
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
            return best

        nb = Ah.numel() * 8
        extra["pcie_gbs"] = {"h2d": nb / copy_ms(Ad, Ah) / 1e9, "d2h": nb / copy_ms(Ah, Ad) / 1e9,
                             "note": "one %.1f MB pinned copy each way, best of 5, after the timed loop" % (nb / 1e6)}
        del Ad
    if world == 1:  # the per-step spread (PCIe on the shared host varies; value is the mean)
        extra["step_ms_min"] = 1e3 * min(times)
        extra["step_ms_median"] = 1e3 * statistics.median(times)
    return {"value": world * float(m) * l * n / per, "unit": UNIT, "ms_per_step": per * 1e3,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(Ch.numel() * 8), **extra,
            "path": ("sg_m4rm_host (C ABI; pinned host planes; A and C in row pieces, the first piece's product "
                     "consuming B's k-chunks as they land, D2H of each piece behind its product)"
                     if world == 1 else "rank-0 H2D of B + broadcast in row blocks overlapped with the chunk products "
                     "(dist.sharded_multiply), per-rank H2D of A rows, D2H of C rows (wall clock, max over ranks)")}


# ----------------------------------------------------------------------------- CPU (oracle port)
def cpu_estimate(field, m, l, n, sample_rows, threads):
    """Time the restated reference path (oracle/, C + pthreads) on a row sample and extrapolate.

    Each of `threads` workers builds every k-block table (as the reference's row-partition
    contract does) and processes rows_per_thread rows.  Two sample sizes give the
    table-build time a and the per-row time b; the full product costs a + b * ceil(m / threads).
    """
    import numpy as np

    import oracle
    rng = np.random.default_rng(0)
    rows = max(threads * sample_rows, threads)
    A = rng.integers(0, ORDER[field], size=(rows, l), dtype=np.uint8)
    B = rng.integers(0, ORDER[field], size=(l, n), dtype=np.uint8)
    Ap, Bp = oracle.pack(field, A), oracle.pack(field, B)

    def run(r_per_thread):
        rr = r_per_thread * threads
        t0 = time.perf_counter()
        oracle.m4rm(field, Ap[:, :rr], Bp, l, n, 8, threads=threads, canonical=False)
        return time.perf_counter() - t0

    t1 = min(run(1) for _ in range(2))
    ts = min(run(sample_rows) for _ in range(2)) if sample_rows > 1 else t1
    b = max((ts - t1) / max(sample_rows - 1, 1), 1e-9)
    a = max(t1 - b, 0.0)
    full = a + b * -(-m // threads)
    return {"value": float(m) * l * n / full, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": (f"oracle/sg_oracle.c M4RM (restated reference path, k=8) on {threads} threads: full table "
                       f"builds for all {-(-l // 8)} k-blocks of a {l}x{n} B, with 1 and {sample_rows} A rows per thread "
                       f"(best of 2 each: {t1:.3f} s, {ts:.3f} s); extrapolated linearly to {m} rows"),
            "est_seconds_full": full}


def cpu_sample_rows(field, l, n, threads, budget_s=8.0):
    """Pick rows per thread so one sample run takes roughly budget_s (per-row cost model)."""
    ops_per_row = (l / 8.0) * (n / 64.0) * {"f2": 2, "f3": 14, "f5": 80, "f7": 60, "gf4": 8}[field]
    rate = 1.5e9  # 64-bit word-ops per second per core, rough
    table_s = (l / 8.0) * 255 * (n / 64.0) * {"f2": 2, "f3": 8, "f5": 24, "f7": 20, "gf4": 3}[field] / rate
    r = int(max(2, (budget_s - table_s) / max(ops_per_row / rate, 1e-9)))
    return min(r, 512)


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    name, field, m, l, n = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    sample = cpu_sample_rows(field, l, n, threads, budget_s=max(2.0, 60.0 / max(args.steps + args.warmup, 1)))
    for _ in range(args.warmup):
        cpu_estimate(field, m, l, n, 1, threads)
    vals = []
    last = None
    for _ in range(args.steps):
        last = cpu_estimate(field, m, l, n, sample, threads)
        vals.append(last["value"])
    value = statistics.median(vals)
    ms = float(m) * l * n / value * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64 (bitsliced boolean words)", "data": "synthetic",
            "config": {"workload": name, "field": field, "m": m, "l": l, "n": n, "k": 8,
                       "parallelism": f"{threads} host threads, rows sharded"},
            "cpu_baseline": {**last, "value": value},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- main
def relaunch_cmd(gpus, argv, port):
    """torch.distributed.run command that runs this script with one rank per GPU."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def relaunch(gpus, argv):
    """`bench.py --gpus N` without a launcher: re-run under torch.distributed.run (NCCL ranks)."""
    import socket
    if not os.environ.get("SG_BENCH_BACKEND"):
        try:
            import torch
            have = torch.cuda.device_count()
        except Exception:  # noqa: BLE001
            have = 0
        if have < gpus:
            log(f"error: --gpus {gpus} needs {gpus} visible GPUs, this host has {have}")
            return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator lines on stderr: proof of the NCCL ranks
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    log("bench.py: launching %d ranks: %s" % (gpus, " ".join(relaunch_cmd(gpus, argv, port))))
    return subprocess.call(relaunch_cmd(gpus, argv, port), env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=HEADLINE, help="index into BASELINE.json configs")
    ap.add_argument("--no-per-config", action="store_true", help="skip the other BASELINE configs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline")
    args = ap.parse_args()
    if args.gpus < 1:
        log(f"error: --gpus must be >= 1 (got {args.gpus})")
        sys.exit(2)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # not under a launcher: start one rank per GPU ourselves (the same command the driver runs)
        sys.exit(relaunch(args.gpus, sys.argv[1:]))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"error: --gpus {args.gpus} but WORLD_SIZE={world}: the run would not measure {args.gpus} GPUs")
        sys.exit(2)

    if args.impl == "reference":
        sys.exit(run_reference(args, world, rank))

    import torch
    import torch.distributed as dist
    from paper_0901_1413_b200 import m4rm as M

    if args.warmup < 3:
        log("warning: the contract needs >= 3 warm-up steps; using 3")
        args.warmup = 3
    # SG_BENCH_BACKEND=gloo: functional check of the N > 1 code path on a one-GPU box (ranks share
    # cuda:0, collectives through gloo); its numbers are not measurements.
    backend = os.environ.get("SG_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)

    pk = M.probe_peaks(local)
    peaks = {"lop3_per_clk_per_sm": pk["lop3_per_clk_per_sm"], "lds_bytes_per_clk_per_sm": pk["lds_bytes_per_clk_per_sm"],
             "probe_sm_mhz": pk["sm_mhz"], "clock_mhz_for_peak": 1965.0,
             "clock_note": "max SM clock, conservative; probe ran at %.0f MHz" % pk["sm_mhz"]}

    head = CONFIGS[args.config]
    res = run_config(head, args, world, rank, device, peaks, e2e=False)
    per_config = {}
    if not args.no_per_config:
        for i, cfg in enumerate(CONFIGS):
            if i == args.config:
                continue
            r = run_config(cfg, args, world, rank, device, peaks, e2e=False)
            per_config[cfg[0]] = {"value": r["value"], "ms_per_step": r["ms_per_step"],
                                  "roofline_frac": r["roofline"]["frac"], "bound": r["roofline"]["bound"],
                                  "own_ops_frac": r["roofline"]["own_ops"]["frac"],
                                  "scaling": r["scaling"], "m_per_gpu": r["m_per_gpu"],
                                  "kernel_ms": r["roofline"]["kernel_ms"],
                                  "achieved_muladds_per_s": r["roofline"]["achieved_muladds_per_s"],
                                  "plan": r["plan"], "clocks": r["clocks"]}
    pack_unpack = run_pack_unpack(device) if not args.no_per_config else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        name, field, m, l, n = head
        threads = os.cpu_count() or 1
        cpu = cpu_estimate(field, m, l, n, cpu_sample_rows(field, l, n, threads, budget_s=10.0), threads)
    # e2e last, on fresh inputs of the headline config: the host<->device copies are the part of
    # this run most exposed to the shared host's PCIe, so they go after everything else
    res["e2e"] = e2e_for(head, args, world, rank, device)
    if world == 1 and not args.no_per_config:
        # the host-buffer path on the other configs too (5 steps each; informational)
        class Short:
            steps, warmup = min(args.steps, 5), 3
        for i, cfg in enumerate(CONFIGS):
            if i != args.config and cfg[0] in per_config:
                e = e2e_for(cfg, Short, world, rank, device)
                per_config[cfg[0]]["e2e"] = {k: e[k] for k in ("value", "ms_per_step", "verified_vs_device_path",
                                                               "streamed_b_calls", "pcie_gbs")}
    if world > 1:
        dist.barrier()
    if rank == 0:
        name, field, m, l, n = head
        line = {"metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
                "scaling": res["scaling"] if world > 1 else "weak", "vs_baseline": None,
                "dtype": "u32 (bitsliced boolean words)",
                "data": "synthetic (seeded uniform residues, torch.randint on device)",
                "config": {"workload": name, "field": field, "m_per_gpu": res["m_per_gpu"], "m_total":
                           m * world if res["scaling"] == "weak" else m, "l": l, "n": n, "k": 8,
                           "parallelism": (f"rows of A/C sharded over {world} GPUs, B broadcast from rank 0 by "
                                           f"{backend.upper()} inside every step (row blocks overlapped with the "
                                           "chunk products)" if world > 1 else "1 GPU"),
                           "l2": "flushed (256 MiB write) before every timed step"},
                "e2e": res["e2e"], "gpu_launches": res["gpu_launches"], "clocks": res["clocks"],
                "roofline": res["roofline"], "plan": res["plan"], "cpu_baseline": cpu,
                "step_breakdown_ms": {"index_prepass": res["transpose_ms"], "m4rm": res["roofline"]["kernel_ms"],
                                      "reduce": res["reduce_ms"],
                                      "note": "events around each launch (serialised, sg_set_timing)"},
                "peaks_probe": peaks, "per_config": per_config, "pack_unpack": pack_unpack}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
