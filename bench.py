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

# Algorithmic shared-memory bytes per field mul-add: the table lookups, NI lookups x
# R planes x 16 B per (row, k-block of 8, 128-column slab) -- F3 / GF(4) 2 x 2, F5 / F7 3 x 3, F2 1 x 1.
SMEM_PER_MULADD = {"f2": 4 / 256, "f3": 16 / 256, "f5": 36 / 256, "f7": 36 / 256, "gf4": 16 / 256}
# ... and what this kernel's lookups move: GF(4) at k = 8 reads Karatsuba tables (T0[g0], T1[g1],
# T0^T1[g0^g1]: three one-plane lookups instead of two two-plane ones), 12 / 256 B per mul-add
KERNEL_SMEM_PER_MULADD = dict(SMEM_PER_MULADD, gf4=12 / 256)
# Integer-pipe work per (row, k-block, slab): counted from this kernel's compiled SASS -- the lookup
# warps' main loop / RT (profiles/*_sass_mix.json, tools/sass_mix.py; LOP3 + PRMT + LEA + ... on the
# ALU pipe, IMAD on the FMA pipe, LDS).  The table build runs on the builder warps and is not counted
# (one build per k-block per CTA; "once per GPU" in SURVEY.md 8d is below 1 % of the lookups).
SASS_MIX = {}
for _f in sorted(os.listdir(os.path.join(ROOT, "profiles"))) if os.path.isdir(os.path.join(ROOT, "profiles")) else []:
    if _f.endswith("_sass_mix.json"):
        with open(os.path.join(ROOT, "profiles", _f)) as _fh:
            SASS_MIX.update(json.load(_fh))
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


def m4rm_roofline(name, field, m, l, n, k_ms, plan, peaks, device):
    """Roofline of the M4RM kernel: it is bound by the integer (ALU) pipe or by
    shared-memory bandwidth.  Per launch:
      * smem: algorithmic table-lookup bytes = m l n x SMEM_PER_MULADD (NI x R x 16 B per row,
        k-block and 128-column slab), against the measured LDS peak;
      * alu: the integer-pipe instructions this kernel's lookup loop issues per (row, k-block,
        slab), counted from its SASS (SASS_MIX), x m x k-blocks x slabs, against the measured
        LOP3 (ALU-pipe) peak.
    frac = the larger of the two fractions (the binding one); both are <= 1 by construction (the
    builder warps' table stores and adds, index loads and address math come on top).  ncu's
    pipe utilizations of the same kernel (all of its instructions and wavefronts) are reported
    beside them from the committed captures."""
    import ctypes

    import torch
    from paper_0901_1413_b200 import _lib
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    clk_hz = peaks["clock_mhz_for_peak"] * 1e6
    p_alu = peaks["lop3_per_clk_per_sm"] * sms * clk_hz
    p_smem = peaks["lds_bytes_per_clk_per_sm"] * sms * clk_hz
    work = float(m) * l * n
    t = k_ms * 1e-3
    kinfo = [ctypes.c_int() for _ in range(8)]
    _lib.load().sg_kernel_info(plan["kernel"], device.index or 0, *(ctypes.byref(x) for x in kinfo))
    _, _, rt, thr, sched = (x.value for x in kinfo[:5])
    key = f"{field}/{rt}/{sched}/{thr}"
    mix = SASS_MIX.get(key)
    nblocks, slabs = -(-l // 8), -(-n // 128)
    smem_bytes = work * SMEM_PER_MULADD[field]
    own_bytes = work * KERNEL_SMEM_PER_MULADD[field]
    r = {"smem": {"achieved": smem_bytes / t / 1e12, "peak": p_smem / 1e12, "unit": "TB/s",
                  "frac": smem_bytes / t / p_smem, "algorithmic_bytes_per_launch": smem_bytes,
                  "kernel_lookup_bytes_per_launch": own_bytes, "kernel_lookup_frac": own_bytes / t / p_smem}}
    if mix:
        units = float(m) * nblocks * slabs
        alu = units * mix["alu_per_row_block"]
        lop3 = units * mix["lop3_per_row_block"]
        r["alu"] = {"achieved": alu / t / 1e12, "peak": p_alu / 1e12, "unit": "T ALU-ops/s", "frac": alu / t / p_alu,
                    "ops_per_launch": alu, "lop3_only_frac": lop3 / t / p_alu,
                    "per_row_block": {k: round(v, 3) for k, v in mix["per_row_block"].items()},
                    "sass_kernel": key, "sass_loop": mix["loop"],
                    "includes_table_build": mix.get("includes_table_build", False)}
    bind = "alu" if "alu" in r and r["alu"]["frac"] >= r["smem"]["frac"] else "smem"
    b = r[bind]
    out = {"bound": "alu (integer pipe, SASS-counted lookup-loop instructions)" if bind == "alu"
           else "smem (algorithmic table-lookup bytes, LDS bandwidth)",
           "achieved": b["achieved"], "peak": b["peak"], "unit": b["unit"], "frac": b["frac"],
           "pipes": r,
           "definition": ("frac = max over {ALU pipe: lookup-loop integer instructions counted from this kernel's "
                          "SASS per (row, k-block, slab); shared memory: algorithmic lookup bytes}; both <= 1, the "
                          "rest of each pipe's time goes to the table build, index loads and stalls "
                          "(see measured_pipes)"),
           "traffic": TRAFFIC.get(name), "traffic_source": TRAFFIC.get("_source") if name in TRAFFIC else None,
           "measured_pipes": PIPES.get(name), "measured_pipes_source": PIPES.get("_source") if name in PIPES else None,
           "kernel_ms": k_ms, "achieved_muladds_per_s": work / t,
           "peak_source": ("sg_probe_peaks on this GPU: %.1f ALU (LOP3) ops/clk/SM, %.1f LDS B/clk/SM, x %d SMs x "
                           "%.0f MHz (%s)" % (peaks["lop3_per_clk_per_sm"], peaks["lds_bytes_per_clk_per_sm"], sms,
                                              peaks["clock_mhz_for_peak"], peaks["clock_note"]))}
    return out


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

    roof = m4rm_roofline(name, field, m, l, n, k_ms, plan, peaks, device)
    roof["kernel_share_of_step"] = k_ms / ms_per_step if world == 1 else None
    out = {"value": value, "ms_per_step": ms_per_step, "gpu_launches": launches, "clocks": clk.summary(),
           "scaling": "strong" if name in STRONG else "weak", "m_per_gpu": m,
           "roofline": roof, "plan": plan, "transpose_ms": statistics.median(tr), "reduce_ms": statistics.median(red)}

    if e2e:
        out["e2e"] = run_e2e(f, A, B, m, l, n, args, world, device)
    del A, B, C, flush
    torch.cuda.empty_cache()
    return out


def run_next_rows(args, device, n=8192):
    """SURVEY.md 8(f) rows beside the BASELINE configs: the other rings of the same kernel family
    (GF(8) direct, Z8, Z4, F2) at n^3, bench-style steps (L2 flushed, events per step)."""
    import torch
    import paper_0901_1413_b200 as sg
    out = {}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    params = sg.M4rmParams(8)
    steps = max(3, min(args.steps, 5))
    for field in ("gf8", "z8", "z4", "f2"):
        f, A, B = make_inputs(field, n, n, n, 0, device, True)
        C = sg.BitslicedMatrix.zero(f, n, n, device=device)
        for _ in range(3):
            sg.m4rm_multiply(A, B, params, out=C)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for i in range(steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record()
            sg.m4rm_multiply(A, B, params, out=C)
            ev[i][1].record()
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ev) / steps
        p = sg.plan(f, n, n, n, 8)
        out[f"{field} {n}x{n}x{n} k=8"] = {"value": float(n) ** 3 / (ms * 1e-3), "ms_per_step": ms, "steps": steps,
                                          "plan": {k: p[k] for k in ("rows_per_cta", "splits", "ctas", "schedule")}}
        del A, B, C
    del flush
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
    # page-locked operands written by one thread on one CPU (BitslicedMatrix.pin_memory: on the
    # B200 box, a VM, H2D from buffers written by several threads at once ran at 15-25 GB/s)
    Ah = A.pin_memory().planes
    Bh = B.pin_memory().planes
    Ch = sg.BitslicedMatrix.pinned_zero(f, m, n).planes
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
        # what an unmodified reference caller passes: pageable numpy planes (no page-locking), through
        # the public API (m4rm_multiply on host matrices -> sg_m4rm_host), C returned as numpy planes
        import numpy as np
        # (copies: ascontiguousarray of the page-locked tensors' views would still be page-locked)
        An = np.array(Ah.numpy().view(np.uint64), copy=True)
        Bn = np.array(Bh.numpy().view(np.uint64), copy=True)
        Ahm = sg.BitslicedMatrix.from_planes(f, An, l, device="cpu")
        Bhm = sg.BitslicedMatrix.from_planes(f, Bn, n, device="cpu")
        for _ in range(2):
            sg.m4rm_multiply(Ahm, Bhm, sg.M4rmParams(8))
        pts = []
        for _ in range(max(3, min(args.steps, 10))):
            t0 = time.perf_counter()
            Cn = sg.m4rm_multiply(Ahm, Bhm, sg.M4rmParams(8)).planes_numpy()
            pts.append(time.perf_counter() - t0)
        extra["pageable"] = {"value": float(m) * l * n / statistics.mean(pts), "unit": UNIT,
                             "ms_per_step": 1e3 * statistics.mean(pts), "step_ms_min": 1e3 * min(pts),
                             "verified_vs_device_path": bool(np.array_equal(Cn, Ch.numpy().view(np.uint64))),
                             "step_ms_median": 1e3 * statistics.median(pts),
                             "operands_page_locked": bool(Ahm.planes.is_pinned() or Bhm.planes.is_pinned()),
                             "path": "m4rm_multiply(BitslicedMatrix over pageable numpy planes) -> sg_m4rm_host"}
    if world == 1:
        # the same product through the public Python call on the page-locked operands (C allocated
        # page-locked by m4rm_multiply, returned as a BitslicedMatrix)
        Apm, Bpm = sg.BitslicedMatrix(f, m, l, Ah), sg.BitslicedMatrix(f, l, n, Bh)
        # (warm-up results kept alive together: the page-locked allocator then has the two blocks
        # the timed loop alternates between; a fresh cudaHostAlloc costs tens of milliseconds)
        keep = [sg.m4rm_multiply(Apm, Bpm, sg.M4rmParams(8)) for _ in range(3)]
        del keep
        qts = []
        for _ in range(max(3, min(args.steps, 10))):
            t0 = time.perf_counter()
            Cp = sg.m4rm_multiply(Apm, Bpm, sg.M4rmParams(8))
            qts.append(time.perf_counter() - t0)
        extra["public_api_page_locked"] = {"ms_per_step": 1e3 * statistics.mean(qts), "step_ms_median": 1e3 * statistics.median(qts),
                                           "step_ms_min": 1e3 * min(qts),
                                           "verified_vs_device_path": bool(torch.equal(Cp.planes, Ch)),
                                           "path": "m4rm_multiply(page-locked BitslicedMatrix operands) -> sg_m4rm_host"}
    extra["host_buffers"] = ("page-locked, allocated and written by one thread on one CPU "
                             "(BitslicedMatrix.pin_memory / pinned_zero)")
    return {"value": world * float(m) * l * n / per, "unit": UNIT, "ms_per_step": per * 1e3,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(Ch.numel() * 8), **extra,
            "path": ("sg_m4rm_host (C ABI; pinned host planes; A and C in row pieces, the first piece's product "
                     "consuming B's k-chunks as they land, D2H of each piece behind its product)"
                     if world == 1 else "rank-0 H2D of B + broadcast in row blocks overlapped with the chunk products "
                     "(dist.sharded_multiply), per-rank H2D of A rows, D2H of C rows (wall clock, max over ranks)")}


# ----------------------------------------------------------------------------- CPU (oracle port)
def _cpu_inputs(field, rows, l, n):
    import numpy as np

    import oracle
    rng = np.random.default_rng(0)
    A = rng.integers(0, ORDER[field], size=(rows, l), dtype=np.uint8)
    B = rng.integers(0, ORDER[field], size=(l, n), dtype=np.uint8)
    return oracle.pack(field, A), oracle.pack(field, B)


def _cpu_run(field, Ap, Bp, l, n, threads):
    import oracle
    t0 = time.perf_counter()
    oracle.m4rm(field, Ap, Bp, l, n, 8, threads=threads, canonical=False)
    return time.perf_counter() - t0


def cpu_baseline(field, m, l, n, threads, budget_s=20.0, reps=5):
    """The reference CPU path (oracle/sg_oracle.c: the reference's block drivers, Gray table build and
    block loop restated in C, rows sharded over `threads` pthreads -- the reference's row-partition
    contract) timed on this host.

    A two-point row sample (1 and S rows per thread, every k-block table built by every thread)
    predicts the full product.  When `reps` full products fit in `budget_s` they are timed directly
    (median); otherwise the prediction is reported, labelled as an extrapolation."""
    s1, s2 = 4, max(5, min(64, -(-m // threads)))
    Ap, Bp = _cpu_inputs(field, threads * s2, l, n)
    t1 = min(_cpu_run(field, Ap[:, :threads * s1], Bp, l, n, threads) for _ in range(2))
    t2 = min(_cpu_run(field, Ap, Bp, l, n, threads) for _ in range(2))
    b = max((t2 - t1) / (s2 - s1), 1e-9)  # seconds per row per thread
    a = max(t1 - s1 * b, 0.0)              # every thread builds every k-block table
    est = a + b * -(-m // threads)
    if est * min(reps, 3) <= budget_s:
        Ap, Bp = _cpu_inputs(field, m, l, n)
        ts = [_cpu_run(field, Ap, Bp, l, n, threads)]
        while len(ts) < reps and sum(ts) + ts[0] <= budget_s:
            ts.append(_cpu_run(field, Ap, Bp, l, n, threads))
        sec = statistics.median(ts)
        how = (f"full {m}x{l}x{n} product, median of {len(ts)} runs ({', '.join('%.3f' % x for x in ts)} s)")
        kind_note = "timed"
    else:
        sec = est
        how = (f"extrapolated: every k-block table ({-(-l // 8)} blocks of the {l}x{n} B) plus {s1} and {s2} A rows "
               f"per thread timed ({t1:.3f} s, {t2:.3f} s), per-row cost scaled linearly to {m} rows "
               f"(a full run would take ~{est:.0f} s)")
        kind_note = "extrapolated"
    return {"value": float(m) * l * n / sec, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"oracle/sg_oracle.c M4RM k=8 (the restated reference path) on {threads} host threads: {how}",
            "seconds": sec, "method": kind_note}


def run_reference(args, world, rank):
    """The reference arm: the reference's CPU path (its C restatement, all host threads) on the GPU
    arm's config, metric and unit; each timed step is one full product (or, where a full product
    would take minutes, the labelled extrapolation from a row sample)."""
    if rank != 0:
        return 0
    name, field, m, l, n = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    probe = cpu_baseline(field, m, l, n, threads, budget_s=0.0)  # prediction only
    full = probe["seconds"] * (args.steps + args.warmup) <= 240.0
    if full:
        Ap, Bp = _cpu_inputs(field, m, l, n)
        for _ in range(args.warmup):
            _cpu_run(field, Ap, Bp, l, n, threads)
        ts = [_cpu_run(field, Ap, Bp, l, n, threads) for _ in range(args.steps)]
        sec = statistics.median(ts)
        sample = (f"full {m}x{l}x{n} product per step, median of {args.steps} steps after {args.warmup} warm-up "
                  f"(oracle/sg_oracle.c, the restated reference path, {threads} host threads)")
    else:
        sec = probe["seconds"]
        sample = probe["sample"]
    value = float(m) * l * n / sec
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64 (bitsliced boolean words)", "data": "synthetic",
            "config": config_dict(CONFIGS[args.config]),
            "parallelism": f"{threads} host threads, rows sharded (SPEC.md:360)",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_dict(cfg):
    """The workload as both arms name it (identical dicts: the driver compares them)."""
    name, field, m, l, n = cfg
    return {"workload": name, "field": field, "m": m, "l": l, "n": n, "k": 8,
            "inputs": "seeded i.i.d. uniform residues (synthetic)",
            "l2": "GPU arm: L2 flushed (256 MiB write) before every timed step"}


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
    if os.environ.get("SG_BENCH_E2E_FIRST"):  # experiments: the host path before everything else
        res["e2e"] = e2e_for(head, args, world, rank, device)
    per_config = {}
    if not args.no_per_config:
        for i, cfg in enumerate(CONFIGS):
            if i == args.config:
                continue
            r = run_config(cfg, args, world, rank, device, peaks, e2e=False)
            per_config[cfg[0]] = {"value": r["value"], "ms_per_step": r["ms_per_step"],
                                  "roofline_frac": r["roofline"]["frac"], "bound": r["roofline"]["bound"],
                                  "pipes": {k: v["frac"] for k, v in r["roofline"]["pipes"].items()},
                                  "scaling": r["scaling"], "m_per_gpu": r["m_per_gpu"],
                                  "kernel_ms": r["roofline"]["kernel_ms"],
                                  "achieved_muladds_per_s": r["roofline"]["achieved_muladds_per_s"],
                                  "plan": r["plan"], "clocks": r["clocks"]}
    pack_unpack = run_pack_unpack(device) if not args.no_per_config else None
    if pack_unpack is not None:  # a three-plane field beside it (its bit gather is heavier per byte)
        p5 = run_pack_unpack(device, field="f5", m=16384, n=16384)
        pack_unpack["f5_16384x16384"] = {k: p5[k] for k in ("pack_ms", "unpack_ms", "pack_gbps", "unpack_gbps",
                                                             "pack_frac", "unpack_frac", "bytes_per_call")}
    next_rows = run_next_rows(args, device) if (world == 1 and not args.no_per_config) else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        name, field, m, l, n = head
        cpu = cpu_baseline(field, m, l, n, threads)
        for i, cfg in enumerate(CONFIGS):
            if cfg[0] in per_config:
                per_config[cfg[0]]["cpu_baseline"] = cpu_baseline(cfg[1], cfg[2], cfg[3], cfg[4], threads)
    # e2e last, on fresh inputs of the headline config: the host<->device copies are the part of
    # this run most exposed to the shared host's PCIe, so they go after everything else
    if "e2e" not in res:
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
                "config": config_dict(head),
                "parallelism": (f"rows of A/C sharded over {world} GPUs, B broadcast from rank 0 by "
                                f"{backend.upper()} inside every step (geometric row blocks overlapped with the "
                                "chunk products)" if world > 1 else "1 GPU"),
                "m_per_gpu": res["m_per_gpu"], "m_total": m * world if res["scaling"] == "weak" else m,
                "e2e": res["e2e"], "gpu_launches": res["gpu_launches"], "clocks": res["clocks"],
                "roofline": res["roofline"], "plan": res["plan"], "cpu_baseline": cpu,
                "step_breakdown_ms": {"index_prepass": res["transpose_ms"], "m4rm": res["roofline"]["kernel_ms"],
                                      "reduce": res["reduce_ms"],
                                      "note": "events around each launch (serialised, sg_set_timing)"},
                "peaks_probe": peaks, "per_config": per_config, "pack_unpack": pack_unpack,
                "next_rows": next_rows}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
