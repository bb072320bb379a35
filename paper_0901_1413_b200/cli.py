"""Command-line front end mirroring the reference's `slicegemm` CLI.

  python -m paper_0901_1413_b200.cli verify [--fields f3,f5,f9] [--max-dim 65] [--trials 20] [--seed 0]
  python -m paper_0901_1413_b200.cli bench  [--fields f3,f5,f7,f4] [--dims 100,500,1000,2500] [--reps 5]
                                            [--format csv|table]
  python -m paper_0901_1413_b200.cli ffops  [--field f3] [--min 64] [--max 192] [--step 1] [--reps 5]

verify: random products against an independent exact check (a float32 GEMM mod p on the GPU,
exact because every dot product stays below 2^24); exit 0 iff all pass.
bench: Table 1 of the paper on the GPU: median of `reps` multiplies of
seeded n x n matrices, CSV `field,n,algorithm,ms,gffops` with gffops = 2 n^3 / t (SPEC.md:595,
609) and `#` metadata lines.  ffops: the same metric over a dimension sweep (Fig. 1, the
"jigsaw" around word boundaries).  The program search subcommand is not part
of this path.  SLICEGEMM_SEED overrides the default seed 0.
"""

from __future__ import annotations

import argparse
import os
import statistics
import sys

import numpy as np
import torch

from . import _lib
from .extension import EXT_FIELDS, ExtMatrix, ext_multiply
from .fields import FIELDS
from .m4rm import M4rmParams, m4rm_multiply
from .matrix import BitslicedMatrix

ALL = {**FIELDS, **EXT_FIELDS}


def _seed(args):
    return int(os.environ.get("SLICEGEMM_SEED", args.seed))


def _random(spec, m, n, seed):
    if spec.name in EXT_FIELDS:
        g = np.random.Generator(np.random.PCG64(seed))
        return ExtMatrix.from_dense(spec, [g.integers(0, spec.base.order, size=(m, n)) for _ in range(spec.degree)])
    return BitslicedMatrix.random(spec, m, n, seed)


def _multiply(spec, A, B, method="karatsuba"):
    return ext_multiply(A, B, method=method) if spec.name in EXT_FIELDS else m4rm_multiply(A, B, M4rmParams(8))


def _exact_dense(spec, A, B):
    """Independent check: float32 GEMMs of the coefficient matrices, reduced mod p and by the
    defining polynomial (plain arithmetic, no bit tricks)."""
    torch.backends.cuda.matmul.allow_tf32 = False
    if spec.name in EXT_FIELDS:
        p, deg = spec.base.order, spec.degree
        a = [torch.from_numpy(x.astype(np.float32)).cuda() for x in A.to_dense()]
        b = [torch.from_numpy(x.astype(np.float32)).cuda() for x in B.to_dense()]
        prod = [0] * (2 * deg - 1)
        for i in range(deg):
            for j in range(deg):
                prod[i + j] = prod[i + j] + torch.remainder(a[i] @ b[j], p)
        for top in range(2 * deg - 2, deg - 1, -1):
            for k in range(deg):
                prod[top - deg + k] = prod[top - deg + k] - spec.modulus[k] * prod[top]
        return [torch.remainder(prod[i], p).to(torch.uint8).cpu().numpy() for i in range(deg)]
    a = torch.from_numpy(A.to_dense().astype(np.float32)).cuda()
    b = torch.from_numpy(B.to_dense().astype(np.float32)).cuda()
    return torch.remainder(a @ b, spec.order).to(torch.uint8).cpu().numpy()


def cmd_verify(args) -> int:
    rng = np.random.default_rng(_seed(args))
    names = args.fields.split(",")
    failures = 0
    runs = 0
    for name in names:
        spec = ALL[name.lower()]
        for t in range(args.trials):
            m, l, n = (int(x) for x in rng.integers(1, args.max_dim + 1, size=3))
            seed = int(rng.integers(0, 1 << 31))
            A, B = _random(spec, m, l, seed), _random(spec, l, n, seed + 1)
            C = _multiply(spec, A, B)
            got = C.to_dense()
            want = _exact_dense(spec, A, B)
            ok = all(np.array_equal(g, w) for g, w in zip(got, want)) if isinstance(got, list) else \
                np.array_equal(got, want)
            runs += 1
            if not ok:
                failures += 1
                print(f"FAIL {name} m={m} l={l} n={n} seed={seed}")
    print(f"verify: {runs} products, {failures} failures")
    return 1 if failures else 0


def _time_ms(spec, n, reps, seed, method="karatsuba"):
    A, B = _random(spec, n, n, seed), _random(spec, n, n, seed + 1)
    _multiply(spec, A, B, method)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _multiply(spec, A, B, method)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def _header(args, extra=""):
    dev = torch.cuda.get_device_properties(0)
    print(f"# device={dev.name} sms={dev.multi_processor_count} W=64 lanes/word (32-bit kernel words) "
          f"reps={args.reps} seed={_seed(args)} median-of-reps {extra}".rstrip())


def cmd_bench(args) -> int:
    dims = [int(x) for x in args.dims.split(",")]
    names = args.fields.split(",")
    rows = []
    for name in names:
        spec = ALL[name.lower()]
        for n in dims:
            # extension fields: ext_multiply's route (--ext-method: the reference's Karatsuba over
            # the base field, or one direct power-basis product where the field has one: F4, F8)
            method = args.ext_method
            if spec.name in EXT_FIELDS and method == "auto":
                method = "direct" if getattr(spec, "direct", None) is not None else "karatsuba"
            ms = _time_ms(spec, n, args.reps, _seed(args), method)
            rows.append((spec.name, n, "m4rm" if spec.name not in EXT_FIELDS else f"ext_multiply({method})", ms,
                         2.0 * n ** 3 / (ms * 1e-3) / 1e9))
    _header(args)
    if args.format == "csv":
        print("field,n,algorithm,ms,gffops")
        for r in rows:
            print(f"{r[0]},{r[1]},{r[2]},{r[3]:.6f},{r[4]:.3f}")
    else:
        print(f"{'field':>6} " + " ".join(f"{n:>12}" for n in dims) + "   (ms)")
        for name in names:
            spec = ALL[name.lower()]
            print(f"{spec.name:>6} " + " ".join(f"{r[3]:12.4f}" for r in rows if r[0] == spec.name))
    return 0


def cmd_ffops(args) -> int:
    spec = ALL[args.field.lower()]
    _header(args, f"field={spec.name}")
    print("field,n,algorithm,ms,gffops")
    for n in range(args.min, args.max + 1, args.step):
        ms = _time_ms(spec, n, args.reps, _seed(args))
        print(f"{spec.name},{n},m4rm,{ms:.6f},{2.0 * n ** 3 / (ms * 1e-3) / 1e9:.3f}")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_0901_1413_b200.cli")
    sub = ap.add_subparsers(dest="cmd", required=True)
    v = sub.add_parser("verify")
    v.add_argument("--fields", default="f2,f3,f5,f7,z4,z8,f4,f8,f9,f25,f27")
    v.add_argument("--max-dim", type=int, default=65)
    v.add_argument("--trials", type=int, default=20)
    v.add_argument("--seed", type=int, default=0)
    b = sub.add_parser("bench")
    b.add_argument("--fields", default="f3,f5,f7,f4")
    b.add_argument("--dims", default="100,500,1000,2500")
    b.add_argument("--reps", type=int, default=5)
    b.add_argument("--format", choices=["csv", "table"], default="csv")
    b.add_argument("--ext-method", choices=["auto", "karatsuba", "direct"], default="karatsuba",
                   help="ext_multiply route for extension fields (default: the reference's Karatsuba)")
    b.add_argument("--seed", type=int, default=0)
    f = sub.add_parser("ffops")
    f.add_argument("--field", default="f3")
    f.add_argument("--min", type=int, default=64)
    f.add_argument("--max", type=int, default=192)
    f.add_argument("--step", type=int, default=1)
    f.add_argument("--reps", type=int, default=5)
    f.add_argument("--seed", type=int, default=0)
    args = ap.parse_args(argv)
    _lib.load()
    if not torch.cuda.is_available():
        print("no CUDA device: the B200 path has no CPU fallback", file=sys.stderr)
        return 2
    return {"verify": cmd_verify, "bench": cmd_bench, "ffops": cmd_ffops}[args.cmd](args)


if __name__ == "__main__":
    sys.exit(main())
