"""Generate the committed golden fixtures from the reference implementation itself.

Runs ONLY in the build container, where /root/reference exists (it never runs on the
GPU box; the fixtures it writes are what travel).  It imports the surviving reference
modules (`_core_py`, `fields`, `oracle`, `kernels`, `programs`) through a stub package
because `import slicegemm` fails on the missing `matrix.py`
(/root/reference/pkg/src/slicegemm/__init__.py:15).  The missing glue (pack, Gray
table build, block loop, Karatsuba for GF(4)) is written here from its SPEC contract,
as test-side code, and drives the reference's own block drivers:

  pack/layout  SPEC.md:216-236 (planes [r][rows][words], column c -> word c>>6 bit c&63,
               padding lanes canonical zero)            -- layout implied by _core_py.py:186-192
  build_table  SPEC.md:313-325 (Gray order, 2^kp - 1 row add/sub, T[0] = 0, indexed by mask)
  m4rm loop    SPEC.md:326-332, 354-357 (blocks ascending; narrow final block)
  block driver _core_py.py:205-222 (f2, f3), 241-281 (f5, f7)
  GF(4)        SPEC.md:393-399 (Karatsuba: 3 F2 products, C0 = P0+P2, C1 = P1+P2)

Outputs (all small, committed):
  kernel_cases.json  every KERNELS entry's exhaustive lane table (kernels.py:466-509, 550-590)
  m4rm_<field>.npz   seeded inputs, the reference path's raw output planes, and
                     oracle_multiply's dense result (oracle.py:74-79)
  gf4.npz            GF(4) inputs/outputs via Karatsuba over the reference F2 driver and
                     oracle_ext_multiply (oracle.py:192-215)
  m4rm_z4/z8.npz     the reference's ring drivers m4rm_block_z4/z8 (_core_py.py:225-238, 284-286)
  ext_<f>.npz        oracle_ext_multiply over F8, F9, F25, F27 (fields.py:216-219) on seeded
                     coefficient matrices: the targets of the GPU extension-field paths
  blocks_<f>.npz     one call of the pure backend's m4rm_block_<f> / classical_<f>, reached
                     through the reference's own backend registry (_core.set_active("pure");
                     _core.active(), _core.py:15-61), on raw inputs: C holding arbitrary legal
                     patterns (F5 5/6/7, F7 7), tables from the Gray build or random raw rows
                     with T[0] != 0, partial row ranges, ragged widths -- the raw output bits
                     the "cuda" backend must reproduce (_core_cuda)

Usage:  python tests/golden/make_golden.py     (from the repo root, in this container)
"""

from __future__ import annotations

import importlib
import json
import os
import sys
import types

import numpy as np

REF = "/root/reference/pkg/src/slicegemm"
OUT = os.path.dirname(os.path.abspath(__file__))


def load_reference():
    pkg = types.ModuleType("slicegemm")
    pkg.__path__ = [REF]
    sys.modules["slicegemm"] = pkg
    mods = {}
    for name in ("fields", "programs", "oracle", "_core_py", "kernels", "_core"):
        mods[name] = importlib.import_module(f"slicegemm.{name}")
    return mods


R = load_reference()
fields, oracle, core, kernels, registry = R["fields"], R["oracle"], R["_core_py"], R["kernels"], R["_core"]
W = 64


# --------------------------------------------------------------------------- glue
def pack(field, dense):
    """Dense residues -> canonical patterns -> plane-major uint64 words."""
    m, n = dense.shape
    words = (n + W - 1) // W
    pat = np.asarray(field.canonical_table, dtype=np.uint64)[dense.astype(np.int64)]
    planes = np.zeros((field.bits, m, words), dtype=np.uint64)
    for d in range(field.bits):
        bits = ((pat >> np.uint64(d)) & np.uint64(1)).astype(np.uint8)
        padded = np.zeros((m, words * W), dtype=np.uint8)
        padded[:, :n] = bits
        b = np.packbits(padded.reshape(m, words, W), axis=2, bitorder="little")
        planes[d] = b.view("<u8").reshape(m, words)
    return planes


def unpack(field, planes, n):
    r, m, words = planes.shape
    pat = np.zeros((m, n), dtype=np.int64)
    for d in range(r):
        b = np.unpackbits(planes[d].view(np.uint8).reshape(m, words * 8), axis=1,
                          bitorder="little")[:, :n]
        pat |= b.astype(np.int64) << d
    dec = np.array([(-1 if e is None else e) for e in field.decode_table], dtype=np.int64)
    out = dec[pat]
    assert (out >= 0).all(), "illegal pattern in planes"
    return out


def tail_mask(n):
    rem = n % W
    return np.uint64((1 << rem) - 1) if rem else np.uint64((1 << 64) - 1)


def row_add(field, T, dst, src, n, sub=False):
    """T[dst] (+|-)= T-row 'src' (a list of plane rows) via the reference kernels."""
    name = field.name
    d = [T[p][dst] for p in range(field.bits)]
    if name == "f2":
        core.f2_add(d[0], src[0])
    elif name == "f3":
        (core.f3_sub if sub else core.f3_add)(d[0], d[1], src[0], src[1])
    elif name == "f5":
        (core.f5_sub if sub else core.f5_add)(d[0], d[1], d[2], src[0], src[1], src[2])
    elif name == "f7":
        if sub:
            core.f7_sub(d[0], d[1], d[2], src[0], src[1], src[2], tail_mask(n))
        else:
            core.f7_add(d[0], d[1], d[2], src[0], src[1], src[2])
    elif name == "z4":
        (core.z4_sub if sub else core.z4_add)(d[0], d[1], src[0], src[1])
    elif name == "z8":
        (core.z8_sub if sub else core.z8_add)(d[0], d[1], d[2], src[0], src[1], src[2])
    else:
        raise ValueError(name)


def build_table(field, Bp, s, k, kp, n):
    """Gray-code table of all 0/1 combinations of B rows s*k .. s*k+kp-1."""
    r, _, words = Bp.shape
    T = [np.zeros((1 << kp, words), dtype=np.uint64) for _ in range(r)]
    prev = 0
    for i in range(1, 1 << kp):
        g = i ^ (i >> 1)
        t = (g ^ prev).bit_length() - 1
        row = s * k + t
        T_g = [T[p][g] for p in range(r)]
        for p in range(r):
            T_g[p][...] = T[p][prev]
        src = [Bp[p][row] for p in range(r)]
        row_add(field, T, g, src, n, sub=not (g >> t) & 1)
        prev = g
    return T


def ref_m4rm(field, Ap, Bp, l, n, k):
    """The reference CPU path: per k-block, build the table, call m4rm_block_<field>."""
    r, m, _ = Ap.shape
    words = Bp.shape[2]
    C = [np.zeros((m, words), dtype=np.uint64) for _ in range(r)]
    A = [np.ascontiguousarray(Ap[p]) for p in range(r)]
    drv = getattr(core, f"m4rm_block_{field.name}")
    for s in range((l + k - 1) // k):
        col0 = s * k
        kp = min(k, l - col0)
        T = build_table(field, Bp, s, k, kp, n)
        drv(*C, *A, col0, kp, *T, 0, m)
    return np.stack(C) if m else np.zeros((r, 0, words), dtype=np.uint64)


def canonicalize(field, planes):
    out = planes.copy()
    if field.name == "f5":
        core.f5_reduce(out[0], out[1], out[2])
    elif field.name == "f7":
        core.f7_reduce(out[0], out[1], out[2])
    return out


def choose_k(l):
    """clamp(floor(log2 l) - 2, 1, 10)."""
    return max(1, min(10, l.bit_length() - 1 - 2)) if l >= 1 else 1


# --------------------------------------------------------------------------- cases
def kernel_cases():
    out = {}
    for name, info in kernels.KERNELS.items():
        if info.field is not None and info.field.name in ("z4", "z8"):
            continue
        cases = [[list(inp), sorted(list(o) for o in acc)] for inp, acc in info.cases]
        # confirm the reference's own fast form against its table before exporting it
        for inp, acc in info.cases:
            got = info.run_fast([int(b) for b in inp], ones=1)
            got = tuple(int(x) & 1 for x in got)
            assert got in acc, (name, inp, got)
        out[name] = {"field": info.field.name if info.field else None,
                     "n_out": info.n_out, "exact_ops": info.exact_ops,
                     "max_ops": info.max_ops, "op_count": info.program.op_count,
                     "cases": cases}
    return out


def m4rm_fixture(field, rng_cases):
    recs = {}
    for idx, (m, l, n, k, sa, sb) in enumerate(rng_cases):
        A = oracle.DenseMatrix.random(field, m, l, sa)
        B = oracle.DenseMatrix.random(field, l, n, sb)
        Cd = oracle.oracle_multiply(A, B).entries
        Ap, Bp = pack(field, A.entries), pack(field, B.entries)
        Craw = ref_m4rm(field, Ap, Bp, l, n, k)
        Ccan = canonicalize(field, Craw)
        assert np.array_equal(unpack(field, Craw, n), Cd), (field.name, m, l, n, k)
        assert np.array_equal(Ccan, pack(field, Cd)), (field.name, m, l, n, k)
        key = f"c{idx}"
        recs[key + "_shape"] = np.array([m, l, n, k, sa, sb], dtype=np.int64)
        recs[key + "_A"] = A.entries.astype(np.uint8)
        recs[key + "_B"] = B.entries.astype(np.uint8)
        recs[key + "_C"] = Cd.astype(np.uint8)
        recs[key + "_Craw"] = Craw
    recs["count"] = np.array(len(rng_cases))
    return recs


def shape_grid(field_seed):
    rng = np.random.default_rng(1234 + field_seed)
    cases = []
    # SPEC.md:649 acceptance #3: random (m, l, n) <= 65, squares {100, 257}, k in 1..8
    for i in range(60):
        m, l, n = (int(x) for x in rng.integers(1, 66, size=3))
        k = int(rng.integers(1, 9))
        cases.append((m, l, n, k, 100 + i, 500 + i))
    for nsq in (100, 257):
        cases.append((nsq, nsq, nsq, 8, 7, 8))
    for k in range(1, 9):                        # k-invariance on one fixed input
        cases.append((40, 70, 130, k, 3, 4))
    cases.append((3, 3, 3, 2, 11, 12))
    cases.append((65, 65, 65, choose_k(65), 21, 22))  # SPEC.md:331 word-boundary case
    cases.append((1, 1, 1, 1, 5, 6))
    cases.append((64, 128, 64, 8, 31, 32))
    cases.append((33, 130, 70, 5, 41, 42))
    cases.append((128, 1024, 200, 8, 51, 52))    # many blocks, ragged n
    return cases


def gf4_fixture():
    F4, F2 = fields.F4, fields.F2
    recs = {}
    cases = [(1, 1, 1, 1, 1, 2), (5, 7, 9, 3, 3, 4), (65, 65, 65, 8, 5, 6),
             (100, 100, 100, 8, 7, 8), (33, 130, 70, 8, 9, 10), (257, 257, 257, 8, 11, 12)]
    for idx, (m, l, n, k, sa, sb) in enumerate(cases):
        # coefficient planes: element = c0 + c1*x, drawn as one residue in [0, 4)
        ga = np.random.Generator(np.random.PCG64(sa)).integers(0, 4, size=(m, l), dtype=np.int64)
        gb = np.random.Generator(np.random.PCG64(sb)).integers(0, 4, size=(l, n), dtype=np.int64)
        Ac = [oracle.DenseMatrix(F2, (ga >> i) & 1) for i in range(2)]
        Bc = [oracle.DenseMatrix(F2, (gb >> i) & 1) for i in range(2)]
        Cc = oracle.oracle_ext_multiply(F4, Ac, Bc)
        Cd = Cc[0].entries | (Cc[1].entries << 1)
        # Karatsuba over the reference F2 block driver
        A0, A1 = pack(F2, Ac[0].entries), pack(F2, Ac[1].entries)
        B0, B1 = pack(F2, Bc[0].entries), pack(F2, Bc[1].entries)
        P0 = ref_m4rm(F2, A0, B0, l, n, k)
        P2 = ref_m4rm(F2, A1, B1, l, n, k)
        P1 = ref_m4rm(F2, A0 ^ A1, B0 ^ B1, l, n, k) ^ P0 ^ P2
        C0, C1 = P0 ^ P2, P1 ^ P2
        Ckar = unpack(F2, C0, n) | (unpack(F2, C1, n) << 1)
        assert np.array_equal(Ckar, Cd), ("gf4", m, l, n)
        key = f"c{idx}"
        recs[key + "_shape"] = np.array([m, l, n, k, sa, sb], dtype=np.int64)
        recs[key + "_A"] = ga.astype(np.uint8)
        recs[key + "_B"] = gb.astype(np.uint8)
        recs[key + "_C"] = Cd.astype(np.uint8)
        recs[key + "_Craw"] = np.concatenate([C0, C1])
    recs["count"] = np.array(len(cases))
    # over F4, [alpha]*[alpha] = [alpha + 1]  (alpha = x -> pattern 2; x+1 -> 3)
    assert oracle.poly_mul_mod(F4, (0, 1), (0, 1)) == (1, 1)
    return recs


def ext_fixture(spec, cases):
    """oracle_ext_multiply over `spec` on seeded coefficient matrices (oracle.py:192-215)."""
    recs = {}
    base = spec.base
    for idx, (m, l, n, sa, sb) in enumerate(cases):
        Ac = [oracle.DenseMatrix.random(base, m, l, sa + 17 * i) for i in range(spec.degree)]
        Bc = [oracle.DenseMatrix.random(base, l, n, sb + 17 * i) for i in range(spec.degree)]
        Cc = oracle.oracle_ext_multiply(spec, Ac, Bc)
        key = f"c{idx}"
        recs[key + "_shape"] = np.array([m, l, n, sa, sb], dtype=np.int64)
        recs[key + "_A"] = np.stack([a.entries for a in Ac]).astype(np.uint8)
        recs[key + "_B"] = np.stack([b.entries for b in Bc]).astype(np.uint8)
        recs[key + "_C"] = np.stack([c.entries for c in Cc]).astype(np.uint8)
    recs["count"] = np.array(len(cases))
    recs["degree"] = np.array(spec.degree)
    recs["modulus"] = np.array(spec.modulus)
    recs["p"] = np.array(base.order)
    # 1x1 products: the whole multiplication table of the field (acceptance #4)
    q = base.order
    elems = list(__import__("itertools").product(range(q), repeat=spec.degree))
    table = np.zeros((len(elems), len(elems), spec.degree), dtype=np.uint8)
    for i, a in enumerate(elems):
        for j, b in enumerate(elems):
            table[i, j] = oracle.poly_mul_mod(spec, a, b)
    recs["elems"] = np.array(elems, dtype=np.uint8)
    recs["mul_table"] = table
    return recs


def pack_patterns(bits, pat):
    """Raw patterns (m, n) -> plane-major uint64 words (no canonicalization)."""
    m, n = pat.shape
    words = (n + W - 1) // W
    planes = np.zeros((bits, m, words), dtype=np.uint64)
    for d in range(bits):
        b = ((pat >> d) & 1).astype(np.uint8)
        padded = np.zeros((m, words * W), dtype=np.uint8)
        padded[:, :n] = b
        planes[d] = np.packbits(padded.reshape(m, words, W), axis=2, bitorder="little").view("<u8").reshape(m, words)
    return planes


def raw_patterns(field, rng, shape):
    """Uniform over the field's legal patterns, redundant encodings included (F5 5..7, F7 7)."""
    legal = np.array(sorted(p for p, e in enumerate(field.decode_table) if e is not None), dtype=np.int64)
    return legal[rng.integers(0, len(legal), size=shape)]


def block_fixture(field, seed):
    """Raw single calls of the pure backend's block and classical drivers via the registry."""
    registry.set_active("pure")
    be = registry.active()
    assert be.NAME == "pure"
    rng = np.random.default_rng(seed)
    recs = {}
    cases = [(9, 40, 70, 3, 8, 0, 9, "gray"), (33, 130, 200, 64, 8, 5, 30, "gray"), (17, 24, 65, 10, 6, 0, 17, "gray"),
             (50, 200, 129, 120, 8, 11, 12, "random"), (6, 10, 1, 2, 5, 0, 6, "random"), (70, 70, 64, 62, 8, 1, 69, "gray"),
             (40, 300, 100, 290, 10, 3, 37, "random"), (12, 16, 16, 8, 8, 0, 12, "gray")]
    for idx, (m, la, n, col0, kp, row0, row1, tkind) in enumerate(cases):
        kp = min(kp, la - col0)
        Cpat = raw_patterns(field, rng, (m, n))
        Adense = rng.integers(0, field.order, size=(m, la))
        Ap = pack(field, Adense)
        Cp = pack_patterns(field.bits, Cpat)
        if tkind == "gray":
            Bd = rng.integers(0, field.order, size=(col0 + kp, n))
            # the table of B rows col0 .. col0+kp-1 (the Gray build over those rows)
            Bblk = pack(field, Bd[col0:col0 + kp])
            T = build_table(field, Bblk, 0, kp, kp, n)
            Tp = np.stack(T)
        else:
            Tp = pack_patterns(field.bits, raw_patterns(field, rng, (1 << kp, n)))
        C = [Cp[d].copy() for d in range(field.bits)]
        A = [np.ascontiguousarray(Ap[d]) for d in range(field.bits)]
        Tl = [np.ascontiguousarray(Tp[d]) for d in range(field.bits)]
        getattr(be, f"m4rm_block_{field.name}")(*C, *A, col0, kp, *Tl, row0, row1)
        key = f"b{idx}"
        recs[key + "_args"] = np.array([m, la, n, col0, kp, row0, row1], dtype=np.int64)
        recs[key + "_C0"], recs[key + "_A"], recs[key + "_T"] = Cp, Ap, Tp
        recs[key + "_C1"] = np.stack(C)
    recs["nblock"] = np.array(len(cases))
    ccases = [(5, 7, 9), (20, 65, 70), (33, 130, 64), (3, 1, 200), (64, 64, 129)]
    for idx, (m, l, n) in enumerate(ccases):
        Cp = pack_patterns(field.bits, raw_patterns(field, rng, (m, n)))
        Ap = pack(field, rng.integers(0, field.order, size=(m, l)))
        Bp = pack_patterns(field.bits, raw_patterns(field, rng, (l, n)))
        C = [Cp[d].copy() for d in range(field.bits)]
        getattr(be, f"classical_{field.name}")(*C, *[np.ascontiguousarray(Ap[d]) for d in range(field.bits)],
                                              *[np.ascontiguousarray(Bp[d]) for d in range(field.bits)])
        key = f"k{idx}"
        recs[key + "_args"] = np.array([m, l, n], dtype=np.int64)
        recs[key + "_C0"], recs[key + "_A"], recs[key + "_B"] = Cp, Ap, Bp
        recs[key + "_C1"] = np.stack(C)
    recs["nclassical"] = np.array(len(ccases))
    return recs


def main_blocks():
    for i, fname in enumerate(("f2", "f3", "f5", "f7", "z4", "z8")):
        recs = block_fixture(fields.FIELDS[fname], 900 + i)
        np.savez_compressed(os.path.join(OUT, f"blocks_{fname}.npz"), **recs)
        print(fname, "block cases", int(recs["nblock"]), "classical cases", int(recs["nclassical"]))


def main():
    main_blocks()
    with open(os.path.join(OUT, "kernel_cases.json"), "w") as f:
        json.dump(kernel_cases(), f, indent=0)
    for i, fname in enumerate(("z4", "z8")):
        field = fields.FIELDS[fname]
        recs = m4rm_fixture(field, shape_grid(10 + i)[:40] + shape_grid(10 + i)[60:70])
        np.savez_compressed(os.path.join(OUT, f"m4rm_{fname}.npz"), **recs)
        print(fname, "cases", int(recs["count"]))
    ext_cases = [(1, 1, 1, 1, 2), (5, 7, 9, 3, 4), (32, 32, 32, 5, 6), (65, 70, 33, 7, 8), (100, 100, 100, 9, 10)]
    for name in ("f8", "f9", "f25", "f27"):
        recs = ext_fixture(fields.EXT_FIELDS[name], ext_cases)
        np.savez_compressed(os.path.join(OUT, f"ext_{name}.npz"), **recs)
        print(name, "ext cases", int(recs["count"]))
    for i, fname in enumerate(("f2", "f3", "f5", "f7")):
        field = fields.FIELDS[fname]
        recs = m4rm_fixture(field, shape_grid(i))
        np.savez_compressed(os.path.join(OUT, f"m4rm_{fname}.npz"), **recs)
        print(fname, "cases", int(recs["count"]))
    np.savez_compressed(os.path.join(OUT, "gf4.npz"), **gf4_fixture())
    print("gf4 done")


if __name__ == "__main__":
    if sys.argv[1:] == ["blocks"]:
        main_blocks()  # only the block / classical driver fixtures
    else:
        main()
