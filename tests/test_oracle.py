"""CPU tests: the oracle (test infrastructure) pinned against the reference's own outputs.

tests/golden/* were produced by make_golden.py from the reference modules themselves
(_core_py block drivers + SPEC glue, oracle.oracle_multiply, oracle_ext_multiply,
kernels.KERNELS exhaustive tables)."""

import numpy as np
import pytest

import oracle
from tests import _golden

FIELDS = ("f2", "f3", "f5", "f7")


@pytest.mark.parametrize("field", FIELDS + ("gf4", "z4", "z8"))
def test_dense_oracle_matches_reference_oracle(field):
    for c in _golden.cases(field):
        got = oracle.dense_multiply(field, c["A"], c["B"])
        assert np.array_equal(got, c["C"]), (field, c["m"], c["l"], c["n"])


@pytest.mark.parametrize("field", FIELDS + ("gf4", "z4", "z8"))
def test_bitsliced_oracle_matches_reference_path(field):
    for c in _golden.cases(field):
        Ap, Bp = oracle.pack(field, c["A"]), oracle.pack(field, c["B"])
        raw = oracle.m4rm(field, Ap, Bp, c["l"], c["n"], c["k"], threads=2, canonical=False)
        # decode-equal to the reference oracle
        assert np.array_equal(oracle.unpack(field, raw, c["n"]), c["C"])
        # canonical planes equal the canonicalized reference raw planes
        assert np.array_equal(oracle.canonicalize(field, raw), oracle.canonicalize(field, c["Craw"]))
        if field in ("f2", "f3", "gf4", "z4", "z8"):  # unique encodings: raw bits are pinned
            assert np.array_equal(raw, c["Craw"])


@pytest.mark.parametrize("name", ["f8", "f9", "f25", "f27"])
def test_ext_fixture_self_consistency(name):
    """The GF(8) closed form of the oracle equals oracle_ext_multiply(F8); the other fixtures are
    consistent with their own multiplication tables (checked on 1x1 entries)."""
    import os
    z = np.load(os.path.join(_golden.GOLDEN, f"ext_{name}.npz"))
    if name == "f8":
        for i in range(int(z["count"])):
            A = sum(z[f"c{i}_A"][d] << d for d in range(3)).astype(np.uint8)
            B = sum(z[f"c{i}_B"][d] << d for d in range(3)).astype(np.uint8)
            C = sum(z[f"c{i}_C"][d] << d for d in range(3)).astype(np.uint8)
            assert np.array_equal(oracle.dense_multiply("gf8", A, B), C)
    t = z["mul_table"]
    assert t.shape[0] == t.shape[1] == int(z["p"]) ** int(z["degree"])


def test_pack_layout_matches_reference_layout():
    # the reference path's raw planes are packed with column c -> word c>>6, bit c&63
    for c in _golden.cases("f3")[:10]:
        C = oracle.pack("f3", c["C"])
        assert np.array_equal(C, c["Craw"])


def test_kernel_formulas_exhaustive():
    """Every plane kernel of the oracle against kernels.KERNELS' exhaustive lane tables."""
    table = _golden.kernel_cases()
    names = [n for n in table if n not in ("z4_add", "f5_fold5_wide")]
    assert {"f3_add", "f3_sub", "f3_neg", "f5_add", "f5_fold5", "f5_double", "f5_neg", "f5_reduce",
            "f7_add", "f7_double", "f7_neg", "f7_reduce"} <= set(names)
    for name in names:
        info = table[name]
        for inp, acceptable in info["cases"]:
            words = [(np.uint64((1 << 64) - 1) if b else np.uint64(0)) for b in inp]
            out = oracle.word_op(name, words)
            bits = [int(int(o) & 1) for o in out[: info["n_out"]]]
            assert bits in acceptable, (name, inp, bits)


def test_op_count_ledger():
    """The reference's op-count budgets as recorded in the fixture."""
    t = _golden.kernel_cases()
    exact = {"f3_add": 6, "f3_sub": 6, "f3_neg": 1, "f7_add": 17, "f7_double": 0, "f7_neg": 3,
             "f7_reduce": 5, "f5_fold5": 8, "f5_add": 20}
    for k, v in exact.items():
        assert t[k]["op_count"] == v
    for k, v in {"f5_double": 5, "f5_neg": 6, "f5_reduce": 8}.items():
        assert t[k]["op_count"] <= v


def test_random_dense_chunking_is_one_stream():
    full = np.random.Generator(np.random.PCG64(3)).integers(0, 7, size=(37, 29), dtype=np.int64)
    for chunk in (1, 5, 37):
        assert np.array_equal(oracle.random_dense("f7", 37, 29, 3, chunk_rows=chunk), full.astype(np.uint8))


def test_spec_known_answers():
    # SPEC.md:330  [[1,2],[0,1]] . [[1,1],[1,0]] = [[0,1],[1,0]] over F3
    A = np.array([[1, 2], [0, 1]], np.uint8)
    B = np.array([[1, 1], [1, 0]], np.uint8)
    want = np.array([[0, 1], [1, 0]], np.uint8)
    assert np.array_equal(oracle.dense_multiply("f3", A, B), want)
    C = oracle.m4rm("f3", oracle.pack("f3", A), oracle.pack("f3", B), 2, 2, 8)
    assert np.array_equal(oracle.unpack("f3", C, 2), want)
    # SPEC.md:336-339 / 487: 1x1 [6].[6] = [1] over F7, [2].[3] = [6]
    for a, b, r in ((6, 6, 1), (2, 3, 6)):
        C = oracle.m4rm("f7", oracle.pack("f7", np.array([[a]], np.uint8)), oracle.pack("f7", np.array([[b]], np.uint8)), 1, 1, 1)
        assert oracle.unpack("f7", C, 1)[0, 0] == r
    # over F4, alpha * alpha = alpha + 1  (alpha = x = 2, x + 1 = 3)
    assert oracle.dense_multiply("gf4", np.array([[2]], np.uint8), np.array([[2]], np.uint8))[0, 0] == 3
    C = oracle.m4rm("gf4", oracle.pack("gf4", np.array([[2]], np.uint8)), oracle.pack("gf4", np.array([[2]], np.uint8)), 1, 1, 1)
    assert oracle.unpack("gf4", C, 1)[0, 0] == 3
    # identity: I . B = B
    B = oracle.random_dense("f5", 65, 65, 9)
    I = np.eye(65, dtype=np.uint8)
    C = oracle.m4rm("f5", oracle.pack("f5", I), oracle.pack("f5", B), 65, 65, 8)
    assert np.array_equal(oracle.unpack("f5", C, 65), B)


def test_thread_count_invariance():
    A = oracle.random_dense("f7", 50, 90, 1)
    B = oracle.random_dense("f7", 90, 70, 2)
    Ap, Bp = oracle.pack("f7", A), oracle.pack("f7", B)
    r1 = oracle.m4rm("f7", Ap, Bp, 90, 70, 8, threads=1, canonical=False)
    r4 = oracle.m4rm("f7", Ap, Bp, 90, 70, 8, threads=4, canonical=False)
    assert np.array_equal(r1, r4)


def test_checker_is_live():
    """Fault injection: one flipped bit must be caught by the comparison."""
    c = _golden.cases("f3")[0]
    C = oracle.pack("f3", c["C"])
    bad = C.copy()
    bad[0, 0, 0] ^= np.uint64(1)
    assert not np.array_equal(bad, C)
