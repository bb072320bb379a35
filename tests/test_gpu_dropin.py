"""GPU halves of the drop-in API checks: the "cuda" backend's block and classical drivers
against fixtures made by the pure backend through the reference's registry (raw bits,
tests/golden/blocks_<f>.npz), RowRef / row_accumulate, to_dense returning
a DenseMatrix, BitslicedMatrix.random against the reference draws, the
extension counter, input checks that run inside the kernels, and argument
checks that must fire before any device access."""

import ctypes

import numpy as np
import pytest
import torch

import oracle
import paper_0901_1413_b200 as sg
from paper_0901_1413_b200 import _core_cuda, _lib, extension
from tests import _golden

pytestmark = pytest.mark.gpu

BLOCK_FIELDS = ["f2", "f3", "f5", "f7", "z4", "z8"]


def _fixture(fname):
    return np.load(f"{_golden.GOLDEN}/blocks_{fname}.npz")


@pytest.mark.parametrize("fname", BLOCK_FIELDS)
def test_block_driver_raw_bits_match_pure_backend(fname):
    """_core_cuda.m4rm_block_<f>(C.., A.., col0, kp, T.., row0, row1) in place on numpy planes
    reproduces the pure backend's raw output bits (redundant patterns, T[0] != 0, row ranges)."""
    z = _fixture(fname)
    drv = getattr(_core_cuda, f"m4rm_block_{fname}")
    for i in range(int(z["nblock"])):
        m, la, n, col0, kp, row0, row1 = (int(x) for x in z[f"b{i}_args"])
        C = [p.copy() for p in z[f"b{i}_C0"]]
        drv(*C, *list(z[f"b{i}_A"]), col0, kp, *list(z[f"b{i}_T"]), row0, row1)
        assert np.array_equal(np.stack(C), z[f"b{i}_C1"]), (fname, i)


@pytest.mark.parametrize("fname", BLOCK_FIELDS)
def test_block_driver_on_device_tensors_in_place(fname):
    z = _fixture(fname)
    drv = getattr(_core_cuda, f"m4rm_block_{fname}")
    m, la, n, col0, kp, row0, row1 = (int(x) for x in z["b1_args"])
    C = [torch.from_numpy(p.view(np.int64).copy()).cuda() for p in z["b1_C0"]]
    A = [torch.from_numpy(p.view(np.int64).copy()).cuda() for p in z["b1_A"]]
    T = [torch.from_numpy(p.view(np.int64).copy()).cuda() for p in z["b1_T"]]
    drv(*C, *A, col0, kp, *T, row0, row1)
    got = np.stack([c.cpu().numpy().view(np.uint64) for c in C])
    assert np.array_equal(got, z["b1_C1"])


@pytest.mark.parametrize("fname", BLOCK_FIELDS)
def test_classical_drivers_raw_bits_match_pure_backend(fname):
    z = _fixture(fname)
    drv = getattr(_core_cuda, f"classical_{fname}")
    for i in range(int(z["nclassical"])):
        C = [p.copy() for p in z[f"k{i}_C0"]]
        drv(*C, *list(z[f"k{i}_A"]), *list(z[f"k{i}_B"]))
        assert np.array_equal(np.stack(C), z[f"k{i}_C1"]), (fname, i)


def test_block_driver_rejects_out_of_range_arguments_before_launch():
    z = _fixture("f3")
    C = [p.copy() for p in z["b1_C0"]]
    A, T = list(z["b1_A"]), list(z["b1_T"])
    m = C[0].shape[0]
    with pytest.raises(IndexError):
        _core_cuda.m4rm_block_f3(*C, *A, 0, 8, *T, 0, m + 1)          # rows past C
    with pytest.raises(IndexError):
        _core_cuda.m4rm_block_f3(*C, *A, 64 * A[0].shape[1] - 4, 8, *T, 0, m)  # columns past A
    with pytest.raises(IndexError):
        _core_cuda.m4rm_block_f3(*C, *A, 0, 8, *[t[:100] for t in T], 0, m)     # table too short
    with pytest.raises(ValueError):
        _core_cuda.m4rm_block_f3(*C, *A, 0, 8, *[np.ascontiguousarray(t[:, :1]) for t in T], 0, m)
    assert np.array_equal(np.stack(C), z["b1_C0"])  # nothing was written


@pytest.mark.parametrize("fname", ["f2", "f3", "f5", "f7", "z4", "z8"])
def test_bitsliced_random_equals_packed_reference_draw(fname):
    f = sg.by_name(fname)
    for c in _golden.cases(fname)[::7]:
        M = sg.BitslicedMatrix.random(f, c["m"], c["l"], c["seed_a"])
        assert np.array_equal(M.planes_numpy(), oracle.pack(fname, c["A"])), (fname, c["m"], c["l"])


def test_to_dense_returns_dense_matrix():
    for fname in ("f3", "f5", "f7", "gf4"):
        f = sg.by_name(fname)
        D = sg.DenseMatrix.random(f, 37, 130, 5)
        M = sg.BitslicedMatrix.from_dense(f, D)  # a DenseMatrix goes in ...
        out = M.to_dense()                       # ... and one comes out
        assert isinstance(out, sg.DenseMatrix) and out.field is f
        assert out == D and out.entries.dtype == np.int64 and (out.nrows, out.ncols) == (37, 130)
        assert np.array_equal(np.asarray(out), np.asarray(D))
    E = sg.BitslicedMatrix.zero(sg.F7, 0, 5).to_dense()
    assert (E.nrows, E.ncols) == (0, 5)


def test_row_accumulate_spec_examples_and_random_rows():
    # F3 dst=[1,-1,0] + src=[1,1,1] -> [-1,0,1]; src zero -> unchanged; F5 4+4 = 3
    M = sg.BitslicedMatrix.from_dense(sg.F3, np.array([[1, 2, 0], [1, 1, 1], [0, 0, 0]], dtype=np.uint8))
    sg.row_accumulate(M.row(0), M.row(1), "add")
    assert np.asarray(M.to_dense())[0].tolist() == [2, 0, 1]
    before = np.asarray(M.to_dense()).copy()
    sg.row_accumulate(M.row(0), M.row(2))
    assert np.array_equal(np.asarray(M.to_dense()), before)
    F = sg.BitslicedMatrix.from_dense(sg.F5, np.array([[4], [4]], dtype=np.uint8))
    sg.row_accumulate(F.row(0), F.row(1))
    assert F.get(0, 0) == 3
    rng = np.random.default_rng(3)
    for fname in ("f2", "f3", "f5", "f7", "z4", "z8", "gf4", "gf8"):
        f = sg.by_name(fname)
        q = f.order
        d = rng.integers(0, q, size=(4, 130)).astype(np.uint8)
        for mode in ("add", "sub"):
            for device in ("cuda", "cpu"):
                M = sg.BitslicedMatrix.from_dense(f, d, device=device)
                sg.row_accumulate(M.row(1), M.row(3), mode)
                want = d.copy()
                if fname in ("f2", "gf4", "gf8"):
                    want[1] ^= d[3]
                else:
                    want[1] = (d[1].astype(int) + (1 if mode == "add" else -1) * d[3].astype(int)) % q
                got = np.asarray(M.to_dense())
                assert np.array_equal(got, want), (fname, mode, device)
                # padding lanes stay zero (F7 sub complements and re-masks)
                assert int(M.planes[:, :, -1].cpu().numpy().view(np.uint64).max() >> np.uint64(2)) == 0
    with pytest.raises(ValueError):
        sg.row_accumulate(M.row(0), sg.BitslicedMatrix.zero(sg.F3, 1, 130).row(0))
    with pytest.raises(ValueError):
        sg.row_accumulate(M.row(0), sg.BitslicedMatrix.zero(M.field, 1, 129).row(0))
    with pytest.raises(IndexError):
        M.row(4)


def test_ext_multiply_default_is_the_counted_karatsuba():
    """SPEC.md:650 acceptance #4: the instrumented counter reads 3 (quadratic) and 6 (cubic) per
    product on the default route; "direct" is the opt-in power-basis kernel (counter 0)."""
    for spec, want in ((sg.F4, 3), (sg.F8, 6), (sg.F9, 3), (sg.F27, 6)):
        A = sg.ExtMatrix.from_dense(spec, [np.ones((3, 4), dtype=np.uint8)] * spec.degree)
        B = sg.ExtMatrix.from_dense(spec, [np.ones((4, 2), dtype=np.uint8)] * spec.degree)
        sg.ext_multiply(A, B)
        assert extension.base_multiplies == want, spec
    sg.ext_multiply(A, B, method="auto")


def test_pack_range_check_is_stream_ordered():
    """sg_pack does not synchronize; a bad entry is reported by sg_stream_check (SG_ERANGE), and
    from_dense maps it to ValueError (the reference's out-of-range error)."""
    L = _lib.load()
    dense = torch.tensor([[0, 1, 2], [3, 1, 0]], dtype=torch.uint8, device="cuda")  # 3 is not in F3
    planes = torch.empty((2, 2, 1), dtype=torch.int64, device="cuda")
    st = _lib.current_stream_handle()
    vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    assert L.sg_pack(sg.F3.code, vp(dense), 2, 3, 3, vp(planes), st) == _lib.SG_OK
    assert L.sg_stream_check(st) == _lib.SG_ERANGE
    assert L.sg_stream_check(st) == _lib.SG_OK  # cleared
    with pytest.raises(ValueError):
        sg.BitslicedMatrix.from_dense(sg.F3, np.array([[0, 3]], dtype=np.uint8))
    with pytest.raises(ValueError):
        sg.BitslicedMatrix.from_dense(sg.F5, torch.tensor([[7, 1]], dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError):
        sg.BitslicedMatrix.from_dense(sg.F3, np.array([[256]], dtype=np.int64))  # would wrap to 0
    bad = sg.BitslicedMatrix.zero(sg.F3, 1, 3)
    bad.planes[1, 0, 0] = 1  # sign without unit
    with pytest.raises(ValueError):
        bad.to_dense()


def test_host_out_argument_is_checked():
    """m4rm_multiply on host operands validates `out` like the device branch."""
    A = sg.BitslicedMatrix.from_dense(sg.F5, np.ones((4, 6), dtype=np.uint8), device="cpu")
    B = sg.BitslicedMatrix.from_dense(sg.F5, np.ones((6, 5), dtype=np.uint8), device="cpu")
    with pytest.raises(ValueError):
        sg.m4rm_multiply(A, B, out=sg.BitslicedMatrix.zero(sg.F5, 3, 5, device="cpu"))   # too small
    with pytest.raises(ValueError):
        sg.m4rm_multiply(A, B, out=sg.BitslicedMatrix.zero(sg.F7, 4, 5, device="cpu"))   # wrong field
    with pytest.raises(ValueError):
        sg.m4rm_multiply(A, B, out=sg.BitslicedMatrix.zero(sg.F5, 4, 5, device="cuda"))  # not a host buffer
    C = sg.BitslicedMatrix.zero(sg.F5, 4, 5, device="cpu")
    sg.m4rm_multiply(A, B, out=C)
    assert np.array_equal(np.asarray(C.to_dense()), np.full((4, 5), 1, dtype=np.uint8))  # 6 mod 5


def test_tall_product_beyond_grid_y_limit():
    """m > 65535 x 32 rows: the index pre-pass strides over row tiles (grid.y is capped) and the
    planner keeps to launchable grids (F5 3e6 x 64 x 64 used to fail)."""
    m, l, n = 3_000_000, 64, 64
    rng = np.random.default_rng(0)
    A = rng.integers(0, 5, size=(m, l), dtype=np.uint8)
    B = rng.integers(0, 5, size=(l, n), dtype=np.uint8)
    C = sg.m4rm_multiply(sg.BitslicedMatrix.from_dense(sg.F5, A), sg.BitslicedMatrix.from_dense(sg.F5, B))
    want = oracle.m4rm("f5", oracle.pack("f5", A), oracle.pack("f5", B), l, n, 8, threads=8)
    assert np.array_equal(C.planes_numpy(), want)
