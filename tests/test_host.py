"""CPU tests of the host-side mirror of the reference API (no GPU needed)."""

import numpy as np
import pytest
import torch

import paper_0901_1413_b200 as sg
from paper_0901_1413_b200 import dist as sgdist


def test_field_tables_match_reference_encodings():
    # fields.py:88-101: F3 0 -> 00, 1 -> 01, -1 -> 11; pattern 10 illegal
    assert sg.F3.canonical_table == (0, 1, 3)
    with pytest.raises(ValueError):
        sg.F3.decode(2)
    assert [sg.F5.decode(p) for p in range(8)] == [0, 1, 2, 3, 4, 0, 1, 2]
    assert [sg.F7.decode(p) for p in range(8)] == [0, 1, 2, 3, 4, 5, 6, 0]
    assert sg.GF4.order == 4 and sg.GF4.bits == 2 and sg.GF8.bits == 3
    assert sg.by_name("GF4") is sg.GF4 and sg.by_name("f3") is sg.F3 and sg.by_name("z8") is sg.Z8
    # extension-field objects match fields.py:215-219
    assert (sg.F4.modulus, sg.F8.modulus, sg.F9.modulus, sg.F25.modulus, sg.F27.modulus) == (
        (1, 1, 1), (1, 1, 0, 1), (1, 0, 1), (3, 0, 1), (1, 2, 0, 1))
    assert [f.order for f in (sg.F4, sg.F8, sg.F9, sg.F25, sg.F27)] == [4, 8, 9, 25, 27]
    with pytest.raises(ValueError):
        sg.ExtFieldSpec("bad", sg.F3, 2, (2, 0, 1))  # x^2 + 2 = x^2 - 1 has roots
    with pytest.raises(ValueError):
        sg.by_name("f11")


def test_choose_k_spec_examples():
    # SPEC.md:343-345
    assert sg.choose_k(8) == 1
    assert sg.choose_k(1024) == 8
    assert sg.choose_k(1) == 1
    assert sg.choose_k(1 << 20) == 10


def test_params_validation():
    assert sg.M4rmParams(8).k == 8
    with pytest.raises(ValueError):
        sg.M4rmParams(0)
    with pytest.raises(ValueError):
        sg.M4rmParams(17)


def test_matrix_container_validation():
    z = sg.BitslicedMatrix.zero(sg.F5, 1, 70, device="cpu")
    assert z.words_per_row == 2 and z.planes.shape == (3, 1, 2)
    e = sg.BitslicedMatrix.zero(sg.F7, 0, 5, device="cpu")
    assert e.nrows == 0
    with pytest.raises(ValueError):
        sg.BitslicedMatrix(sg.F3, 2, 2, torch.zeros((3, 2, 1), dtype=torch.int64))
    with pytest.raises(ValueError):
        sg.BitslicedMatrix.from_dense(sg.F3, np.array([[0, 3]]))
    with pytest.raises(ValueError):
        sg.BitslicedMatrix.from_dense(sg.F5, np.array([[-1, 2]]))


def test_multiply_argument_checks_before_any_device_work():
    a = sg.BitslicedMatrix.zero(sg.F3, 2, 3, device="cpu")
    b = sg.BitslicedMatrix.zero(sg.F3, 4, 2, device="cpu")
    with pytest.raises(ValueError, match="inner dimensions"):
        sg.m4rm_multiply(a, b)
    c = sg.BitslicedMatrix.zero(sg.F5, 3, 2, device="cpu")
    with pytest.raises(ValueError, match="field mismatch"):
        sg.m4rm_multiply(a, c)


def test_from_planes_roundtrip_layout():
    import oracle
    d = oracle.random_dense("f7", 5, 130, 4)
    planes = oracle.pack("f7", d)
    M = sg.BitslicedMatrix.from_planes(sg.F7, planes, 130, device="cpu")
    assert np.array_equal(M.planes_numpy(), planes)
    assert M.get(2, 129) == d[2, 129] and M.get(4, 0) == d[4, 0]
    M.set(2, 129, 6)
    assert M.get(2, 129) == 6


def test_row_partition():
    for m in (0, 1, 7, 4096, 32768):
        for w in (1, 2, 3, 8):
            parts = sgdist.row_partition(m, w)
            assert parts[0][0] == 0 and parts[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [r1 - r0 for r0, r1 in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        sgdist.row_partition(4, 0)


def test_ext_matrix_validation():
    c = sg.BitslicedMatrix.zero(sg.F2, 3, 4, device="cpu")
    E = sg.ExtMatrix(sg.F4, [c, c.copy()])
    assert (E.nrows, E.ncols) == (3, 4)
    G = E.as_direct()
    assert G.field is sg.GF4 and G.planes.shape == (2, 3, 1)
    with pytest.raises(ValueError):
        sg.ExtMatrix(sg.F4, [c])
    with pytest.raises(ValueError):
        sg.ExtMatrix(sg.F4, [c, sg.BitslicedMatrix.zero(sg.F2, 3, 5, device="cpu")])
