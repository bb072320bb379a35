"""Drop-in API pieces of the reference's exports (slicegemm/__init__.py:13-20) that need no GPU:
DenseMatrix (oracle.py:17-66), FieldSpec's basis data (fields.py:16-75), and the "cuda" backend
module registered in the reference's own backend registry (_core.py:15-61).

The tests that read /root/reference run in the build container only (the reference does not
travel to the GPU box); the GPU halves of these checks are in tests/test_gpu_dropin.py."""

import importlib
import inspect
import os
import sys
import types

import numpy as np
import pytest

import paper_0901_1413_b200 as sg
from tests import _golden

REF = "/root/reference/pkg/src/slicegemm"
needs_ref = pytest.mark.skipif(not os.path.isdir(REF), reason="the reference is only in the build container")


def _reference():
    if "slicegemm" not in sys.modules:
        pkg = types.ModuleType("slicegemm")
        pkg.__path__ = [REF]
        sys.modules["slicegemm"] = pkg
    return {n: importlib.import_module(f"slicegemm.{n}") for n in ("fields", "_core_py", "_core", "oracle")}


@pytest.mark.parametrize("fname", ["f2", "f3", "f5", "f7", "z4", "z8"])
def test_dense_random_is_the_reference_stream(fname):
    """DenseMatrix.random(field, m, n, seed) reproduces the reference's draws (oracle.py:47-50)
    on every fixture case -- the A and B of tests/golden were drawn by the reference itself."""
    f = sg.by_name(fname)
    for c in _golden.cases(fname):
        A = sg.DenseMatrix.random(f, c["m"], c["l"], c["seed_a"])
        B = sg.DenseMatrix.random(f, c["l"], c["n"], c["seed_b"])
        assert np.array_equal(A.entries, c["A"].astype(np.int64))
        assert np.array_equal(np.asarray(B), c["B"])


def test_dense_matrix_api():
    D = sg.DenseMatrix(sg.F5, [[1, 2], [3, 4]])
    assert (D.nrows, D.ncols) == (2, 2) and D.entries.dtype == np.int64
    assert D == D.copy() and D.equals(sg.DenseMatrix(sg.F5, np.array([[1, 2], [3, 4]])))
    assert not D.equals(sg.DenseMatrix(sg.F7, [[1, 2], [3, 4]]))
    assert sg.DenseMatrix.zero(sg.F3, 2, 3).entries.sum() == 0
    assert np.array_equal(sg.DenseMatrix.identity(sg.F7, 3).entries, np.eye(3, dtype=np.int64))
    with pytest.raises(ValueError):
        sg.DenseMatrix(sg.F3, [[3]])
    with pytest.raises(ValueError):
        sg.DenseMatrix(sg.F3, [[-1]])
    with pytest.raises(ValueError):
        sg.DenseMatrix(sg.F3, [1, 2])
    a = sg.DenseMatrix.random(sg.F7, 5, 6, 3)
    assert a == sg.DenseMatrix.random(sg.F7, 5, 6, 3) and a != sg.DenseMatrix.random(sg.F7, 5, 6, 4)


@needs_ref
def test_field_specs_match_reference_fields():
    """Every base ring's tables, basis (alpha and extraction rule), is_field and valid patterns
    equal the reference's FieldSpec (fields.py:16-158)."""
    rf = _reference()["fields"]
    for name in ("f2", "f3", "f5", "f7", "z4", "z8"):
        ours, ref = sg.by_name(name), rf.FIELDS[name]
        assert (ours.order, ours.char, ours.bits) == (ref.order, ref.char, ref.bits)
        assert ours.decode_table == ref.decode_table and ours.canonical_table == ref.canonical_table
        assert ours.is_field == ref.is_field and ours.valid_patterns == ref.valid_patterns
        assert [(b.alpha, b.extract) for b in ours.basis] == [(b.alpha, b.extract) for b in ref.basis]
        for p in range(1 << ours.bits):
            assert ours.basis_coefficients(p) == ref.basis_coefficients(p), (name, p)


@needs_ref
def test_cuda_backend_registers_in_the_reference_registry():
    """The "cuda" module slots into the reference's backend registry (_core._BACKENDS,
    set_active, active, active_name) and exposes every hot-path function of the pure backend
    with the same name and parameter list (_core_py.py:24-366); the out-of-scope names are the
    packed-integer baselines and the program-search engine."""
    from paper_0901_1413_b200 import _core_cuda
    R = _reference()
    core, pure = R["_core"], R["_core_py"]
    core._BACKENDS["cuda"] = _core_cuda
    try:
        core.set_active("cuda")
        assert core.active() is _core_cuda and core.active_name() == "cuda"
        assert "cuda" in core.available()
        public = [n for n, f in vars(pure).items() if inspect.isfunction(f) and not n.startswith("_")
                  and f.__module__ == pure.__name__]
        missing = [n for n in public if not hasattr(_core_cuda, n)]
        assert sorted(missing) == sorted(_core_cuda.OUT_OF_SCOPE), missing
        for n in public:
            if n in _core_cuda.OUT_OF_SCOPE:
                continue
            ref_params = list(inspect.signature(getattr(pure, n)).parameters)
            our_params = list(inspect.signature(getattr(_core_cuda, n)).parameters)
            assert our_params == ref_params, (n, our_params, ref_params)
    finally:
        core.set_active("pure")
        core._BACKENDS.pop("cuda", None)


def test_exports_cover_the_reference_hot_path_names():
    """The names of slicegemm/__init__.py:13-20 on the multiply path are exported here."""
    for name in ("BitslicedMatrix", "DenseMatrix", "ExtMatrix", "M4rmParams", "RowRef", "F2", "F3", "F4", "F5",
                 "F7", "F8", "F9", "F25", "F27", "Z4", "Z8", "FIELDS", "EXT_FIELDS", "backend_name", "build_table",
                 "choose_k", "classical_multiply", "ext_multiply", "m4rm_multiply", "row_accumulate"):
        assert hasattr(sg, name), name


def test_one_cpu_writer_restores_affinity_and_threads():
    """BitslicedMatrix.pin_memory's writer context (CPU side): inside, the calling thread is on
    one CPU and torch's CPU ops are single-threaded; both are restored on exit, also on error."""
    import torch
    from paper_0901_1413_b200.matrix import one_cpu_writer
    if not hasattr(os, "sched_getaffinity"):
        pytest.skip("no sched_getaffinity on this platform")
    mask, threads = os.sched_getaffinity(0), torch.get_num_threads()
    with one_cpu_writer():
        assert len(os.sched_getaffinity(0)) == 1 and os.sched_getaffinity(0) <= mask
        assert torch.get_num_threads() == 1
    assert os.sched_getaffinity(0) == mask and torch.get_num_threads() == threads
    with pytest.raises(RuntimeError):
        with one_cpu_writer():
            raise RuntimeError("boom")
    assert os.sched_getaffinity(0) == mask and torch.get_num_threads() == threads
