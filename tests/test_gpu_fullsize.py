"""Full BASELINE-size checks (BASELINE.json configs 0-4, one GPU).

Checks, all bit-exact:
  * the CPU oracle (oracle/sg_oracle.c, the restated reference path, on every host core):
    C's planes equal the oracle's canonical planes (the north star's "bit-exact C versus the CPU
    oracle for every config"; oracle.py:74-79 semantics);
  * the planes are canonical, checked on the device for every size (F3: no sign-without-unit
    lane; F5: every lane < 5; F7: no lane holding 7; padding lanes zero);
  * a second, independent route: C equals (A_f32 @ B_f32) mod p computed by cuBLAS fp32 with TF32 disabled -- exact,
    since every partial sum is an integer below l*(p-1)^2 <= 294,912 < 2^24;
  * size-independent: Freivalds' identity C x = A (B x) mod p for random x, computed on the host
    in int64 from the unpacked matrices.
Inputs are the DenseMatrix.random streams: A = seed 0, B = seed 1."""

import os

import numpy as np
import pytest
import torch

import oracle
import paper_0901_1413_b200 as sg

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CONFIGS = [("f3", 1024, 1024, 1024), ("f5", 4096, 4096, 4096), ("gf4", 8192, 8192, 8192),
           ("f7", 16384, 8192, 16384), ("f3", 32768, 32768, 32768)]
FIELDS = {"f3": sg.F3, "f5": sg.F5, "f7": sg.F7, "gf4": sg.GF4}


def exact_gpu_product(fname, A, B):
    """(A @ B) over the field with an exact fp32 GEMM, returned as dense uint8 (host)."""
    torch.backends.cuda.matmul.allow_tf32 = False
    m, n = A.shape[0], B.shape[1]
    out = np.empty((m, n), dtype=np.uint8)
    Bt = torch.from_numpy(B).cuda()
    if fname == "gf4":
        b0, b1 = (Bt & 1).float(), (Bt >> 1).float()
    else:
        bf = Bt.float()
    step = 4096
    for r0 in range(0, m, step):
        a = torch.from_numpy(A[r0:r0 + step]).cuda()
        if fname == "gf4":
            a0, a1 = (a & 1).float(), (a >> 1).float()
            p11 = a1 @ b1
            c0 = torch.remainder(a0 @ b0 + p11, 2)
            c1 = torch.remainder(a0 @ b1 + a1 @ b0 + p11, 2)
            c = c0.to(torch.uint8) | (c1.to(torch.uint8) << 1)
        else:
            c = torch.remainder(a.float() @ bf, oracle.ORDER[fname]).to(torch.uint8)
        out[r0:r0 + step] = c.cpu().numpy()
    return out


def _matvec(M, x, p, step=2048):
    """(M @ x) mod p in int64, row-chunked (no full-size int64 temporaries)."""
    out = np.empty(M.shape[0], dtype=np.int64)
    for r0 in range(0, M.shape[0], step):
        out[r0:r0 + step] = (M[r0:r0 + step].astype(np.int64) @ x) % p
    return out


def freivalds(fname, A, B, C, trials=6):
    rng = np.random.default_rng(0)
    if fname == "gf4":  # both coefficient planes of the closed form, over F2
        a0, a1 = A & 1, A >> 1
        b0, b1 = B & 1, B >> 1
        c0, c1 = C & 1, C >> 1
        for _ in range(trials):
            x = rng.integers(0, 2, size=B.shape[1], dtype=np.int64)
            bx0, bx1 = _matvec(b0, x, 2), _matvec(b1, x, 2)
            assert np.array_equal(_matvec(c0, x, 2), (_matvec(a0, bx0, 2) + _matvec(a1, bx1, 2)) % 2)
            assert np.array_equal(_matvec(c1, x, 2),
                                  (_matvec(a0, bx1, 2) + _matvec(a1, bx0, 2) + _matvec(a1, bx1, 2)) % 2)
        return
    p = oracle.ORDER[fname]
    for _ in range(trials):
        x = rng.integers(0, p, size=B.shape[1], dtype=np.int64)
        assert np.array_equal(_matvec(C, x, p), _matvec(A, _matvec(B, x, p), p))


def assert_canonical_on_device(fname, C):
    """Every lane of C holds its field's canonical pattern, padding lanes zero."""
    P = C.planes  # (R, m, W) int64 on the device
    if fname == "f3":
        bad = P[1] & ~P[0]                 # sign without unit: the illegal pattern 10
    elif fname == "f5":
        bad = P[2] & (P[1] | P[0])         # 5, 6, 7 are redundant encodings of 0, 1, 2
    elif fname == "f7":
        bad = P[2] & P[1] & P[0]           # 7 is the redundant encoding of 0
    else:
        bad = torch.zeros_like(P[0])       # GF(4): every pattern is canonical
    assert int(torch.count_nonzero(bad)) == 0, f"{fname}: non-canonical lanes in C"
    rem = C.ncols % 64
    if rem:
        tail = P[:, :, -1]
        pad = torch.tensor(~((1 << rem) - 1) & ((1 << 63) - 1), dtype=torch.int64, device=P.device)
        pad = pad | torch.tensor(-(1 << 63), dtype=torch.int64, device=P.device)  # bit 63
        assert int(torch.count_nonzero(tail & pad)) == 0, f"{fname}: padding lanes set"


@pytest.mark.parametrize("fname,m,l,n", CONFIGS)
def test_baseline_config_exact(fname, m, l, n):
    A = oracle.random_dense(fname, m, l, 0)
    B = oracle.random_dense(fname, l, n, 1)
    f = FIELDS[fname]
    C = sg.m4rm_multiply(sg.BitslicedMatrix.from_dense(f, A), sg.BitslicedMatrix.from_dense(f, B), sg.M4rmParams(8))
    assert_canonical_on_device(fname, C)
    got = C.planes_numpy()
    # 1. the CPU oracle (restated reference path), every host thread
    want = oracle.m4rm(fname, oracle.pack(fname, A), oracle.pack(fname, B), l, n, 8, threads=os.cpu_count() or 1)
    assert np.array_equal(got, want), f"{fname} {m}x{l}x{n}: C differs from the CPU oracle"
    del want
    # 2. an independent exact route (fp32 GEMM) and Freivalds' identity on the dense result
    Cd = np.asarray(C.to_dense())
    freivalds(fname, A, B, Cd)
    assert np.array_equal(Cd, exact_gpu_product(fname, A, B))
