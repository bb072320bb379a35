"""GPU parity tests: the CUDA path (through the C ABI) against the oracle and the reference's
golden outputs.  Bar: bit-exact planes (F5/F7 outputs are canonical, compared against the
canonicalized reference)."""

import os

import numpy as np
import pytest
import torch

import oracle
import paper_0901_1413_b200 as sg
from paper_0901_1413_b200 import _core_cuda, _lib, m4rm as m4rm_mod
from tests import _golden

pytestmark = pytest.mark.gpu

FIELDS = {"f2": sg.F2, "f3": sg.F3, "f5": sg.F5, "f7": sg.F7, "gf4": sg.GF4, "gf8": sg.GF8, "z4": sg.Z4, "z8": sg.Z8}


def gpu_multiply(fname, A, B, k=8):
    f = FIELDS[fname]
    Ag = sg.BitslicedMatrix.from_dense(f, A)
    Bg = sg.BitslicedMatrix.from_dense(f, B)
    return sg.m4rm_multiply(Ag, Bg, sg.M4rmParams(k))


def expect(fname, A, B):
    return oracle.pack(fname, oracle.dense_multiply(fname, A, B))


@pytest.fixture(autouse=True)
def _reset_override():
    m4rm_mod.set_plan_override(0, 0)
    yield
    m4rm_mod.set_plan_override(0, 0)


# ---------------------------------------------------------------- formulas, lane by lane
def test_plane_kernels_exhaustive_on_device():
    """Each device formula against kernels.KERNELS' exhaustive lane tables (kernels.py:466-509)."""
    table = _golden.kernel_cases()
    n_in = {"f3_add": (2, 2), "f3_sub": (2, 2), "f3_neg": (2, 0), "f5_add": (3, 3), "f5_double": (3, 0),
            "f5_neg": (3, 0), "f5_reduce": (3, 0), "f7_add": (3, 3), "f7_double": (3, 0), "f7_neg": (3, 0),
            "f7_reduce": (3, 0), "f5_fold5": (3, 1)}
    for name, (nd, ns) in n_in.items():
        info = table[name]
        cases = info["cases"]
        words = np.zeros(nd + ns, dtype=np.uint64)
        for lane, (inp, _) in enumerate(cases):
            for j, b in enumerate(inp):
                if b:
                    words[j] |= np.uint64(1 << lane)
        dst = [torch.from_numpy(words[j:j + 1].view(np.int64).copy()).cuda() for j in range(nd)]
        src = [torch.from_numpy(words[j:j + 1].view(np.int64).copy()).cuda() for j in range(nd, nd + ns)]
        tail = (1 << len(cases)) - 1 if name in ("f7_neg",) else (1 << 64) - 1
        _core_cuda._op(name, dst, src, tail=tail)
        out = [int(t.cpu().numpy().view(np.uint64)[0]) for t in dst]
        for lane, (inp, acceptable) in enumerate(cases):
            bits = [(out[d] >> lane) & 1 for d in range(info["n_out"])]
            assert bits in acceptable, (name, inp, bits)


# ---------------------------------------------------------------- pack / unpack
@pytest.mark.parametrize("fname", list(FIELDS))
def test_pack_unpack_roundtrip(fname):
    for (m, n) in [(1, 1), (3, 31), (5, 32), (7, 33), (2, 64), (9, 65), (4, 130), (33, 1000), (0, 5), (5, 0)]:
        d = oracle.random_dense(fname, m, n, m * 131 + n)
        M = sg.BitslicedMatrix.from_dense(FIELDS[fname], d)
        assert np.array_equal(M.planes_numpy(), oracle.pack(fname, d)), (fname, m, n)
        assert np.array_equal(M.to_dense(), d)


def test_pack_rejects_out_of_range_on_device():
    d = torch.tensor([[0, 1, 2, 3]], dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        sg.BitslicedMatrix.from_dense(sg.F3, d)


def test_unpack_rejects_illegal_f3_pattern():
    M = sg.BitslicedMatrix.zero(sg.F3, 1, 5)
    M.planes[1, 0, 0] = 1  # sign without unit
    with pytest.raises(ValueError):
        M.to_dense()


# ---------------------------------------------------------------- golden fixtures
@pytest.mark.parametrize("fname", sorted(_golden.FIELD_FILES))
def test_m4rm_matches_reference_golden(fname):
    for c in _golden.cases(fname):
        C = gpu_multiply(fname, c["A"], c["B"], c["k"])
        got = C.planes_numpy()
        assert np.array_equal(got, oracle.canonicalize(fname, c["Craw"])), (fname, c["m"], c["l"], c["n"], c["k"])
        if fname in ("f2", "f3", "gf4", "z4", "z8"):
            assert np.array_equal(got, c["Craw"])
        assert np.array_equal(C.to_dense(), c["C"])


@pytest.mark.parametrize("fname", list(FIELDS))
def test_spec3_random_grid(fname):
    """200 random (m, l, n) <= 65 per field, exact."""
    rng = np.random.default_rng(99)
    for t in range(200):
        m, l, n = (int(x) for x in rng.integers(1, 66, size=3))
        A = oracle.random_dense(fname, m, l, 1000 + t)
        B = oracle.random_dense(fname, l, n, 2000 + t)
        C = gpu_multiply(fname, A, B)
        assert np.array_equal(C.planes_numpy(), expect(fname, A, B)), (fname, m, l, n)


@pytest.mark.parametrize("fname", list(FIELDS))
def test_k_invariance(fname):
    A = oracle.random_dense(fname, 100, 257, 5)
    B = oracle.random_dense(fname, 257, 300, 6)
    want = expect(fname, A, B)
    for k in range(1, 17):
        assert np.array_equal(gpu_multiply(fname, A, B, k).planes_numpy(), want), (fname, k)


@pytest.mark.parametrize("fname", list(FIELDS))
def test_every_compiled_plan(fname):  # noqa: F811
    """Force every rows-per-thread variant, every schedule and several k-splits, with B staged by
    cp.async (n = 777: odd 64-bit word count) and by TMA bulk copies (n = 768), l = 1001 leaving
    a partial last k-block (zero-filled B rows)."""
    ran = 0
    for n in (777, 768):
        A = oracle.random_dense(fname, 700, 1001, 7)
        B = oracle.random_dense(fname, 1001, n, 8)
        want = expect(fname, A, B)
        for rt in (1, 2, 4, 8, 16):
            for pipe in (0, 1, 2, 5):
                for nt in (256, 512):
                    for splits in (1, 2, 5, 16):
                        m4rm_mod.set_plan_override(rt, splits, pipe, nt)
                        try:
                            C = gpu_multiply(fname, A, B)
                        except RuntimeError as e:
                            assert "no compiled" in str(e)
                            continue
                        ran += 1
                        assert np.array_equal(C.planes_numpy(), want), (fname, n, rt, pipe, nt, splits)
    assert ran >= 80


@pytest.mark.parametrize("fname", list(FIELDS))
def test_fused_small_plans(fname):
    """The fused one-launch variants (A's words staged by the kernel, split-K summed inside it at
    per-tile arrival counters): every rows-per-thread variant, both schedules, split counts up to
    the co-resident limit, ragged shapes; repeated calls (the counters must come back to zero)
    and a second stream (its own counters); bit-identical to the oracle."""
    ran = 0
    for (m, l, n) in [(700, 1001, 777), (700, 1001, 768), (1024, 1024, 1024), (1, 5, 3), (257, 64, 129),
                      (100, 2000, 40)]:
        A = oracle.random_dense(fname, m, l, m + 5)
        B = oracle.random_dense(fname, l, n, n + 6)
        want = expect(fname, A, B)
        for rt in (1, 2, 4):
            for pipe in (m4rm_mod.FUSED_SERIAL, m4rm_mod.FUSED_PIPELINED):
                for splits in (1, 2, 5, 16, 37):
                    m4rm_mod.set_plan_override(rt, splits, pipe, 256)
                    try:
                        p = m4rm_mod.plan(fname, m, l, n)
                    except RuntimeError as e:
                        assert "no compiled" in str(e)
                        continue
                    assert p["schedule"].startswith("fused")
                    for _ in range(2):
                        C = gpu_multiply(fname, A, B)
                        assert np.array_equal(C.planes_numpy(), want), (fname, m, l, n, rt, pipe, splits)
                    ran += 1
        s2 = torch.cuda.Stream()
        with torch.cuda.stream(s2):
            m4rm_mod.set_plan_override(4, 5, m4rm_mod.FUSED_PIPELINED, 256)
            try:
                C = gpu_multiply(fname, A, B)
                s2.synchronize()
                assert np.array_equal(C.planes_numpy(), want)
            except RuntimeError as e:
                assert "no compiled" in str(e)
    m4rm_mod.set_plan_override()
    assert ran >= 30


@pytest.mark.parametrize("fname", ["f3", "gf4", "f7", "f5", "gf8", "z8", "z4", "f2"])
def test_tmem_accumulator_variant(fname):
    """Schedule 6: a second set of row-slots per lookup thread parked in tensor memory (F3 /
    GF(4) / Z4 / F2 16 + 16 = 8192 rows per table, F7 / GF(8) / Z8 8 + 8 = 4096; F5 8 + 8 with the
    row-slots rotating through three TMEM regions in groups of 4; the three-plane fields and
    GF(4) with just-in-time index staging in two slots); forced split-K and stream-K plans on
    ragged shapes, bit-identical."""
    ran = 0
    for (m, l, n) in [(700, 1001, 777), (8200, 1000, 768), (16384, 512, 512), (3000, 64, 1000), (9000, 40, 2000), (20000, 300, 640)]:
        A = oracle.random_dense(fname, m, l, m + 11)
        B = oracle.random_dense(fname, l, n, n + 12)
        want = expect(fname, A, B)
        # row-slots per thread, both sets (F2 also 32 + 32: 16384 rows per table)
        rts = (16,) if fname in ("f7", "f5", "gf8", "z8") else (32, 64) if fname == "f2" else (32,)
        for splits, rt in [(sp, r) for sp in (1, 2, 5, -1) for r in rts]:
            m4rm_mod.set_plan_override(rt, splits, 6, 256)
            try:
                p = m4rm_mod.plan(fname, m, l, n)
            except RuntimeError as e:
                assert "no compiled" in str(e)
                continue
            assert p["rows_per_cta"] == 256 * rt and p["schedule"].startswith("warp-specialized (4 builder warps, TMEM")
            C = gpu_multiply(fname, A, B)
            assert np.array_equal(C.planes_numpy(), want), (m, l, n, splits, rt)
            ran += 1
    m4rm_mod.set_plan_override()
    assert ran >= 12


@pytest.mark.parametrize("fname", list(FIELDS))
def test_streamk_forced(fname):
    """Stream-K (splits = -1): CTA ranges that start and end mid-tile, span several whole tiles
    (written straight to C) or lie inside one tile, every schedule and CTA shape, ragged m / l / n;
    bit-identical to the oracle."""
    ran = 0
    for (m, l, n) in [(700, 1000, 777), (3000, 64, 1000), (1111, 333, 200), (257, 2500, 129), (9000, 40, 2000),
                      (5000, 200, 768)]:
        A = oracle.random_dense(fname, m, l, m + l)
        B = oracle.random_dense(fname, l, n, n + 3)
        want = expect(fname, A, B)
        for rt in (1, 2, 4, 8, 16):
            for pipe in (0, 1, 2, 5):
                for nt in (256, 512):
                    m4rm_mod.set_plan_override(rt, -1, pipe, nt)
                    try:
                        C = gpu_multiply(fname, A, B)
                    except RuntimeError as e:
                        assert "no compiled" in str(e)
                        continue
                    assert m4rm_mod.plan(fname, m, l, n)["splits"] == -1
                    ran += 1
                    assert np.array_equal(C.planes_numpy(), want), (fname, m, l, n, rt, pipe, nt)
    m4rm_mod.set_plan_override()
    assert ran >= 12


@pytest.mark.parametrize("fname", ["f3", "f5", "gf4", "f2"])
def test_streamk_hybrid_whole_tile_waves(fname):
    """Stream-K with at least one tile per CTA: the leading whole waves go tile by tile (CTA c:
    tiles c, c + G, ...) and only the last partial wave is cut into unit ranges, with the
    reduction kernel offset to the first stream-K tile.  Tile counts just above G, far above it,
    and an exact multiple of G (empty stream-K tail); bit-identical to the oracle."""
    hybrid = 0
    for (m, l, n) in [(2048, 256, 4096), (4500, 96, 5000), (9000, 40, 2000), (1200, 130, 16384)]:
        A = oracle.random_dense(fname, m, l, m + 5)
        B = oracle.random_dense(fname, l, n, n + 6)
        want = expect(fname, A, B)
        for rt, pipe in ((1, 0), (1, 1), (2, 0), (4, 2), (8, 2)):
            m4rm_mod.set_plan_override(rt, -1, pipe, 256)
            try:
                p = m4rm_mod.plan(fname, m, l, n)
            except RuntimeError as e:
                assert "no compiled" in str(e)
                continue
            tiles = -(-m // p["rows_per_cta"]) * -(-n // 128)
            hybrid += tiles >= p["ctas"]
            C = gpu_multiply(fname, A, B)
            assert np.array_equal(C.planes_numpy(), want), (fname, m, l, n, rt, pipe, tiles, p["ctas"])
    # an exact multiple of the CTA count: every tile goes whole, the stream-K tail is empty
    m4rm_mod.set_plan_override(1, -1, 0, 256)
    G = m4rm_mod.plan(fname, 2048, 256, 4096)["ctas"]
    m, l, n = 256 * 2, 72, 128 * G
    A = oracle.random_dense(fname, m, l, 31)
    B = oracle.random_dense(fname, l, n, 32)
    p = m4rm_mod.plan(fname, m, l, n)
    assert p["splits"] == -1 and 2 * (n // 128) == 2 * p["ctas"]
    C = gpu_multiply(fname, A, B)
    assert np.array_equal(C.planes_numpy(), expect(fname, A, B))
    m4rm_mod.set_plan_override()
    assert hybrid >= 4


@pytest.mark.parametrize("fname", list(FIELDS))
def test_general_k_pipelined_straddle(fname):
    """k = 5 (blocks straddle 32-bit words) through the pipelined schedule."""
    A = oracle.random_dense(fname, 300, 333, 17)
    B = oracle.random_dense(fname, 333, 200, 18)
    m4rm_mod.set_plan_override(1, 0, 1, 256)
    C = gpu_multiply(fname, A, B, k=5)
    assert np.array_equal(C.planes_numpy(), expect(fname, A, B))


@pytest.mark.parametrize("fname,m,l,n", [("f3", 1024, 1024, 1024), ("f5", 1000, 3000, 700), ("f7", 513, 2049, 1500),
                                         ("gf4", 1500, 1200, 1300), ("f2", 800, 4000, 900)])
def test_medium_shapes_against_dense_oracle(fname, m, l, n):
    A = oracle.random_dense(fname, m, l, 0)
    B = oracle.random_dense(fname, l, n, 1)
    C = gpu_multiply(fname, A, B)
    assert np.array_equal(C.planes_numpy(), expect(fname, A, B))


def test_f3_1024_config0_against_bitsliced_oracle():
    """BASELINE config 0: F3 1024^3, seeds 0/1, k=8, vs the restated reference path."""
    A = oracle.random_dense("f3", 1024, 1024, 0)
    B = oracle.random_dense("f3", 1024, 1024, 1)
    ref = oracle.m4rm("f3", oracle.pack("f3", A), oracle.pack("f3", B), 1024, 1024, 8, threads=8)
    assert np.array_equal(gpu_multiply("f3", A, B).planes_numpy(), ref)


# ---------------------------------------------------------------- API semantics
def test_spec_known_answers_on_gpu():
    C = gpu_multiply("f3", np.array([[1, 2], [0, 1]]), np.array([[1, 1], [1, 0]]))
    assert np.array_equal(C.to_dense(), [[0, 1], [1, 0]])
    C = gpu_multiply("f7", np.array([[6]]), np.array([[6]]))
    assert C.to_dense()[0, 0] == 1
    C = gpu_multiply("gf4", np.array([[2]]), np.array([[2]]))
    assert C.to_dense()[0, 0] == 3  # alpha * alpha = alpha + 1
    B = oracle.random_dense("f5", 65, 65, 9)
    C = gpu_multiply("f5", np.eye(65, dtype=np.uint8), B)
    assert np.array_equal(C.to_dense(), B)


def test_empty_and_degenerate_shapes():
    for (m, l, n) in [(0, 5, 5), (5, 0, 5), (5, 5, 0), (1, 1, 1)]:
        A = oracle.random_dense("f7", m, l, 1)
        B = oracle.random_dense("f7", l, n, 2)
        C = gpu_multiply("f7", A, B)
        assert (C.nrows, C.ncols) == (m, n)
        assert np.array_equal(C.planes_numpy(), expect("f7", A, B))


def test_host_buffers_e2e_path():
    for fname in FIELDS:
        A = oracle.random_dense(fname, 300, 500, 3)
        B = oracle.random_dense(fname, 500, 200, 4)
        Ah = sg.BitslicedMatrix.from_planes(FIELDS[fname], oracle.pack(fname, A), 500, device="cpu")
        Bh = sg.BitslicedMatrix.from_planes(FIELDS[fname], oracle.pack(fname, B), 200, device="cpu")
        C = sg.m4rm_multiply(Ah, Bh)
        assert C.device.type == "cpu"
        assert np.array_equal(C.planes_numpy(), expect(fname, A, B))


def test_host_small_calls_replay():
    """Small host-buffer products (C < 1 MB) run on one stream, and a call repeated on the same
    page-locked buffers replays a captured CUDA graph (from the third call on): the graph must
    re-read the caller's buffers on every replay (new contents, same addresses) and a changed
    plan override must not reuse a graph captured under another plan."""
    for fname in ("f3", "f5", "gf4", "f7"):
        m, l, n = 300, 520, 200
        f = FIELDS[fname]
        Ap = torch.empty((f.bits, m, (l + 63) // 64), dtype=torch.int64).pin_memory()
        Bp = torch.empty((f.bits, l, (n + 63) // 64), dtype=torch.int64).pin_memory()
        Cp = torch.empty((f.bits, m, (n + 63) // 64), dtype=torch.int64).pin_memory()
        A_, B_, C_ = sg.BitslicedMatrix(f, m, l, Ap), sg.BitslicedMatrix(f, l, n, Bp), sg.BitslicedMatrix(f, m, n, Cp)
        for i in range(5):
            if i == 3:
                m4rm_mod.set_plan_override(2, 4, m4rm_mod.FUSED_PIPELINED, 256)
            A = oracle.random_dense(fname, m, l, 40 + i)
            B = oracle.random_dense(fname, l, n, 50 + i)
            Ap.copy_(torch.from_numpy(oracle.pack(fname, A).view(np.int64)))
            Bp.copy_(torch.from_numpy(oracle.pack(fname, B).view(np.int64)))
            Cp.fill_(-1)
            C = sg.m4rm_multiply(A_, B_, sg.M4rmParams(8), out=C_)
            assert C is C_ and np.array_equal(C.planes_numpy(), expect(fname, A, B)), (fname, i)
        m4rm_mod.set_plan_override()
        # a larger host product on the same device grows the library's buffers (workspace,
        # staging): the graphs captured over the old ones must not be replayed
        big = 6000 + 64 * "f3 f5 gf4 f7".split().index(fname)
        Ab = oracle.random_dense(fname, big, 700, 61)
        Bb = oracle.random_dense(fname, 700, 900, 62)
        Cb = sg.m4rm_multiply(sg.BitslicedMatrix.from_planes(f, oracle.pack(fname, Ab), 700, device="cpu"),
                              sg.BitslicedMatrix.from_planes(f, oracle.pack(fname, Bb), 900, device="cpu"))
        assert np.array_equal(Cb.planes_numpy(), expect(fname, Ab, Bb))
        for i in range(3):
            A = oracle.random_dense(fname, m, l, 70 + i)
            B = oracle.random_dense(fname, l, n, 80 + i)
            Ap.copy_(torch.from_numpy(oracle.pack(fname, A).view(np.int64)))
            Bp.copy_(torch.from_numpy(oracle.pack(fname, B).view(np.int64)))
            Cp.fill_(-1)
            C = sg.m4rm_multiply(A_, B_, sg.M4rmParams(8), out=C_)
            assert np.array_equal(C.planes_numpy(), expect(fname, A, B)), (fname, "after growth", i)


def test_host_buffers_pipelined_chunks():
    """sg_m4rm_host's pipeline: the default chunking at m >= 4096, and every (k-chunks, row
    pieces) pair forced through SG_HOST_KCHUNKS / SG_HOST_CHUNKS on ragged shapes."""
    for fname, m in (("f7", 5000), ("f3", 9001)):
        A = oracle.random_dense(fname, m, 300, 5)
        B = oracle.random_dense(fname, 300, 200, 6)
        Ah = sg.BitslicedMatrix.from_planes(FIELDS[fname], oracle.pack(fname, A), 300, device="cpu")
        Bh = sg.BitslicedMatrix.from_planes(FIELDS[fname], oracle.pack(fname, B), 200, device="cpu")
        C = sg.m4rm_multiply(Ah, Bh)
        assert np.array_equal(C.planes_numpy(), expect(fname, A, B))
    try:
        for fname in FIELDS:
            for (m, l, n) in ((600, 1000, 200), (7, 129, 65), (300, 64, 100), (333, 65, 7)):
                A = oracle.random_dense(fname, m, l, m + n)
                B = oracle.random_dense(fname, l, n, l + 1)
                want = expect(fname, A, B)
                Ah = sg.BitslicedMatrix.from_planes(FIELDS[fname], oracle.pack(fname, A), l, device="cpu")
                Bh = sg.BitslicedMatrix.from_planes(FIELDS[fname], oracle.pack(fname, B), n, device="cpu")
                for pk in (1, 2, 3, 4):
                    for pr in (1, 3, 4):
                        os.environ["SG_HOST_KCHUNKS"], os.environ["SG_HOST_CHUNKS"] = str(pk), str(pr)
                        C = sg.m4rm_multiply(Ah, Bh)
                        assert np.array_equal(C.planes_numpy(), want), (fname, m, l, n, pk, pr)
                for pr in (1, 2, 3):  # row x column piece grid
                    for pc in (2, 3, 4):
                        os.environ["SG_HOST_CHUNKS"], os.environ["SG_HOST_CCHUNKS"] = str(pr), str(pc)
                        C = sg.m4rm_multiply(Ah, Bh)
                        assert np.array_equal(C.planes_numpy(), want), (fname, m, l, n, pr, pc)
                os.environ.pop("SG_HOST_CCHUNKS", None)
    finally:
        os.environ.pop("SG_HOST_KCHUNKS", None)
        os.environ.pop("SG_HOST_CHUNKS", None)
        os.environ.pop("SG_HOST_CCHUNKS", None)


def test_host_streamed_b():
    """sg_m4rm_host with B streamed into a running product (host_streamed, sg_host.cu): the first
    row piece's product waits per k-block for B's chunk flags and takes each tile's k-blocks in
    arrival order (streamed_order).  Forced stream-K warp-specialized plans, every field, ragged
    m / l, first B chunk of 1..64 groups (chunks double), 1..3 row pieces: bit-exact against the oracle, and the streamed path
    must have run (sg_host_streamed_count); l with k-blocks % 4 != 0 falls back."""
    L = _lib.load()
    rt = {"f2": 16, "f3": 8, "gf4": 8, "z4": 8, "f5": 4, "f7": 4, "gf8": 4, "z8": 4}
    try:
        for fname in FIELDS:
            for (m, l, n) in ((2500, 1024, 384), (700, 990, 512), (1800, 2048, 256)):
                A = oracle.random_dense(fname, m, l, m + 7)
                B = oracle.random_dense(fname, l, n, n + 3)
                want = expect(fname, A, B)
                Ah = sg.BitslicedMatrix.from_planes(FIELDS[fname], oracle.pack(fname, A), l, device="cpu")
                Bh = sg.BitslicedMatrix.from_planes(FIELDS[fname], oracle.pack(fname, B), n, device="cpu")
                Ap = sg.BitslicedMatrix(FIELDS[fname], m, l, Ah.planes.pin_memory())
                Bp = sg.BitslicedMatrix(FIELDS[fname], l, n, Bh.planes.pin_memory())
                m4rm_mod.set_plan_override(rt[fname], -1, 2)
                try:
                    for rows in (m, m // 3):
                        m4rm_mod.plan(FIELDS[fname], rows, l, n)
                    forced = True
                except Exception:  # no stream-K warp-specialized variant fits (F2: 2 CTAs per SM)
                    m4rm_mod.set_plan_override(0, 0)
                    forced = False
                for g0, pr, pinned in (("1", "1", 0), ("3", "2", 1), ("16", "3", 0), ("64", "2", 1), ("7", "1", 1)):
                    os.environ["SG_HOST_BFIRST"], os.environ["SG_HOST_CHUNKS"] = g0, pr
                    c0 = L.sg_host_streamed_count()
                    try:
                        C = sg.m4rm_multiply(*((Ap, Bp) if pinned else (Ah, Bh)), sg.M4rmParams(8))
                    except Exception as e:
                        raise AssertionError((fname, m, l, n, g0, pr, pinned)) from e
                    assert C.planes.is_pinned() == bool(pinned)
                    assert np.array_equal(C.planes_numpy(), want), (fname, m, l, n, g0, pr)
                    if forced:
                        assert L.sg_host_streamed_count() == c0 + 1, (fname, m, l, n, g0, pr)
        A = oracle.random_dense("f5", 2500, 1000, 1)  # 125 k-blocks: not streamable
        B = oracle.random_dense("f5", 1000, 256, 2)
        Ah = sg.BitslicedMatrix.from_planes(sg.F5, oracle.pack("f5", A), 1000, device="cpu")
        Bh = sg.BitslicedMatrix.from_planes(sg.F5, oracle.pack("f5", B), 256, device="cpu")
        m4rm_mod.set_plan_override(rt["f5"], -1, 2)
        c0 = L.sg_host_streamed_count()
        assert np.array_equal(sg.m4rm_multiply(Ah, Bh, sg.M4rmParams(8)).planes_numpy(), expect("f5", A, B))
        assert L.sg_host_streamed_count() == c0
    finally:
        os.environ.pop("SG_HOST_BFIRST", None)
        os.environ.pop("SG_HOST_CHUNKS", None)


def test_elementwise_ops_match_dense():
    for fname in ("f2", "f3", "f5", "f7", "gf4", "gf8", "z4", "z8"):
        f = FIELDS[fname]
        a = oracle.random_dense(fname, 13, 131, 1)
        b = oracle.random_dense(fname, 13, 131, 2)
        A, B = sg.BitslicedMatrix.from_dense(f, a), sg.BitslicedMatrix.from_dense(f, b)
        if fname in ("gf4", "gf8"):
            assert np.array_equal(A.add(B).to_dense(), a ^ b)
            assert np.array_equal(A.sub(B).to_dense(), a ^ b)
            for c in range(oracle.ORDER[fname]):  # c * a over GF(4) / GF(8)
                want = oracle.dense_multiply(fname, a.reshape(-1, 1), np.array([[c]], np.uint8)).reshape(a.shape)
                assert np.array_equal(A.scalar_mul(c).to_dense(), want)
            continue
        q = oracle.ORDER[fname]
        assert np.array_equal(A.add(B).to_dense(), (a.astype(int) + b) % q)
        assert np.array_equal(A.sub(B).to_dense(), (a.astype(int) - b) % q)
        assert np.array_equal(A.neg().to_dense(), (-a.astype(int)) % q)
        for c in range(q):
            assert np.array_equal(A.scalar_mul(c).to_dense(), (a.astype(int) * c) % q)
        # padding lanes stay zero
        for M in (A.add(B), A.sub(B), A.neg()):
            tailbits = M.planes_numpy()[:, :, -1] >> np.uint64(131 % 64)
            assert not tailbits.any()


def test_equals_canonicalizes():
    M = sg.BitslicedMatrix.zero(sg.F5, 1, 3)
    N = sg.BitslicedMatrix.zero(sg.F5, 1, 3)
    M.set(0, 1, 1)
    N.planes[1, 0, 0] = 2  # pattern 6 == 1 (mod 5) in column 1
    N.planes[2, 0, 0] = 2
    assert M.equals(N)
    N.set(0, 2, 3)
    assert not M.equals(N)


def test_plugin_block_api_reproduces_product():
    """The _core-style block API (build_table + m4rm_block_<f>) drives a whole product."""
    for fname in ("f2", "f3", "f5", "f7", "gf4", "gf8", "z4", "z8"):
        f = FIELDS[fname]
        m, l, n, k = 70, 45, 130, 6
        A = oracle.random_dense(fname, m, l, 11)
        B = oracle.random_dense(fname, l, n, 12)
        Ag, Bg = sg.BitslicedMatrix.from_dense(f, A), sg.BitslicedMatrix.from_dense(f, B)
        C = torch.zeros_like(Ag.planes[:, :, :1].expand(-1, -1, (n + 63) // 64)).contiguous()
        drv = getattr(_core_cuda, f"m4rm_block_{fname}")
        for s in range((l + k - 1) // k):
            T = sg.build_table(Bg, s, k)
            kp = min(k, l - s * k)
            drv(*[C[d] for d in range(f.bits)], *[Ag.planes[d] for d in range(f.bits)], s * k, kp,
                *[T[d] for d in range(f.bits)], 0, m)
        got = oracle.canonicalize(fname, C.cpu().numpy().view(np.uint64))
        assert np.array_equal(got, expect(fname, A, B)), fname


def test_plugin_accepts_numpy_planes():
    a = oracle.pack("f3", oracle.random_dense("f3", 4, 100, 1))
    b = oracle.pack("f3", oracle.random_dense("f3", 4, 100, 2))
    want = oracle.pack("f3", (oracle.unpack("f3", a, 100).astype(int) + oracle.unpack("f3", b, 100)) % 3)
    _core_cuda.f3_add(a[0], a[1], b[0], b[1])
    assert np.array_equal(a, want)


def test_ext_multiply_matches_karatsuba_golden():
    from paper_0901_1413_b200 import extension
    for c in _golden.cases("gf4"):
        f2 = [sg.BitslicedMatrix.from_dense(sg.F2, (c["A"] >> i) & 1) for i in range(2)]
        g2 = [sg.BitslicedMatrix.from_dense(sg.F2, (c["B"] >> i) & 1) for i in range(2)]
        for method in ("direct", "karatsuba"):
            C = sg.ext_multiply(sg.ExtMatrix(sg.F4, f2), sg.ExtMatrix(sg.F4, g2), method=method)
            got = np.concatenate([C.coeffs[0].planes_numpy(), C.coeffs[1].planes_numpy()])
            assert np.array_equal(got, c["Craw"]), method
            assert extension.base_multiplies == (0 if method == "direct" else 3)


@pytest.mark.parametrize("name", ["f8", "f9", "f25", "f27"])
def test_ext_fields_match_reference_oracle(name):
    """oracle_ext_multiply fixtures (tests/golden/ext_<f>.npz) for every extension field, both
    routes where both exist; 1x1 products reproduce the whole multiplication table."""
    from paper_0901_1413_b200 import extension
    spec = sg.EXT_FIELDS[name]
    z = np.load(f"{_golden.GOLDEN}/ext_{name}.npz")
    methods = ("direct", "karatsuba") if spec.direct is not None else ("karatsuba",)
    for i in range(int(z["count"])):
        A = sg.ExtMatrix.from_dense(spec, list(z[f"c{i}_A"]))
        B = sg.ExtMatrix.from_dense(spec, list(z[f"c{i}_B"]))
        for method in methods:
            C = sg.ext_multiply(A, B, method=method)
            assert np.array_equal(np.stack(C.to_dense()), z[f"c{i}_C"]), (name, i, method)
            if method == "karatsuba":
                assert extension.base_multiplies == (3 if spec.degree == 2 else 6)
    elems, table = z["elems"], z["mul_table"]
    q = len(elems)
    # all q x q products at once: A = column of all elements (q x 1), B = row (1 x q)
    A = sg.ExtMatrix.from_dense(spec, [elems[:, d].reshape(q, 1) for d in range(spec.degree)])
    B = sg.ExtMatrix.from_dense(spec, [elems[:, d].reshape(1, q) for d in range(spec.degree)])
    for method in methods:
        C = np.stack(sg.ext_multiply(A, B, method=method).to_dense(), axis=-1)
        assert np.array_equal(C, table), (name, method)


@pytest.mark.parametrize("fname", ["z4", "z8"])
def test_rings_match_reference_golden(fname):
    for c in _golden.cases(fname):
        C = gpu_multiply(fname, c["A"], c["B"], c["k"])
        assert np.array_equal(C.planes_numpy(), c["Craw"]), (fname, c["m"], c["l"], c["n"], c["k"])


def test_checker_detects_a_corrupted_result():
    """Fault injection: flip one table-sourced bit of a correct result; parity must fail."""
    A = oracle.random_dense("f5", 64, 64, 1)
    B = oracle.random_dense("f5", 64, 64, 2)
    C = gpu_multiply("f5", A, B)
    good = C.planes_numpy()
    assert np.array_equal(good, expect("f5", A, B))
    C.planes[0, 3, 0] ^= 1 << 5
    assert not np.array_equal(C.planes_numpy(), expect("f5", A, B))


def test_stream_ordering_on_side_stream():
    A = oracle.random_dense("f7", 300, 900, 1)
    B = oracle.random_dense("f7", 900, 300, 2)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        Ag = sg.BitslicedMatrix.from_dense(sg.F7, A)
        Bg = sg.BitslicedMatrix.from_dense(sg.F7, B)
        C = sg.m4rm_multiply(Ag, Bg)
    s.synchronize()
    assert np.array_equal(C.planes_numpy(), expect("f7", A, B))


def test_cli_verify_bench_ffops(capsys):
    """The reference CLI's subcommands on the GPU path."""
    from paper_0901_1413_b200 import cli
    assert cli.main(["verify", "--fields", "f3,f7,z8,f4,f8,f9,f25,f27", "--max-dim", "33", "--trials", "5"]) == 0
    out = capsys.readouterr().out
    assert "40 products, 0 failures" in out
    assert cli.main(["bench", "--fields", "f3,f5", "--dims", "64,100", "--reps", "2"]) == 0
    lines = [l for l in capsys.readouterr().out.splitlines() if l and not l.startswith("#")]
    assert lines[0] == "field,n,algorithm,ms,gffops" and len(lines) == 5
    for l in lines[1:]:
        f, n, alg, ms, gff = l.split(",")
        assert abs(float(gff) - 2 * int(n) ** 3 / (float(ms) * 1e-3) / 1e9) <= 1e-3 * float(gff) + 1e-3
    assert cli.main(["ffops", "--field", "f3", "--min", "64", "--max", "80", "--reps", "1"]) == 0
    rows = [l for l in capsys.readouterr().out.splitlines() if l and not l.startswith("#")]
    assert len(rows) == 1 + 17  # header + 64..80 (SPEC.md:613 example)


def test_no_writes_outside_c():
    """Guard words around C stay untouched for ragged shapes and every schedule (stand-in for a
    memcheck run: compute-sanitizer is closed on this pool)."""
    import ctypes
    from paper_0901_1413_b200 import _lib
    L = _lib.load()
    guard = 4096
    cases = [("f3", (77, 301, 130), None), ("f7", (513, 257, 65), None), ("gf4", (1, 9, 1), None),
             ("f5", (300, 1000, 700), None)]
    # the tensor-memory variants (row-slots per thread, both sets), split-K and stream-K, on rows
    # that leave their 4096- / 8192- / 16384-row tiles mostly empty or ragged; and the stream-K
    # hybrid (more tiles than CTAs: whole-tile waves plus a stream-K tail)
    for fname, rt in (("f3", 32), ("gf4", 32), ("z4", 32), ("f2", 32), ("f2", 64), ("f5", 16), ("f7", 16), ("gf8", 16),
                      ("z8", 16)):
        cases += [(fname, (4099, 130, 200), ((rt, 6, 1), (rt, 6, 3), (rt, 6, -1))),
                  (fname, (8200, 72, 129), ((rt, 6, -1),))]
    cases += [("f3", (2300, 64, 4100), ((1, 0, -1), (2, 1, -1))), ("f5", (2300, 64, 4100), ((1, 0, -1), (4, 2, -1)))]
    for fname, (m, l, n), plans in cases:
        f = FIELDS[fname]
        A = sg.BitslicedMatrix.from_dense(f, oracle.random_dense(fname, m, l, 1))
        B = sg.BitslicedMatrix.from_dense(f, oracle.random_dense(fname, l, n, 2))
        want = expect(fname, oracle.unpack(fname, A.planes_numpy(), l), oracle.unpack(fname, B.planes_numpy(), n))
        words = f.bits * m * ((n + 63) // 64)
        for rt, sched, splits in (plans or ((1, 0, 1), (2, 1, 3), (4, 2, 2), (8, 2, 1))):
            m4rm_mod.set_plan_override(rt, splits, sched, 256)
            buf = torch.full((words + 2 * guard,), 0x5A5A5A5A5A5A5A5A, dtype=torch.int64, device="cuda")
            try:
                rc = L.sg_m4rm(f.code, ctypes.c_void_p(A.planes.data_ptr()), ctypes.c_void_p(B.planes.data_ptr()),
                               ctypes.c_void_p(buf.data_ptr() + guard * 8), m, l, n, 8, None, 0,
                               _lib.current_stream_handle())
            finally:
                m4rm_mod.set_plan_override(0, 0, -1, 0)
            if rc == _lib.SG_EUNSUPPORTED:
                continue
            _lib.check(rc)
            torch.cuda.synchronize()
            g = buf.cpu().numpy().view(np.uint64)
            assert (g[:guard] == 0x5A5A5A5A5A5A5A5A).all() and (g[guard + words:] == 0x5A5A5A5A5A5A5A5A).all(), \
                (fname, rt, sched, splits)
            got = g[guard:guard + words].reshape(f.bits, m, -1)
            assert np.array_equal(got, want), (fname, rt, sched, splits)


@pytest.mark.parametrize("fname", list(FIELDS))
def test_classical_multiply_cross_check(fname):
    """classical_multiply (no tables) agrees with m4rm_multiply and the oracle."""
    f = FIELDS[fname]
    for (m, l, n) in ((1, 1, 1), (33, 65, 70), (100, 130, 257)):
        A = oracle.random_dense(fname, m, l, m + l)
        B = oracle.random_dense(fname, l, n, n)
        Ag, Bg = sg.BitslicedMatrix.from_dense(f, A), sg.BitslicedMatrix.from_dense(f, B)
        Cc = sg.classical_multiply(Ag, Bg)
        assert np.array_equal(Cc.planes_numpy(), expect(fname, A, B)), (fname, m, l, n)
        assert np.array_equal(Cc.planes_numpy(), sg.m4rm_multiply(Ag, Bg).planes_numpy())


def test_sharded_multiply_chunked_on_device():
    """dist.sharded_multiply's overlapped path (B in row blocks, per-chunk products summed on the
    GPU) in a one-rank gloo group: bit-identical to the oracle for every field and chunk count."""
    import tempfile

    import torch.distributed as dist

    from paper_0901_1413_b200 import dist as sgdist
    store = tempfile.NamedTemporaryFile(delete=False)
    dist.init_process_group("gloo", init_method=f"file://{store.name}", rank=0, world_size=1)
    try:
        for fname in FIELDS:
            m, l, n = 70, 333, 150
            A = oracle.random_dense(fname, m, l, 5)
            B = oracle.random_dense(fname, l, n, 6)
            want = expect(fname, A, B)
            Am = sg.BitslicedMatrix.from_dense(FIELDS[fname], A)
            Bm = sg.BitslicedMatrix.from_dense(FIELDS[fname], B)
            for chunks in (1, 2, 3, 4, 6):
                C, Bl = sgdist.sharded_multiply(Am, Bm, FIELDS[fname], l, n, chunks=chunks)
                assert np.array_equal(C.planes_numpy(), want), (fname, chunks)
                assert np.array_equal(Bl.planes_numpy(), Bm.planes_numpy())
    finally:
        dist.destroy_process_group()


def test_host_path_thread_safety():
    """Pure functions, safe from any thread: concurrent host-buffer products on
    one device (ctypes drops the GIL) each get their own correct result."""
    import threading
    jobs = []
    for i, fname in enumerate(("f3", "f5", "f7", "gf4", "f2", "z8")):
        m, l, n = 300 + 37 * i, 500 + 11 * i, 200 + 5 * i
        A = oracle.random_dense(fname, m, l, 40 + i)
        B = oracle.random_dense(fname, l, n, 50 + i)
        Ah = sg.BitslicedMatrix.from_planes(FIELDS[fname], oracle.pack(fname, A), l, device="cpu")
        Bh = sg.BitslicedMatrix.from_planes(FIELDS[fname], oracle.pack(fname, B), n, device="cpu")
        jobs.append((fname, Ah, Bh, expect(fname, A, B)))
    errors = []

    def run(job):
        fname, Ah, Bh, want = job
        try:
            for _ in range(5):
                C = sg.m4rm_multiply(Ah, Bh)
                if not np.array_equal(C.planes_numpy(), want):
                    errors.append(fname)
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    threads = [threading.Thread(target=run, args=(j,)) for j in jobs]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors


def test_host_streamed_missing_chunk_fails_cleanly():
    """A B chunk that never lands (SG_HOST_DROP_FLAG test hook): the streamed product's builder
    warps give up after their 10 s wait limit, sg_m4rm_host reports the chunk, and the next call
    on the same device works -- the spin-wait can never hang the GPU."""
    f = sg.F5
    A = oracle.random_dense("f5", 2048, 1024, 81)
    B = oracle.random_dense("f5", 1024, 512, 82)
    want = expect("f5", A, B)
    Ah = sg.BitslicedMatrix(f, 2048, 1024, sg.BitslicedMatrix.from_planes(
        f, oracle.pack("f5", A), 1024, device="cpu").planes.pin_memory())
    Bh = sg.BitslicedMatrix(f, 1024, 512, sg.BitslicedMatrix.from_planes(
        f, oracle.pack("f5", B), 512, device="cpu").planes.pin_memory())
    m4rm_mod.set_plan_override(8, -1, 2)
    try:
        os.environ["SG_HOST_DROP_FLAG"] = "0"
        with pytest.raises(_lib.SliceGemmError, match="timed out waiting for B chunk 0"):
            sg.m4rm_multiply(Ah, Bh, sg.M4rmParams(8))
        os.environ.pop("SG_HOST_DROP_FLAG")
        C = sg.m4rm_multiply(Ah, Bh, sg.M4rmParams(8))
        assert np.array_equal(C.planes_numpy(), want)
    finally:
        os.environ.pop("SG_HOST_DROP_FLAG", None)
        m4rm_mod.set_plan_override(0, 0)


def test_host_streamed_thread_safety():
    """Concurrent streamed-B host products (pinned buffers, the headline's F5 shape class at
    2048 x 1024 x 512) from several threads on one device: each gets its own correct result, and
    the streamed path ran for every call (the per-device pipeline state is serialized, the chunk
    flags carry per-call epochs)."""
    import threading
    L = _lib.load()
    jobs = []
    for i, fname in enumerate(("f5", "f7", "f3", "gf4")):
        m, l, n = 2048 + 256 * i, 1024, 512
        A = oracle.random_dense(fname, m, l, 60 + i)
        B = oracle.random_dense(fname, l, n, 70 + i)
        Ah = sg.BitslicedMatrix(FIELDS[fname], m, l, sg.BitslicedMatrix.from_planes(
            FIELDS[fname], oracle.pack(fname, A), l, device="cpu").planes.pin_memory())
        Bh = sg.BitslicedMatrix(FIELDS[fname], l, n, sg.BitslicedMatrix.from_planes(
            FIELDS[fname], oracle.pack(fname, B), n, device="cpu").planes.pin_memory())
        jobs.append((fname, Ah, Bh, expect(fname, A, B)))
    m4rm_mod.set_plan_override(0, -1, 2)  # stream-K, warp-specialized: streamable
    errors = []
    c0 = L.sg_host_streamed_count()

    def run(job):
        fname, Ah, Bh, want = job
        try:
            for _ in range(4):
                C = sg.m4rm_multiply(Ah, Bh, sg.M4rmParams(8))
                if not np.array_equal(C.planes_numpy(), want):
                    errors.append(fname)
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    try:
        threads = [threading.Thread(target=run, args=(j,)) for j in jobs]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=300)
    finally:
        m4rm_mod.set_plan_override(0, 0)
    assert not errors, errors
    assert L.sg_host_streamed_count() - c0 == 4 * len(jobs)


@pytest.mark.parametrize("fname", ["f3", "f5", "f7", "gf4", "f2"])
def test_extreme_aspect_ratios(fname):
    """Matrix-vector and long-inner-dimension shapes: one tile over 12500 k-blocks (every CTA of
    a stream-K wave on the same tile), one row, one column, a single wide row of C."""
    for (m, l, n) in [(3, 100000, 70), (1, 4096, 4096), (4096, 4096, 1), (1, 1, 20000), (2, 9, 130000)]:
        A = oracle.random_dense(fname, m, l, m + 1)
        B = oracle.random_dense(fname, l, n, n + 2)
        C = gpu_multiply(fname, A, B)
        assert np.array_equal(C.planes_numpy(), expect(fname, A, B)), (fname, m, l, n)


def test_kernel_info_registry():
    """sg_kernel_info: every field has k = 1..8 instantiations that fit on the B200, and the
    warp-specialized ones launch 128 builder threads on top of the lookup threads."""
    info = m4rm_mod.kernel_info(0)
    assert info and all(i["occupancy"] >= 1 and i["regs"] > 0 for i in info if i["k"] == 8)
    for code in range(8):
        assert {i["k"] for i in info if i["field"] == code} == set(range(1, 9))
    assert any(i["schedule"] == 2 for i in info)


def test_multi_device_entry_point():
    """sg_m4rm_multi (one process, several devices; here device 0 listed 1-3 times, i.e. the
    sharding, the B replication and the row reassembly on one GPU): bit-identical to the oracle."""
    from paper_0901_1413_b200 import dist as sgdist
    for fname in ("f3", "f5", "f7", "gf4"):
        m, l, n = 1001, 777, 300
        A = oracle.random_dense(fname, m, l, 11)
        B = oracle.random_dense(fname, l, n, 12)
        want = expect(fname, A, B)
        Ah = sg.BitslicedMatrix.from_planes(FIELDS[fname], oracle.pack(fname, A), l, device="cpu")
        Bh = sg.BitslicedMatrix.from_planes(FIELDS[fname], oracle.pack(fname, B), n, device="cpu")
        for devs in ([0], [0, 0], [0, 0, 0]):
            C = sgdist.multi_device_multiply(Ah, Bh, devs)
            assert np.array_equal(C.planes_numpy(), want), (fname, devs)
    with pytest.raises(ValueError):
        sgdist.multi_device_multiply(Ah, Bh, [99])


def test_sm_reserve_plans_fewer_ctas():
    """sg_set_sm_reserve: a stream-K plan uses (SMs - reserve) x occupancy CTAs; results unchanged."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    A = oracle.random_dense("f5", 4096, 512, 1)
    B = oracle.random_dense("f5", 512, 1024, 2)
    want = expect("f5", A, B)
    try:
        m4rm_mod.set_plan_override(0, -1, 2, 256)
        full = m4rm_mod.plan("f5", 4096, 512, 1024)
        m4rm_mod.set_sm_reserve(8)
        part = m4rm_mod.plan("f5", 4096, 512, 1024)
        assert full["splits"] == part["splits"] == -1
        assert part["ctas"] * sms == full["ctas"] * (sms - 8)
        assert np.array_equal(gpu_multiply("f5", A, B).planes_numpy(), want)
    finally:
        m4rm_mod.set_sm_reserve(0)


def test_fuzz_plans_shapes_fields():
    """Seeded fuzz: random field, shape (incl. word-boundary and tiny / skinny ones), k, and a
    random forced plan (rows per thread, schedule incl. the 8-builder, TMEM-accumulator and fused
    one-launch ones, split count or stream-K, CTA width, SM reserve); every product bit-identical
    to the oracle."""
    rng = np.random.default_rng(2026)
    names = list(FIELDS)
    ran = 0
    for it in range(200):
        fname = names[it % len(names)]
        m = int(rng.choice([1, 7, 63, 64, 65, 200, 513, 1500, 3000]))
        l = int(rng.choice([1, 8, 31, 64, 100, 257, 1000, 2049]))
        n = int(rng.choice([1, 32, 63, 64, 65, 128, 129, 700, 1024]))
        k = int(rng.choice([8, 8, 8, 5, 3, 1, 12]))
        rt = int(rng.choice([0, 1, 2, 4, 8, 16, 32]))
        pipe = int(rng.choice([-1, 0, 1, 2, 5, 6, m4rm_mod.FUSED_SERIAL, m4rm_mod.FUSED_PIPELINED]))
        nt = int(rng.choice([0, 256, 512]))
        splits = int(rng.choice([0, 0, 1, 3, 7, -1]))
        A = oracle.random_dense(fname, m, l, it)
        B = oracle.random_dense(fname, l, n, it + 1000)
        m4rm_mod.set_plan_override(rt, splits, pipe, nt)
        if it % 7 == 0:
            m4rm_mod.set_sm_reserve(8)
        try:
            C = gpu_multiply(fname, A, B, k=k)
        except RuntimeError as e:
            assert "no compiled" in str(e)
            continue
        finally:
            m4rm_mod.set_sm_reserve(0)
        ran += 1
        assert np.array_equal(C.planes_numpy(), expect(fname, A, B)), (fname, m, l, n, k, rt, pipe, nt, splits)
    assert ran >= 40


def test_out_must_not_alias_operands():
    A = sg.BitslicedMatrix.random(sg.F3, 64, 64, seed=0)
    B = sg.BitslicedMatrix.random(sg.F3, 64, 64, seed=1)
    with pytest.raises(ValueError):
        sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=A)
    with pytest.raises(ValueError):
        sg.m4rm_multiply(A, B, sg.M4rmParams(8), out=B)


def test_m4rm_not_slower_than_classical_f3_1024():
    """Acceptance #7 of the reference spec: m4rm_multiply at n = 1024 over F3 is
    at least as fast as classical_multiply (the n^3 / log n advantage); median of 5."""
    import statistics
    A = sg.BitslicedMatrix.random(sg.F3, 1024, 1024, seed=0)
    B = sg.BitslicedMatrix.random(sg.F3, 1024, 1024, seed=1)

    def med(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    t_m4rm = med(lambda: sg.m4rm_multiply(A, B, sg.M4rmParams(8)))
    t_cls = med(lambda: m4rm_mod.classical_multiply(A, B))
    assert t_m4rm <= t_cls, (t_m4rm, t_cls)


def test_c_host_example():
    """examples/c_api_demo.c: the ABI from a plain C host (sg_m4rm_host and sg_pack -> sg_m4rm ->
    sg_unpack), checked against a schoolbook product inside the program."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "examples", "c_api_demo")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(root, "examples")], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "bit-exact" in out.stdout
