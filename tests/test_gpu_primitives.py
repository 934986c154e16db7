"""Parity of the sm_100a primitives with the CPU oracle, through the C-ABI
(Machine / View / Workspace path of include/forge.h).  Sizes and cases follow
SPEC.md:512-522 (size sweep, noncommutative scans, KATs) plus the B200 tile
boundaries and misaligned / strided views."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import COMMUTATIVE_1D, OPS_1D, OPS_2D, SIZES, assert_match, seed_for

pytestmark = pytest.mark.gpu

F = pytest.importorskip("paper_2603_18695_b200.forge")


@pytest.fixture(scope="module")
def m():
    mach = F.Machine(0)
    yield mach
    mach.close()


def upload(m, op, arr, which="T", pad=0):
    buf = F.create_buffer(m, op, max(len(arr) + pad, 1), which=which)
    if len(arr):
        m.write(buf, arr)
    return buf


def view_n(buf, n):
    return F.View(buf, 0, n, 1)


# ---------------------------------------------------------------------------
# mapreduce

@pytest.mark.parametrize("op", COMMUTATIVE_1D)
@pytest.mark.parametrize("n", SIZES)
def test_mapreduce_matches_oracle(m, op, n):
    x = orc.fill(op, n, seed_for(op, n), variant=1 if op == 15 else 0)
    buf = upload(m, op, x)
    ws = F.make_mapreduce_workspace(m, op)
    got, rep = F.mapreduce(m, F.make_semiring(op), view_n(buf, n), ws)
    assert rep.ok
    want, ex, sc = orc.mapreduce(op, x)
    assert_match(op, np.array([got], dtype=F.s_dtype(op)), np.array([want]), ex, sc, f"mapreduce n={n}")
    F.release(m, ws)
    m.destroy_buffer(buf)


def test_mapreduce_kats(m):
    # 1..100 -> 5050, max [3,1,4,1,5] -> 5
    x = np.arange(1, 101, dtype=np.int32)
    b = upload(m, F.I32_SUM, x)
    ws = F.make_mapreduce_workspace(m, F.I32_SUM)
    assert F.mapreduce(m, F.make_semiring(F.I32_SUM), F.make_view(m, b), ws)[0] == 5050
    b2 = upload(m, F.I32_MAX, np.array([3, 1, 4, 1, 5], dtype=np.int32))
    assert F.mapreduce(m, F.make_semiring(F.I32_MAX), F.make_view(m, b2), ws)[0] == 5


def test_mapreduce_errors(m):
    b = upload(m, F.AFFINE_F32, orc.fill(F.AFFINE_F32, 8, 1))
    ws = F.make_mapreduce_workspace(m, F.AFFINE_F32)
    with pytest.raises(F.ForgeError) as e:
        F.mapreduce(m, F.make_semiring(F.AFFINE_F32), F.make_view(m, b), ws)
    assert e.value.name == "InvalidArgument"
    b2 = upload(m, F.I32_SUM, np.zeros(4, np.int32))
    ws2 = F.make_mapreduce_workspace(m, F.I32_SUM)
    empty = F.View(b2, 0, 0, 1)
    assert F.mapreduce(m, F.make_semiring(F.I32_SUM), empty, ws2)[0] == 0
    with pytest.raises(F.ForgeError) as e:
        F.mapreduce(m, F.make_semiring(F.I32_SUM, identity=False), empty, ws2)
    assert e.value.name == "MissingIdentity"


@pytest.mark.parametrize("offset", [1, 2, 3, 5, 7])
@pytest.mark.parametrize("stride", [1, 3])
def test_mapreduce_views(m, offset, stride):
    op = F.F32_SUM
    x = orc.fill(op, 50_000, seed_for(offset, stride))
    b = upload(m, op, x)
    v = F.View(b, offset, (len(x) - offset + stride - 1) // stride, stride)
    ws = F.make_mapreduce_workspace(m, op)
    got, _ = F.mapreduce(m, F.make_semiring(op), v, ws)
    want, ex, sc = orc.mapreduce(op, x[offset::stride])
    assert_match(op, np.array([got], np.float32), np.array([want]), ex, sc)


def test_mapreduce_workspace_reuse(m):
    op = F.I32_SUM
    ws = F.make_mapreduce_workspace(m, op)
    for k in range(20):
        x = orc.fill(op, 3000 + 977 * k, seed_for(k))
        b = upload(m, op, x)
        got, _ = F.mapreduce(m, F.make_semiring(op), F.make_view(m, b), ws)
        assert got == orc.mapreduce(op, x)[0]
        m.destroy_buffer(b)


# ---------------------------------------------------------------------------
# scan

@pytest.mark.parametrize("op", OPS_1D)
@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("inclusive", [True, False])
def test_scan_matches_oracle(m, op, n, inclusive):
    if op in (13,) and n > 100_000:
        pytest.skip("quaternion products: 10^4..10^5 covers SPEC.md:515")
    x = orc.fill(op, n, seed_for(op, n, inclusive), variant=1 if op == 15 else 0)
    a = upload(m, op, x)
    d = F.create_buffer(m, op, max(n, 1), which="S")
    ws = F.make_scan_workspace(m, op, n)
    rep = F.scan(m, F.make_semiring(op), view_n(a, n), view_n(d, n), inclusive, ws)
    assert rep.ok
    got = m.read(d, n, F.s_dtype(op)) if n else np.zeros(0, F.s_dtype(op))
    want, ex, sc = orc.scan(op, inclusive, x)
    assert_match(op, got, want, ex, sc, f"scan n={n} incl={inclusive}")
    F.release(m, ws)
    m.destroy_buffer(a)
    m.destroy_buffer(d)


def test_scan_kats(m):
    # [1,2,3,4] -> [1,3,6,10]; quaternion [i, j] -> [i, k]
    a = upload(m, F.I32_SUM, np.array([1, 2, 3, 4], np.int32))
    d = F.create_buffer(m, F.I32_SUM, 4, which="S")
    ws = F.make_scan_workspace(m, F.I32_SUM, 4)
    F.scan(m, F.make_semiring(F.I32_SUM), F.make_view(m, a), F.make_view(m, d), True, ws)
    assert m.read(d, 4, np.int32).tolist() == [1, 3, 6, 10]
    q = np.zeros(2, dtype=F.QUAT_DTYPE)
    q[0] = (0, 1, 0, 0)
    q[1] = (0, 0, 1, 0)
    aq = upload(m, F.QUAT_F32, q)
    dq = F.create_buffer(m, F.QUAT_F32, 2, which="S")
    wq = F.make_scan_workspace(m, F.QUAT_F32, 2)
    F.scan(m, F.make_semiring(F.QUAT_F32), F.make_view(m, aq), F.make_view(m, dq), True, wq)
    r = m.read(dq, 2, F.QUAT_DTYPE)
    assert tuple(r[0]) == (0, 1, 0, 0) and tuple(r[1]) == (0, 0, 0, 1)


def test_scan_errors(m):
    a = upload(m, F.I32_SUM, np.zeros(4, np.int32))
    d = F.create_buffer(m, F.I32_SUM, 3, which="S")
    ws = F.make_scan_workspace(m, F.I32_SUM, 4)
    with pytest.raises(F.ForgeError) as e:
        F.scan(m, F.make_semiring(F.I32_SUM), F.make_view(m, a), F.make_view(m, d), True, ws)
    assert e.value.name == "DimensionMismatch"
    d4 = F.create_buffer(m, F.I32_SUM, 4, which="S")
    with pytest.raises(F.ForgeError) as e:
        F.scan(m, F.make_semiring(F.I32_SUM, identity=False), F.make_view(m, a), F.make_view(m, d4), False, ws)
    assert e.value.name == "MissingIdentity"
    # a workspace made for 4 elements holds 32 packed tile states: a 100_000-
    # element scan fits (at packed slots), a 10^7-element one does not
    small = F.make_scan_workspace(m, F.I32_SUM, 4)
    mid = upload(m, F.I32_SUM, np.arange(100_000, dtype=np.int32))
    md = F.create_buffer(m, F.I32_SUM, 100_000, which="S")
    assert F.scan(m, F.make_semiring(F.I32_SUM), F.make_view(m, mid), F.make_view(m, md), True, small).ok
    assert np.array_equal(m.read(md, 100_000, np.int32), np.cumsum(np.arange(100_000), dtype=np.int64).astype(np.int32))
    big = upload(m, F.I32_SUM, np.zeros(10_000_000, np.int32))
    bd = F.create_buffer(m, F.I32_SUM, 10_000_000, which="S")
    with pytest.raises(F.ForgeError) as e:
        F.scan(m, F.make_semiring(F.I32_SUM), F.make_view(m, big), F.make_view(m, bd), True, small)
    assert e.value.name == "WorkspaceTooSmall"
    with pytest.raises(F.ForgeError) as e:
        F.scan(m, F.make_semiring(F.I32_SUM), F.make_view(m, a), F.make_view(m, d4), True, ws,
               F.ArchParams(warp_width=64, threads_per_block=256))
    assert e.value.name == "Unsupported"


@pytest.mark.parametrize("op", [F.I32_SUM, F.F32_SUM, F.MAT2_U32, F.AFFINE_F32])
@pytest.mark.parametrize("offset,stride", [(1, 1), (3, 1), (5, 1), (0, 2), (1, 3)])
def test_scan_views(m, op, offset, stride):
    n_all = 20_011
    x = orc.fill(op, n_all, seed_for(op, offset, stride))
    a = upload(m, op, x)
    d = F.create_buffer(m, op, n_all, which="S")
    cnt = (n_all - offset + stride - 1) // stride
    src = F.View(a, offset, cnt, stride)
    dst = F.View(d, offset, cnt, stride)
    ws = F.make_scan_workspace(m, op, cnt)
    F.scan(m, F.make_semiring(op), src, dst, True, ws)
    got = m.read(d, n_all, F.s_dtype(op))[offset::stride]
    want, ex, sc = orc.scan(op, True, x[offset::stride])
    assert_match(op, got, want, ex, sc, "strided/misaligned scan")


def test_scan_workspace_reuse_epochs(m):
    # The tile-state epoch advances every launch: reuse one workspace for many
    # scans of different sizes (stale states must never be consumed).
    op = F.MAT2_U32
    ws = F.make_scan_workspace(m, op, 300_000)
    for k in range(12):
        n = [300_000, 1025, 77_777, 1, 4096, 262_143][k % 6]
        x = orc.fill(op, n, seed_for(k, n))
        a = upload(m, op, x)
        d = F.create_buffer(m, op, n, which="S")
        F.scan(m, F.make_semiring(op), F.make_view(m, a), F.make_view(m, d), k % 2 == 0, ws)
        got = m.read(d, n, F.s_dtype(op))
        want, _, _ = orc.scan(op, k % 2 == 0, x)
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), f"launch {k}"
        m.destroy_buffer(a)
        m.destroy_buffer(d)


def test_scan_mixed_paths_share_workspace(m):
    # The persistent TMA kernel (aligned contiguous input) and the general
    # kernel (misaligned / strided) alternate on ONE workspace: ticket, done
    # counter and epoch must stay consistent across both.
    op = F.I32_SUM
    n_all = 250_001
    x = orc.fill(op, n_all, 4242)
    a = upload(m, op, x)
    d = F.create_buffer(m, op, n_all, which="S")
    ws = F.make_scan_workspace(m, op, n_all)
    for k in range(10):
        off = 0 if k % 2 == 0 else 1 + k
        cnt = n_all - off - (k * 997)
        F.scan(m, F.make_semiring(op), F.View(a, off, cnt, 1), F.View(d, off, cnt, 1), k % 3 != 0, ws)
        got = m.read(d, n_all, np.int32)[off:off + cnt]
        want, _, _ = orc.scan(op, k % 3 != 0, x[off:off + cnt])
        assert np.array_equal(got, want), f"launch {k}"


def test_scan_noncommutative_mat2_exact(m):
    # 2x2 wrapping-integer matrix scan equals the sequential oracle exactly.
    op = F.MAT2_U32
    for n in (10_000, 1_000_003):
        x = orc.fill(op, n, seed_for(n))
        a = upload(m, op, x)
        d = F.create_buffer(m, op, n, which="S")
        ws = F.make_scan_workspace(m, op, n)
        F.scan(m, F.make_semiring(op), F.make_view(m, a), F.make_view(m, d), True, ws)
        got = m.read(d, n, F.s_dtype(op))
        want, _, _ = orc.scan(op, True, x)
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


# ---------------------------------------------------------------------------
# matvec / vecmat / mapreduce_2d

SHAPES = [(1, 10_000), (10, 1_000), (100, 100), (1_000, 10), (10_000, 1), (3, 5), (1024, 1024), (257, 129)]


@pytest.mark.parametrize("op", OPS_2D)
@pytest.mark.parametrize("shape", SHAPES)
def test_matvec_vecmat(m, op, shape):
    n, p = shape
    A = orc.fill(op, n * p, seed_for(op, n, p))
    for which in ("matvec", "vecmat"):
        red, outs = (n, p) if which == "matvec" else (p, n)
        x = orc.fill(op, red, seed_for(op, n, p, 7))
        ab = upload(m, op, A)
        xb = upload(m, op, x)
        yb = F.create_buffer(m, op, outs, which="S")
        ws = F.make_mat_workspace(m, op, red, outs)
        fn = F.matvec if which == "matvec" else F.vecmat
        rep = fn(m, F.make_semiring(op), F.make_view(m, ab), n, p, F.make_view(m, xb), F.make_view(m, yb), ws)
        assert rep.ok
        got = m.read(yb, outs, F.s_dtype(op))
        want, ex, sc = (orc.matvec if which == "matvec" else orc.vecmat)(op, A, n, p, x)
        assert_match(op, got, want, ex, sc, f"{which} {shape}")
        for b in (ab, xb, yb):
            m.destroy_buffer(b)
        F.release(m, ws)


# Shapes that reach the planner's other branches: the 4-column gevm kernel
# with row splits and a partial last column group (p % 4 != 0), and the gemv
# two-level split fold (many column splits per row block).
PLAN_SHAPES = [(65536, 7), (4096, 1021), (2048, 16384), (8, 4099), (24576, 5)]


@pytest.mark.parametrize("op", [F.MV_F32_PLUS_TIMES, F.MV_F32_MIN_PLUS])
@pytest.mark.parametrize("shape", PLAN_SHAPES)
def test_matvec_vecmat_plans(m, op, shape):
    n, p = shape
    A = orc.fill(op, n * p, seed_for(op, n, p, 3))
    for which in ("matvec", "vecmat"):
        red, outs = (n, p) if which == "matvec" else (p, n)
        x = orc.fill(op, red, seed_for(op, n, p, 9))
        ab, xb = upload(m, op, A), upload(m, op, x)
        yb = F.create_buffer(m, op, outs, which="S")
        ws = F.make_mat_workspace(m, op, red, outs)
        fn = F.matvec if which == "matvec" else F.vecmat
        for _ in range(2):  # twice: tickets must reset themselves
            rep = fn(m, F.make_semiring(op), F.make_view(m, ab), n, p, F.make_view(m, xb), F.make_view(m, yb), ws)
            assert rep.ok
            got = m.read(yb, outs, F.s_dtype(op))
            want, ex, sc = (orc.matvec if which == "matvec" else orc.vecmat)(op, A, n, p, x)
            assert_match(op, got, want, ex, sc, f"{which} {shape}")
        for b in (ab, xb, yb):
            m.destroy_buffer(b)
        F.release(m, ws)


def test_matrix_kats(m):
    # identity matvec / vecmat; tropical 2x2.
    op = F.MV_F32_PLUS_TIMES
    ab = upload(m, op, np.array([1, 0, 0, 1], np.float32))
    xb = upload(m, op, np.array([3, 5], np.float32))
    yb = F.create_buffer(m, op, 2, which="S")
    ws = F.make_mat_workspace(m, op, 2, 2)
    F.matvec(m, F.make_semiring(op), F.make_view(m, ab), 2, 2, F.make_view(m, xb), F.make_view(m, yb), ws)
    assert m.read(yb, 2, np.float32).tolist() == [3, 5]
    F.vecmat(m, F.make_semiring(op), F.make_view(m, ab), 2, 2, F.make_view(m, xb), F.make_view(m, yb), ws)
    assert m.read(yb, 2, np.float32).tolist() == [3, 5]
    op = F.MV_F32_MIN_PLUS
    ab = upload(m, op, np.array([0, 1, 2, 0], np.float32))
    xb = upload(m, op, np.array([0, 0], np.float32))
    F.matvec(m, F.make_semiring(op), F.make_view(m, ab), 2, 2, F.make_view(m, xb), F.make_view(m, yb), ws)
    assert m.read(yb, 2, np.float32).tolist() == [0, 0]


def test_mapreduce_2d_kats(m):
    # column sums of 3x2 ones -> [3,3]; row maxima [[1,9],[5,2]] -> [9,5]
    ab = upload(m, F.F32_SUM, np.ones(6, np.float32))
    ob = F.create_buffer(m, F.F32_SUM, 3, which="S")
    ws = F.make_mat_workspace(m, F.F32_SUM, 3, 3)
    F.mapreduce_2d(m, F.make_semiring(F.F32_SUM), F.make_view(m, ab), 3, 2, F.ROWS, F.View(ob, 0, 2, 1), ws)
    assert m.read(ob, 2, np.float32).tolist() == [3, 3]
    A = np.array([1, 5, 9, 2], np.float32)  # column-major [[1,9],[5,2]]
    ab2 = upload(m, F.F32_MAX, A)
    F.mapreduce_2d(m, F.make_semiring(F.F32_MAX), F.make_view(m, ab2), 2, 2, F.COLS, F.View(ob, 0, 2, 1), ws)
    assert m.read(ob, 2, np.float32).tolist() == [9, 5]


@pytest.mark.parametrize("op", [F.F32_SUM, F.I32_MAX, F.MAT2_U32, F.F32_MIN])
@pytest.mark.parametrize("axis", [0, 1])
def test_mapreduce_2d_matches_oracle(m, op, axis):
    n, p = 300, 170
    A = orc.fill(op, n * p, seed_for(op, axis))
    ab = upload(m, op, A)
    outs = p if axis == 0 else n
    ob = F.create_buffer(m, op, outs, which="S")
    ws = F.make_mat_workspace(m, op, n if axis == 0 else p, outs)
    F.mapreduce_2d(m, F.make_semiring(op), F.make_view(m, ab), n, p, axis, F.make_view(m, ob), ws)
    got = m.read(ob, outs, F.s_dtype(op))
    want, ex, sc = (orc.matvec if axis == 0 else orc.vecmat)(op, A, n, p, None)
    assert_match(op, got, want, ex, sc, "mapreduce_2d")


def test_matvec_strided_x_and_y(m):
    op = F.MV_F32_PLUS_TIMES
    n, p = 500, 300
    A = orc.fill(op, n * p, 11)
    x = orc.fill(op, 2 * n, 12)
    ab, xb = upload(m, op, A), upload(m, op, x)
    yb = F.create_buffer(m, op, 3 * p, which="S")
    ws = F.make_mat_workspace(m, op, n, p)
    F.matvec(m, F.make_semiring(op), F.make_view(m, ab), n, p, F.View(xb, 1, n, 2), F.View(yb, 2, p, 3), ws)
    got = m.read(yb, 3 * p, np.float32)[2::3]
    want, ex, sc = orc.matvec(op, A, n, p, np.ascontiguousarray(x[1::2]))
    assert_match(op, got, want, ex, sc, "strided matvec")


def test_matrix_errors(m):
    op = F.MV_F32_PLUS_TIMES
    ab = upload(m, op, np.zeros(6, np.float32))
    xb = upload(m, op, np.zeros(3, np.float32))
    yb = F.create_buffer(m, op, 3, which="S")
    ws = F.make_mat_workspace(m, op, 3, 3)
    with pytest.raises(F.ForgeError) as e:
        F.matvec(m, F.make_semiring(op), F.make_view(m, ab), 2, 2, F.make_view(m, xb), F.make_view(m, yb), ws)
    assert e.value.name == "DimensionMismatch"
    with pytest.raises(F.ForgeError) as e:
        F.matvec(m, F.make_semiring(op), F.View(ab, 0, 6, 1), 3, 2, F.View(xb, 0, 3, 1), F.View(yb, 0, 2, 1), ws)
        F.matvec(m, F.make_semiring(op), F.View(ab, 0, 3, 2), 3, 1, F.View(xb, 0, 3, 1), F.View(yb, 0, 1, 1), ws)
    assert e.value.name == "InvalidArgument"


def test_matrix_empty_reduction_fills_identity(m):
    op = F.MV_F32_MIN_PLUS
    ab = upload(m, op, np.zeros(1, np.float32))
    xb = upload(m, op, np.zeros(1, np.float32))
    yb = F.create_buffer(m, op, 4, which="S")
    ws = F.make_mat_workspace(m, op, 0, 4)
    F.matvec(m, F.make_semiring(op), F.View(ab, 0, 0, 1), 0, 4, F.View(xb, 0, 0, 1), F.make_view(m, yb), ws)
    assert np.all(np.isinf(m.read(yb, 4, np.float32)))
    with pytest.raises(F.ForgeError) as e:
        F.matvec(m, F.make_semiring(op, identity=False), F.View(ab, 0, 0, 1), 0, 4, F.View(xb, 0, 0, 1),
                 F.make_view(m, yb), ws)
    assert e.value.name == "MissingIdentity"


# ---------------------------------------------------------------------------
# vcopy

@pytest.mark.parametrize("n", [0, 1, 3, 31, 4099, 1_000_003, 4_000_004])
@pytest.mark.parametrize("desc,dtype", [("f32", np.float32), ("u8", np.uint8), ("f64", np.float64),
                                        ("struct(u8@0,f64@8,u16@16;size=24)", np.dtype((np.void, 24)))])
def test_vcopy(m, n, desc, dtype):
    rng = np.random.default_rng(n)
    src = rng.integers(0, 256, size=n * np.dtype(dtype).itemsize, dtype=np.uint8).view(dtype)
    a = m.create_buffer(desc, n + 8)
    b = m.create_buffer(desc, n + 8)
    if n:
        m.write(a, src)
    rep = F.vcopy(m, F.View(a, 0, n, 1), F.View(b, 0, n, 1), 4)
    assert rep.ok
    if n:
        assert np.array_equal(m.read(b, n, dtype).view(np.uint8), src.view(np.uint8))


@pytest.mark.parametrize("off_a,off_b", [(0, 0), (4, 8), (1, 1), (1, 2)])
def test_vcopy_offsets_bulk_sizes(m, off_a, off_b):
    """>= 8 MiB copies take the TMA bulk path when both views are 16-byte
    aligned (offsets 0/4/8 f32), the vector path otherwise; chunk tails included."""
    n = (3 << 20) + 4 * 1237
    rng = np.random.default_rng(off_a * 7 + off_b)
    src = rng.standard_normal(n).astype(np.float32)
    a = m.create_buffer("f32", n + 16)
    b = m.create_buffer("f32", n + 16)
    m.write(a, np.concatenate([np.zeros(off_a, np.float32), src]))
    rep = F.vcopy(m, F.View(a, off_a, n, 1), F.View(b, off_b, n, 1), 4)
    assert rep.ok
    got = m.read(b, n + off_b, np.float32)[off_b:]
    assert np.array_equal(got.view(np.uint32), src.view(np.uint32))
