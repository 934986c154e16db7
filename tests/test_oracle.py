"""Pins the CPU oracle (oracle/oracle.c) before it is trusted as the checker:
  * against the SPEC.md known-answer vectors;
  * against the committed golden outputs of the reference VM
    (tests/golden/reference_vm.npz, made by tests/golden/make_golden.py);
  * live against the reference VM when oracle/_ref/libforge_ref.so is built
    (this container), on both of its backends.
Exact operators must agree bit for bit; floating operators within the stated
tolerance of the 64-bit oracle value."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as orc
from tests.golden.make_golden import MAT_OPS, MR_OPS, SCAN_OPS, SHAPES, SIZES, seed
from tests.helpers import TOL

GOLDEN = Path(__file__).resolve().parent / "golden" / "reference_vm.npz"


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def same(op, got, ref_bytes, exact=None, scale=None, what=""):
    got = np.atleast_1d(got)
    ref = ref_bytes.view(got.dtype)
    if orc.ncomp(op) == 0:
        assert np.array_equal(got.view(np.uint8), ref_bytes), f"{what}: oracle != reference (exact op {op})"
    else:
        ok, rel = orc.within(op, ref, exact, scale, TOL.get(op, 1e-5))
        assert ok, f"{what}: reference VM vs f64 oracle {rel:.2e}"


# ---- SPEC known answers ------------------------------------------------------

def test_kat_mapreduce():
    assert orc.mapreduce(5, np.arange(1, 101, dtype=np.int32))[0] == 5050
    assert orc.mapreduce(6, np.array([3, 1, 4, 1, 5], np.int32))[0] == 5


def test_kat_scan():
    d, _, _ = orc.scan(5, True, np.array([1, 2, 3, 4], np.int32))
    assert d.tolist() == [1, 3, 6, 10]
    q = np.zeros(2, dtype=orc.QUAT)
    q[0] = (0, 1, 0, 0)
    q[1] = (0, 0, 1, 0)
    d, _, _ = orc.scan(13, True, q)
    assert tuple(d[1]) == (0, 0, 0, 1)  # i*j = k
    d, _, _ = orc.scan(5, False, np.array([1, 2, 3, 4], np.int32))
    assert d.tolist() == [0, 1, 3, 6]  # exclusive: dst[0] = identity (primitives.hpp:592)


def test_kat_matrix():
    I2 = np.array([1, 0, 0, 1], np.float32)
    x = np.array([3, 5], np.float32)
    assert orc.matvec(32, I2, 2, 2, x)[0].tolist() == [3, 5]
    assert orc.vecmat(32, I2, 2, 2, x)[0].tolist() == [3, 5]
    trop = np.array([0, 1, 2, 0], np.float32)
    assert orc.matvec(33, trop, 2, 2, np.zeros(2, np.float32))[0].tolist() == [0, 0]
    # mapreduce_2d: SPEC.md:361-362
    assert orc.matvec(0, np.ones(6, np.float32), 3, 2, None)[0].tolist() == [3, 3]
    assert orc.vecmat(2, np.array([1, 5, 9, 2], np.float32), 2, 2, None)[0].tolist() == [9, 5]


def test_kat_vload_pattern():
    assert orc.vload_pattern(0, 4) == [4]
    assert orc.vload_pattern(1, 4) == [1, 2, 1]
    assert orc.vload_pattern(2, 4) == [2, 2]
    assert orc.vload_pattern(3, 8) == [1, 4, 2, 1]
    assert orc.vload_pattern(0, 3) == 3              # InvalidNitem status


def test_vload_pattern_law():
    # segments are powers of two, sum to nitem, each aligned to its size.
    for nitem in (1, 2, 4, 8, 16):
        for off in range(64):
            segs = orc.vload_pattern(off, nitem)
            assert sum(segs) == nitem
            o = off
            for s in segs:
                assert s & (s - 1) == 0 and o % s == 0
                o += s


def test_kat_unitfloat8():
    L = orc.lib()
    assert L.orc_uf8_decode(0) == -1.0 and L.orc_uf8_decode(255) == 1.0
    assert abs(L.orc_uf8_decode(128) - 0.0039216) < 1e-6
    assert all(L.orc_uf8_encode(L.orc_uf8_decode(c)) == c for c in range(256))


def test_generator_is_deterministic_and_offsettable():
    a = orc.fill(0, 1000, 42)
    b = orc.fill(0, 1000, 42)
    assert np.array_equal(a, b)
    c = orc.fill(0, 600, 42, index_base=400)
    assert np.array_equal(a[400:], c)
    assert a.min() >= -1 and a.max() < 1
    v = orc.fill(12, 10, 7)
    assert v.dtype == orc.MAT2


def test_streaming_oracle_matches_materialised():
    for op in (1, 6, 11, 14):
        x = orc.fill(op, 50_000, 99)
        v1, e1, s1 = orc.mapreduce(op, x)
        v2, e2, s2 = orc.mapreduce_synthetic(op, 50_000, 99)
        assert np.array_equal(np.array([v1]).view(np.uint8), np.array([v2]).view(np.uint8))
    for op in (0, 10, 12):
        x = orc.fill(op, 20_000, 5)
        d, _, _ = orc.scan(op, True, x)
        bad, _ = orc.check_scan_synthetic(op, True, 20_000, 5, d, 1e-5)
        assert bad == 0


def test_scan_carry_in():
    x = orc.fill(5, 100, 3)
    full, _, _ = orc.scan(5, True, x)
    tail, _, _ = orc.scan(5, True, x[60:], carry=full[59])
    assert np.array_equal(tail, full[60:])
    ex, _, _ = orc.scan(5, False, x[60:], carry=full[59])
    assert ex[0] == full[59]


# ---- golden fixtures from the reference VM -----------------------------------------

@pytest.mark.parametrize("op", SCAN_OPS)
def test_oracle_scan_matches_reference_golden(golden, op):
    for n in SIZES:
        x = orc.fill(op, n, seed(op, n))
        for incl in (1, 0):
            d, ex, sc = orc.scan(op, bool(incl), x)
            same(op, d, golden[f"scan_{op}_{n}_{incl}"], ex, sc, f"scan op={op} n={n} incl={incl}")


@pytest.mark.parametrize("op", MR_OPS)
def test_oracle_mapreduce_matches_reference_golden(golden, op):
    for n in SIZES:
        x = orc.fill(op, n, seed(op, n, 1))
        v, ex, sc = orc.mapreduce(op, x)
        same(op, np.array([v]), golden[f"mapreduce_{op}_{n}"], ex, sc, f"mapreduce op={op} n={n}")


@pytest.mark.parametrize("op", MAT_OPS)
def test_oracle_matrix_matches_reference_golden(golden, op):
    for n, p in SHAPES:
        A = orc.fill(op, n * p, seed(op, n, p))
        xm = orc.fill(op, n, seed(op, n, p, 1))
        xv = orc.fill(op, p, seed(op, n, p, 2))
        y, ey, sy = orc.matvec(op, A, n, p, xm)
        z, ez, sz = orc.vecmat(op, A, n, p, xv)
        same(op, y, golden[f"matvec_{op}_{n}_{p}"], ey, sy, f"matvec {op} {n}x{p}")
        same(op, z, golden[f"vecmat_{op}_{n}_{p}"], ez, sz, f"vecmat {op} {n}x{p}")


def test_oracle_mapreduce_2d_matches_reference_golden(golden):
    for op in (0, 2, 6, 12):
        n, p = 37, 23
        A = orc.fill(op, n * p, seed(op, 2))
        y, ey, sy = orc.matvec(op, A, n, p, None)
        z, ez, sz = orc.vecmat(op, A, n, p, None)
        same(op, y, golden[f"mr2d_rows_{op}"], ey, sy, "mapreduce_2d rows")
        same(op, z, golden[f"mr2d_cols_{op}"], ez, sz, "mapreduce_2d cols")


def test_oracle_vload_patterns_match_reference_golden(golden):
    for row in golden["vload_patterns"]:
        nitem, off = int(row[0]), int(row[1])
        segs = [int(s) for s in row[2:] if s]
        assert orc.vload_pattern(off, nitem) == segs


def test_reference_error_probes_golden(golden):
    # exclusive w/o identity -> MissingIdentity(4), non-commutative mapreduce ->
    # InvalidArgument(1), empty mapreduce w/o identity -> MissingIdentity(4),
    # warp_width 48 -> InvalidArgument(1), length mismatch -> DimensionMismatch(6)
    assert golden["error_probes"].tolist() == [4, 1, 4, 1, 6]


# ---- live reference VM (only where it was built) -------------------------------------

ref_only = pytest.mark.skipif(not orc.ref_available(), reason="reference VM not built here")


@ref_only
@pytest.mark.parametrize("op", [5, 12, 10, 11, 0])
def test_oracle_vs_live_reference_both_backends(op):
    n = 9001
    x = orc.fill(op, n, 1234 + op)
    d, ex, sc = orc.scan(op, True, x)
    for backend in (orc.SIM, orc.THREADS):
        y, _ = orc.ref_scan(op, True, x, backend=backend, seed=5)
        same(op, d, y.view(np.uint8), ex, sc, f"live scan backend={backend}")


@pytest.mark.parametrize("op", [0, 5, 10, 11, 12])
@pytest.mark.parametrize("inclusive", [True, False])
def test_check_scan_synthetic_at_matches_full_check(op, inclusive):
    """The sampled streaming check (used for the 2^33 C5 size) agrees with the
    oracle's own scan: clean samples pass, one corrupted sample is caught."""
    n, seed = 20_011, 0x5EED0C06
    x = orc.fill(op, n, seed)
    want, _, _ = orc.scan(op, inclusive, x)
    idx = np.array(sorted({0, 1, 2, 4095, 4096, 9999, n - 1}), dtype=np.uint64)
    got_at = want[idx.astype(np.int64)].copy()
    bad, _ = orc.check_scan_synthetic_at(op, inclusive, seed, idx, got_at, 1e-5)
    assert bad == 0
    raw = got_at.view(np.uint8).copy()
    k = 3 * got_at.dtype.itemsize
    raw[k:k + 4] ^= np.frombuffer(np.float32(1.5).tobytes(), np.uint8)
    bad, _ = orc.check_scan_synthetic_at(op, inclusive, seed, idx, raw.view(got_at.dtype), 1e-5)
    assert bad == 1


@pytest.mark.parametrize("op", [2, 3, 11])  # f32 max, f32 min, arg-max
def test_oracle_special_values_order_independent(op):
    # The order-independent max / min / arg-max (NaN canonical or first-NaN,
    # -0 < +0): any permutation of special-value data folds to the same bits,
    # which is what lets a GPU tree match the sequential oracle bit for bit.
    x = orc.fill(op, 20_000, 0xC0FFEE + op, variant=2)
    r0 = np.atleast_1d(orc.mapreduce(op, x)[0]).view(np.uint8).tobytes()
    rng = np.random.default_rng(op)
    for _ in range(5):
        y = x[rng.permutation(len(x))]
        assert np.atleast_1d(orc.mapreduce(op, y)[0]).view(np.uint8).tobytes() == r0
    # and a reassociated fold (pairwise halves) agrees too
    h = len(x) // 2
    a, b = orc.mapreduce(op, x[:h])[0], orc.mapreduce(op, x[h:])[0]
    pair = np.concatenate([np.atleast_1d(a), np.atleast_1d(b)]).astype(x.dtype)
    assert np.atleast_1d(orc.mapreduce(op, pair)[0]).view(np.uint8).tobytes() == r0
