"""Shared helpers for the parity tests: run a primitive through the C-ABI
(paper_2603_18695_b200.forge) and compare with the CPU oracle."""
from __future__ import annotations

import numpy as np

from oracle import oracle as orc

# Parity tolerances: |got - exact_64| <= tol * sum|terms|.
TOL = {0: 1e-5, 1: 1e-5, 4: 1e-12, 10: 1e-5, 13: 1e-5, 14: 1e-5, 15: 1e-5, 32: 1e-5, 36: 1e-12}

# SPEC.md:512's sweep plus BASELINE C1 (2^20: whole 8192-element tiles, no tail)
SIZES = [0, 1, 31, 32, 33, 255, 256, 257, 4095, 4096, 4097, 100_000, 1_000_000, 1 << 20]
OPS_1D = list(range(16))
COMMUTATIVE_1D = [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 11, 14, 15]
OPS_2D = [32, 33, 34, 35, 36, 37]


def seed_for(*parts) -> int:
    s = 0x5EED0000
    for p in parts:
        s = (s * 1_000_003 + int(p)) & 0xFFFFFFFFFFFF
    return s


def assert_match(op, got, want_s, exact, scale, what=""):
    """Exact ops: bitwise equality of the S values; float ops: tolerance."""
    nc = orc.ncomp(op)
    got = np.ascontiguousarray(np.atleast_1d(got))
    want_s = np.ascontiguousarray(np.atleast_1d(want_s))
    if nc == 0:
        g = got.view(np.uint8) if got.dtype.names is None else got.view(np.uint8)
        w = np.atleast_1d(want_s).view(np.uint8)
        if not np.array_equal(g, w):
            gg, ww = np.atleast_1d(got), np.atleast_1d(want_s)
            bad = np.nonzero(gg != ww)[0] if gg.dtype.names is None else np.nonzero(
                np.any(gg.view(np.uint8).reshape(len(gg), -1) != ww.view(np.uint8).reshape(len(ww), -1), axis=1))[0]
            raise AssertionError(f"{what}: op {op} mismatch at {bad[:5]} (of {len(bad)}): "
                                 f"got {gg[bad[:3]]} want {ww[bad[:3]]}")
        return 0.0
    ok, rel = orc.within(op, got, exact, scale, TOL.get(op, 1e-5))
    assert ok, f"{what}: op {op} error/scale {rel:.3e} > tol {TOL.get(op, 1e-5)}"
    return rel
