#!/usr/bin/env python3
"""Generates tests/golden/reference_vm.npz: outputs of the UNMODIFIED reference
primitives (/root/reference/proj, compiled by oracle/ref/build_ref.py into
oracle/_ref/libforge_ref.so) on seeded synthetic inputs.

Inputs are not stored: they are regenerated bit-exactly from
(op, n, seed, variant) by the oracle's generator (oracle.c gen_one), so the
fixture stays small.  Run here (where /root/reference exists):
    python tests/golden/make_golden.py
The committed .npz lets tests pin the oracle against the reference on machines
without /root/reference.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as orc  # noqa: E402
from oracle.ref import build_ref  # noqa: E402

OUT = Path(__file__).resolve().parent / "reference_vm.npz"

SCAN_OPS = list(range(16))
MR_OPS = [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 11, 14, 15]
SIZES = [1, 31, 33, 257, 4097, 10007]
MAT_OPS = [32, 33, 34, 35, 36, 37]
SHAPES = [(1, 300), (10, 100), (64, 64), (300, 3), (1000, 1)]


def seed(*p):
    s = 0x601D0000
    for v in p:
        s = (s * 1_000_003 + int(v)) & 0xFFFFFFFFFFFF
    return s


def main():
    build_ref.build()
    data = {}
    for op in SCAN_OPS:
        for n in SIZES:
            x = orc.fill(op, n, seed(op, n))
            for incl in (1, 0):
                y, _ = orc.ref_scan(op, bool(incl), x, backend=orc.SIM, seed=7)
                data[f"scan_{op}_{n}_{incl}"] = y.view(np.uint8)
    for op in MR_OPS:
        for n in SIZES:
            x = orc.fill(op, n, seed(op, n, 1))
            v, _ = orc.ref_mapreduce(op, x, backend=orc.SIM, seed=3)
            data[f"mapreduce_{op}_{n}"] = np.array([v]).view(np.uint8)
    for op in MAT_OPS:
        for n, p in SHAPES:
            A = orc.fill(op, n * p, seed(op, n, p))
            xm = orc.fill(op, n, seed(op, n, p, 1))
            xv = orc.fill(op, p, seed(op, n, p, 2))
            y, _ = orc.ref_matvec(op, A, n, p, xm, backend=orc.THREADS)
            z, _ = orc.ref_vecmat(op, A, n, p, xv, backend=orc.THREADS)
            data[f"matvec_{op}_{n}_{p}"] = y.view(np.uint8)
            data[f"vecmat_{op}_{n}_{p}"] = z.view(np.uint8)
    for op in (0, 2, 6, 12):  # mapreduce_2d through the reference's own delegation
        n, p = 37, 23
        A = orc.fill(op, n * p, seed(op, 2))
        y, _ = orc.ref_matvec(op, A, n, p, None, backend=orc.THREADS)
        z, _ = orc.ref_vecmat(op, A, n, p, None, backend=orc.THREADS)
        data[f"mr2d_rows_{op}"] = y.view(np.uint8)
        data[f"mr2d_cols_{op}"] = z.view(np.uint8)
    pats = []
    for nitem in (1, 2, 4, 8, 16):
        for off in range(2 * nitem):
            segs = orc.ref_vload_pattern(off, nitem)
            pats.append([nitem, off] + segs + [0] * (16 - len(segs)))
    data["vload_patterns"] = np.array(pats, dtype=np.int32)
    probes = np.array([orc.ref().ref_error_probe(i) for i in range(5)], dtype=np.int32)
    data["error_probes"] = probes
    ws = []
    import ctypes as C
    for prim, acc, n, p in ((0, 4, 4096, 0), (0, 4, 0, 0), (1, 4, 123, 0), (2, 4, 100, 7), (3, 8, 100, 7)):
        out = C.c_uint64()
        orc.ref().ref_required_workspace(prim, acc, n, p, C.byref(out))
        ws.append([prim, acc, n, p, out.value])
    data["required_workspace"] = np.array(ws, dtype=np.int64)
    data["scan_tiles_4096"] = np.array([orc.ref().ref_scan_tiles(4096), orc.ref().ref_scan_tiles(4097)])
    np.savez_compressed(OUT, **data)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(data)} arrays)")


if __name__ == "__main__":
    main()
