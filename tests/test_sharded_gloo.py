"""Multi-process (gloo, world_size 2 and 3, CPU) test of the sharded exchange
logic in paper_2603_18695_b200/sharded.py.  The GPU kernels are replaced by a
test backend computing each rank's LOCAL step with the CPU oracle, so what is
tested here is the distribution: shard bounds, the all-gather of partials /
totals, the rank-order folds, the carry seeding of the local scans.  The result
of the sharded computation must equal the oracle on the whole array (bit for
bit for exact operators)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc

# fold of S values uses the op without its map
OP_ONLY = {1: 0, 14: 0}


class OracleBackend:
    def s_size(self, op):
        return orc.s_dtype(op).itemsize

    def t_size(self, op):
        return orc.t_dtype(op).itemsize

    def new_bytes(self, nbytes):
        return torch.zeros(nbytes, dtype=torch.uint8)

    @staticmethod
    def _arr(t, dtype, n):
        return t.numpy().view(np.uint8)[: n * dtype.itemsize].view(dtype)

    @staticmethod
    def _put(out, value_bytes):
        if value_bytes:
            out[: len(value_bytes)] = torch.frombuffer(bytearray(value_bytes), dtype=torch.uint8)

    def mapreduce(self, op, src, n, out):
        v, _, _ = orc.mapreduce(op, self._arr(src, orc.t_dtype(op), n))
        self._put(out, np.array([v], dtype=orc.s_dtype(op)).tobytes())

    reduce_ordered = mapreduce

    def fold(self, op, values, count, out, exclusive_upto=-1):
        m = count if exclusive_upto < 0 else min(exclusive_upto, count)
        fop = OP_ONLY.get(op, op)
        vals = self._arr(values, orc.s_dtype(op), count)[:m]
        if m:
            v, _, _ = orc.mapreduce(fop, np.ascontiguousarray(vals))
            self._put(out, np.array([v], dtype=orc.s_dtype(op)).tobytes())

    def _block(self, op, A, n, p, lda, a_offset):
        lda = lda or n
        flat = self._arr(A, orc.t_dtype(op), A.numel() // orc.t_dtype(op).itemsize)
        cols = [flat[a_offset + j * lda: a_offset + j * lda + n] for j in range(p)]
        return np.ascontiguousarray(np.concatenate(cols)) if p else flat[:0]

    def matvec(self, op, A, n, p, x, y, lda=0, a_offset=0):
        blk = self._block(op, A, n, p, lda, a_offset)
        v, _, _ = orc.matvec(op, blk, n, p, self._arr(x, orc.t_dtype(op), n))
        self._put(y, v.tobytes())

    def vecmat(self, op, A, n, p, x, z, lda=0, a_offset=0):
        blk = self._block(op, A, n, p, lda, a_offset)
        v, _, _ = orc.vecmat(op, blk, n, p, self._arr(x, orc.t_dtype(op), p))
        self._put(z, v.tobytes())

    def scan(self, op, inclusive, src, dst, n, carry_in):
        carry = None if carry_in is None else self._arr(carry_in, orc.s_dtype(op), 1)[0]
        y, _, _ = orc.scan(op, inclusive, self._arr(src, orc.t_dtype(op), n), carry=carry)
        self._put(dst, y.tobytes())


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_18695_b200 import sharded
    be = OracleBackend()
    results = []
    for kind, op, n, inclusive, seed in cases:
        if kind not in ("matvec", "vecmat"):
            x = orc.fill(op, n, seed)
            sh = sharded.shard_of(n, rank, world)
            src = torch.from_numpy(x[sh.lo:sh.hi].view(np.uint8).copy())
        if kind in ("matvec", "vecmat"):
            (nn, pp), in_place = n, inclusive
            A = orc.fill(op, nn * pp, seed)
            xv = orc.fill(op, nn if kind == "matvec" else pp, seed + 1)
            ss = orc.s_dtype(op).itemsize
            total = pp if kind == "matvec" else nn
            sh = sharded.shard_of(total, rank, world)
            if in_place:
                At = torch.from_numpy(A.view(np.uint8).copy())
            elif kind == "matvec":  # the rank's own column block (contiguous)
                At = torch.from_numpy(A[sh.lo * nn: sh.hi * nn].view(np.uint8).copy())
            else:  # the rank's own row block, column-major with lda = rows
                blk = A.reshape(pp, nn)[:, sh.lo:sh.hi]
                At = torch.from_numpy(np.ascontiguousarray(blk).reshape(-1).view(np.uint8).copy())
            loc = torch.zeros(max(sh.n, 1) * ss, dtype=torch.uint8)
            full = torch.zeros(total * ss, dtype=torch.uint8)
            fn = sharded.sharded_matvec if kind == "matvec" else sharded.sharded_vecmat
            fn(op, At, nn, pp, torch.from_numpy(xv.view(np.uint8).copy()), loc, in_place=in_place,
               gather_into=full, backend=be)
            results.append((loc.numpy().tobytes()[: sh.n * ss], full.numpy().tobytes()))
            continue
        if kind == "mapreduce":
            r = sharded.sharded_mapreduce(op, src, sh.n, backend=be)
            results.append(r.numpy().tobytes()[: orc.s_dtype(op).itemsize])
        else:
            dst = torch.zeros(max(sh.n, 1) * orc.s_dtype(op).itemsize, dtype=torch.uint8)
            sharded.sharded_scan(op, inclusive, src, dst, sh.n, backend=be)
            results.append(dst.numpy().tobytes()[: sh.n * orc.s_dtype(op).itemsize])
    q.put((rank, results))
    dist.barrier()
    dist.destroy_process_group()


CASES = [
    ("mapreduce", 5, 10_001, True, 1),
    ("mapreduce", 6, 777, True, 2),
    ("mapreduce", 11, 5000, True, 3),
    ("mapreduce", 1, 4099, True, 4),
    ("scan", 5, 10_003, True, 5),
    ("scan", 5, 10_003, False, 6),
    ("scan", 12, 3001, True, 7),   # Mat2: exact, non-commutative
    ("scan", 12, 3001, False, 8),
    ("scan", 11, 4097, True, 9),
    ("scan", 0, 20_000, True, 10),
    ("scan", 10, 2048, False, 11),
    ("scan", 5, 2, True, 12),      # fewer elements than ranks for world 3
    # matrix shards: (kind, op, (n, p), in_place, seed); column / row blocks,
    # own blocks and in place in a replicated A (lda), ragged and tiny shapes
    ("matvec", 33, (517, 301), False, 13),   # min-plus: exact
    ("matvec", 35, (300, 7), True, 14),      # i32 plus-times: exact
    ("matvec", 37, (64, 5), False, 15),      # Mat2: ordered, non-commutative
    ("matvec", 32, (1000, 130), True, 16),   # f32
    ("vecmat", 33, (701, 90), False, 17),
    ("vecmat", 35, (257, 33), True, 18),
    ("vecmat", 37, (50, 9), True, 19),
    ("vecmat", 32, (2, 400), False, 20),     # fewer rows than ranks for world 3
]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, (kind, op, n, inclusive, seed) in enumerate(CASES):
        if kind in ("matvec", "vecmat"):
            nn, pp = n
            A = orc.fill(op, nn * pp, seed)
            xv = orc.fill(op, nn if kind == "matvec" else pp, seed + 1)
            want, ex, sc = (orc.matvec if kind == "matvec" else orc.vecmat)(op, A, nn, pp, xv)
            blocks = np.frombuffer(b"".join(got[r][ci][0] for r in range(world)), dtype=orc.s_dtype(op))
            for g in [blocks] + [np.frombuffer(got[r][ci][1], dtype=orc.s_dtype(op)) for r in range(world)]:
                assert len(g) == len(want)
                if orc.ncomp(op):
                    assert orc.within(op, g, ex, sc, 1e-5)[0], (kind, op)
                else:
                    assert g.tobytes() == want.tobytes(), (kind, op, n)
            continue
        x = orc.fill(op, n, seed)
        if kind == "mapreduce":
            want, ex, sc = orc.mapreduce(op, x)
            for r in range(world):
                g = np.frombuffer(got[r][ci], dtype=orc.s_dtype(op))
                if orc.ncomp(op):
                    assert orc.within(op, g, ex, sc, 1e-5)[0]
                else:
                    assert g.tobytes() == np.array([want]).tobytes(), (kind, op, r)
        else:
            want, ex, sc = orc.scan(op, inclusive, x)
            g = np.frombuffer(b"".join(got[r][ci] for r in range(world)), dtype=orc.s_dtype(op))
            assert len(g) == n
            if orc.ncomp(op):
                ok, rel = orc.within(op, g, ex, sc, 1e-5)
                assert ok, (op, rel)
            else:
                assert g.tobytes() == want.tobytes(), (kind, op, inclusive)
