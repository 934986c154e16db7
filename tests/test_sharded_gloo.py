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
        x = orc.fill(op, n, seed)
        sh = sharded.shard_of(n, rank, world)
        src = torch.from_numpy(x[sh.lo:sh.hi].view(np.uint8).copy())
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
