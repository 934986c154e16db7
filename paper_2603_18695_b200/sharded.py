"""Multi-GPU sharding of the primitives, one process per GPU.

  mapreduce  contiguous n/G shard per rank -> one-kernel local mapreduce (the S
             partial stays on the device) -> all-gather of sizeof(S) bytes per
             rank -> every rank folds the G partials IN RANK ORDER on the device
             (deterministic; works for struct types / custom ops where NCCL's
             built-in reductions cannot).
  scan       reduce-then-scan: order-preserving local reduce of the shard ->
             all-gather of the G shard totals -> exclusive rank-order fold of
             totals[0..rank) into a device carry -> local single-pass scan seeded
             with that carry (no host synchronisation anywhere).  HBM traffic
             3n/G per GPU.
  matvec     (gevm, y = x^T A) columns sharded: independent, no collective.
  vecmat     (gemv, z = A x)  rows sharded: each rank holds its (n/G) x p block;
             independent, no collective.

The collective is torch.distributed (NCCL over NVLink/NVSwitch on B200s; gloo in
the CPU tests).  The local compute is a backend object: `DeviceBackend` calls
the sm_100a kernels through the C-ABI; tests inject their own backend to run the
exchange logic on CPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


class DeviceBackend:
    """Local compute on this rank's GPU (libforge.so device-pointer layer)."""

    def __init__(self):
        from . import dev  # noqa: WPS433 (lazy: loads libforge.so)
        self.dev = dev
        # one workspace per layout family: no re-zeroing when calls alternate
        self.ws_reduce, self.ws_scan, self.ws_mat = dev.Workspace(), dev.Workspace(), dev.Workspace()

    def s_size(self, op: int) -> int:
        from .forge import op_info
        return op_info(op)["s_size"]

    def t_size(self, op: int) -> int:
        from .forge import op_info
        return op_info(op)["t_size"]

    def new_bytes(self, nbytes: int) -> torch.Tensor:
        return torch.zeros(nbytes, dtype=torch.uint8, device="cuda")

    def mapreduce(self, op, src, n, out):
        self.dev.mapreduce(op, src, n, out, self.ws_reduce)

    def reduce_ordered(self, op, src, n, out):
        self.dev.reduce_ordered(op, src, n, out, self.ws_reduce)

    def scan(self, op, inclusive, src, dst, n, carry_in):
        self.dev.scan(op, inclusive, src, dst, n, self.ws_scan, carry_in=carry_in)

    def fold(self, op, values, count, out, exclusive_upto=-1):
        self.dev.fold(op, values, count, out, exclusive_upto=exclusive_upto)

    def matvec(self, op, A, n, p, x, y):
        self.dev.matvec(op, A, n, p, x, y, self.ws_mat)

    def vecmat(self, op, A, n, p, x, z):
        self.dev.vecmat(op, A, n, p, x, z, self.ws_mat)


@dataclass
class Shard:
    """The contiguous [lo, hi) range of a length-n array owned by `rank`."""
    lo: int
    hi: int

    @property
    def n(self) -> int:
        return self.hi - self.lo


def shard_of(n: int, rank: int, world: int) -> Shard:
    return Shard(n * rank // world, n * (rank + 1) // world)


def _all_gather_bytes(local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """All-gather of a small byte tensor into one [world * len] tensor in rank order."""
    out = torch.empty(world * local.numel(), dtype=torch.uint8, device=local.device)
    if world == 1:
        out.copy_(local)
        return out
    backend = dist.get_backend(group)
    if backend == "nccl":
        dist.all_gather_into_tensor(out, local, group=group)
    else:
        parts = list(out.view(world, -1).unbind(0))
        dist.all_gather(parts, local, group=group)
        out = torch.cat(parts)
    return out


def _world(group=None) -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def sharded_mapreduce(op: int, local_src, n_local: int, backend=None, group=None) -> torch.Tensor:
    """Global mapreduce of the concatenation of every rank's shard (rank order);
    returns the S value (as bytes) on every rank's device."""
    be = backend or DeviceBackend()
    rank, world = _world(group)
    ss = be.s_size(op)
    part = be.new_bytes(ss)
    be.mapreduce(op, local_src, n_local, part)
    gathered = _all_gather_bytes(part, world, group)
    result = be.new_bytes(ss)
    be.fold(op, gathered, world, result)
    return result


def sharded_scan(op: int, inclusive: bool, local_src, local_dst, n_local: int, backend=None,
                 group=None) -> torch.Tensor:
    """Scan of the global array whose rank-ordered shards are `local_src`;
    writes this rank's slice of the global scan into `local_dst`.  Returns the
    gathered shard totals (bytes, rank order), or None for a single rank (plain
    local scan)."""
    be = backend or DeviceBackend()
    rank, world = _world(group)
    ss = be.s_size(op)
    if world == 1:  # one shard: no carry to compute, no exchange
        be.scan(op, inclusive, local_src, local_dst, n_local, None)
        return None
    total = be.new_bytes(ss)
    be.reduce_ordered(op, local_src, n_local, total)
    totals = _all_gather_bytes(total, world, group)
    carry = None
    if rank > 0:
        carry = be.new_bytes(ss)
        be.fold(op, totals, world, carry, exclusive_upto=rank)
    be.scan(op, inclusive, local_src, local_dst, n_local, carry)
    return totals


def sharded_matvec(op: int, A_local, n: int, p_local: int, x, y_local, backend=None):
    """gevm over a column block: rank r owns columns [lo, hi) of the n x p
    column-major A (contiguous in memory) and produces y[lo:hi]."""
    be = backend or DeviceBackend()
    be.matvec(op, A_local, n, p_local, x, y_local)


def sharded_vecmat(op: int, A_local, n_local: int, p: int, x, z_local, backend=None):
    """gemv over a row block: rank r owns the (n_local x p) column-major block of
    rows [lo, hi) and produces z[lo:hi]."""
    be = backend or DeviceBackend()
    be.vecmat(op, A_local, n_local, p, x, z_local)
