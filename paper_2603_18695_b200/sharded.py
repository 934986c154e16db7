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
  matvec     (gevm, y = x^T A, reference primitives.hpp:776-791) columns
             sharded in contiguous blocks: rank r folds columns
             shard_of(p, r, G) of the column-major A — its own n x p_r block
             (contiguous), or the block IN PLACE in a replicated global A
             (pointer + lo*n, lda = n).  No collective; optional all-gather of
             the y blocks into the full y on every rank.
  vecmat     (gemv, z = A x, primitives.hpp:795-807) rows sharded: rank r
             folds rows shard_of(n, r, G) — its own n_r x p block (lda = n_r),
             or the rows in place in a replicated global A (pointer + lo,
             lda = n; forge_dev_vecmat_lda).  No collective; optional
             all-gather of the z blocks.

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
        # every byte is written by a kernel before it is read: no fill kernel
        return torch.empty(nbytes, dtype=torch.uint8, device="cuda")

    def mapreduce(self, op, src, n, out):
        self.dev.mapreduce(op, src, n, out, self.ws_reduce)

    def reduce_ordered(self, op, src, n, out):
        self.dev.reduce_ordered(op, src, n, out, self.ws_reduce)

    def scan(self, op, inclusive, src, dst, n, carry_in):
        self.dev.scan(op, inclusive, src, dst, n, self.ws_scan, carry_in=carry_in)

    def fold(self, op, values, count, out, exclusive_upto=-1):
        self.dev.fold(op, values, count, out, exclusive_upto=exclusive_upto)

    def _at(self, op, A, a_offset):
        if a_offset == 0:
            return A
        return A.data_ptr() + a_offset * self.t_size(op)

    def matvec(self, op, A, n, p, x, y, lda=0, a_offset=0):
        self.dev.matvec(op, self._at(op, A, a_offset), n, p, x, y, self.ws_mat, lda=lda)

    def vecmat(self, op, A, n, p, x, z, lda=0, a_offset=0):
        self.dev.vecmat(op, self._at(op, A, a_offset), n, p, x, z, self.ws_mat, lda=lda)


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
    if world == 1:  # one shard: the local mapreduce is the result
        result = be.new_bytes(ss)
        be.mapreduce(op, local_src, n_local, result)
        return result
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


def _all_gather_blocks(local: torch.Tensor, total: int, elem_size: int, world: int, out: torch.Tensor,
                       group=None) -> None:
    """All-gather of contiguous output blocks (block r = shard_of(total, r, world),
    ragged) into `out` (total * elem_size bytes) on every rank, in rank order."""
    width = ((total + world - 1) // world) * elem_size
    pad = torch.zeros(width, dtype=torch.uint8, device=local.device)
    nb = local.numel()
    if nb:
        pad[:nb].copy_(local.reshape(-1)[:nb])
    g = _all_gather_bytes(pad, world, group).view(world, width)
    for r in range(world):
        sh = shard_of(total, r, world)
        if sh.n:
            out[sh.lo * elem_size: sh.hi * elem_size].copy_(g[r, : sh.n * elem_size])


def sharded_matvec(op: int, A, n: int, p: int, x, y_local, *, in_place: bool = False, gather_into=None,
                   backend=None, group=None) -> Shard:
    """gevm y = x^T A over the GLOBAL n x p column-major A, columns sharded:
    this rank computes y[lo:hi] for its columns [lo, hi) = shard_of(p, rank, G).
    `A` is this rank's n x (hi-lo) column block, or (in_place=True) the whole
    replicated A whose block is read in place.  `x` is the full length-n vector.
    `gather_into` (optional, p outputs): every rank receives the full y."""
    be = backend or DeviceBackend()
    rank, world = _world(group)
    sh = shard_of(p, rank, world)
    if sh.n:
        be.matvec(op, A, n, sh.n, x, y_local, lda=n, a_offset=sh.lo * n if in_place else 0)
    if gather_into is not None:
        _all_gather_blocks(y_local, p, be.s_size(op), world, gather_into, group)
    return sh


def sharded_vecmat(op: int, A, n: int, p: int, x, z_local, *, in_place: bool = False, gather_into=None,
                   backend=None, group=None) -> Shard:
    """gemv z = A x over the GLOBAL n x p column-major A, rows sharded: this rank
    computes z[lo:hi] for its rows [lo, hi) = shard_of(n, rank, G).  `A` is
    this rank's (hi-lo) x p block (column-major, lda = hi-lo), or
    (in_place=True) the whole replicated A whose rows are read in place
    (lda = n: a row block of a column-major matrix is strided).  `x` is the full
    length-p vector; `gather_into` (optional, n outputs) all-gathers z."""
    be = backend or DeviceBackend()
    rank, world = _world(group)
    sh = shard_of(n, rank, world)
    if sh.n:
        if in_place:
            be.vecmat(op, A, sh.n, p, x, z_local, lda=n, a_offset=sh.lo)
        else:
            be.vecmat(op, A, sh.n, p, x, z_local, lda=sh.n)
    if gather_into is not None:
        _all_gather_blocks(z_local, n, be.s_size(op), world, gather_into, group)
    return sh
