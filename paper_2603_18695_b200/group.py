"""Single-process multi-GPU groups over the C-ABI (include/forge.h forge_group_*,
paper_2603_18695_b200/csrc/group.cu) for torch-tensor callers.

`Group(devices)` holds one shard per listed device (rank order).  Distinct
devices exchange over NCCL (ncclCommInitAll clique); a list repeating ONE
device is the emulated group (G shards on one GPU, same exchange logic, the
all-gather by device copies).  Every shard has its own workspace and stream;
the sharded calls are ordered after the caller's current torch stream on every
shard device and the caller's stream waits for them (`sync=True`, default).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import capi, dev
from .forge import check, op_info


def shard_range(total: int, rank: int, count: int) -> tuple[int, int]:
    lo, hi = C.c_uint64(), C.c_uint64()
    check(capi.load().forge_shard_range(total, rank, count, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def cyclic_quantum(op: int) -> int:
    q = C.c_uint64()
    check(capi.load().forge_cyclic_chunk_quantum(op, C.byref(q)))
    return q.value


def cyclic_local_n(n: int, chunk: int, rank: int, count: int) -> int:
    out = C.c_uint64()
    check(capi.load().forge_cyclic_local_n(n, chunk, rank, count, C.byref(out)))
    return out.value


def cyclic_split(n: int, chunk: int, G: int) -> list[list[tuple[int, int]]]:
    """Global [lo, hi) ranges of every shard's chunks, in its local order."""
    out = [[] for _ in range(G)]
    for c, lo in enumerate(range(0, n, chunk)):
        out[c % G].append((lo, min(lo + chunk, n)))
    return out


def _ptrs(ts) -> C.Array:
    return (C.c_void_p * len(ts))(*[C.c_void_p(t if isinstance(t, int) else t.data_ptr()) for t in ts])


class Group:
    def __init__(self, devices: list[int]):
        self.lib = capi.load()
        self.devices = list(devices)
        arr = (C.c_int32 * len(devices))(*devices)
        h = C.c_void_p()
        check(self.lib.forge_group_create(arr, len(devices), C.byref(h)))
        self.h = h
        cnt, emu = C.c_int32(), C.c_int32()
        check(self.lib.forge_group_size(self.h, C.byref(cnt), C.byref(emu)))
        self.size, self.emulated = cnt.value, bool(emu.value)
        self.streams = []
        for r in range(self.size):
            s = C.c_void_p()
            check(self.lib.forge_group_stream(self.h, r, C.byref(s)))
            self.streams.append(torch.cuda.ExternalStream(s.value, device=torch.device("cuda", devices[r])))
        self.ws = []
        for d in devices:
            with torch.cuda.device(d):
                self.ws.append(dev.Workspace())

    def close(self) -> None:
        if self.h:
            check(self.lib.forge_group_destroy(self.h))
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- plumbing
    def _workspaces(self, prim: int, op: int, ns: list[int], ps: list[int] | None = None):
        ptrs, sizes = [], []
        for r in range(self.size):
            with torch.cuda.device(self.devices[r]):
                if prim == capi.PRIM_SCAN:  # the sharded scan also reduces its shard with this workspace
                    self.ws[r].ensure(dev.workspace_bytes(capi.PRIM_MAPREDUCE, op, ns[r]), self.streams[r])
                p, b = self.ws[r].for_(prim, op, ns[r], ps[r] if ps else 0, stream=self.streams[r])
            ptrs.append(p)
            sizes.append(b)
        return _ptrs(ptrs), (C.c_uint64 * self.size)(*sizes)

    def _enter(self) -> None:  # shard streams wait for the caller's work on each device
        for r in range(self.size):
            with torch.cuda.device(self.devices[r]):
                self.streams[r].wait_stream(torch.cuda.current_stream())

    def _leave(self, sync: bool) -> None:
        if sync:
            for r in range(self.size):
                with torch.cuda.device(self.devices[r]):
                    torch.cuda.current_stream().wait_stream(self.streams[r])

    # -- sharded primitives
    def mapreduce(self, op: int, src: list, ns: list[int], sync: bool = True) -> bytes:
        self._enter()
        ws, wb = self._workspaces(capi.PRIM_MAPREDUCE, op, ns)
        out = (C.c_ubyte * 16)()
        check(self.lib.forge_sharded_mapreduce(self.h, op, _ptrs(src), (C.c_uint64 * self.size)(*ns), ws, wb, out))
        self._leave(sync)
        return bytes(out)[: op_info(op)["s_size"]]

    def scan(self, op: int, inclusive: bool, src: list, dst: list, ns: list[int], sync: bool = True) -> None:
        self._enter()
        ws, wb = self._workspaces(capi.PRIM_SCAN, op, ns)
        check(self.lib.forge_sharded_scan(self.h, op, 1 if inclusive else 0, _ptrs(src), _ptrs(dst),
                                          (C.c_uint64 * self.size)(*ns), ws, wb))
        self._leave(sync)

    def matvec(self, op: int, A_blocks: list, n: int, p: int, xs: list, ys: list, sync: bool = True) -> None:
        self._enter()
        cols = [shard_range(p, r, self.size) for r in range(self.size)]
        ws, wb = self._workspaces(capi.PRIM_MATVEC, op, [n] * self.size, [max(hi - lo, 1) for lo, hi in cols])
        check(self.lib.forge_sharded_matvec(self.h, op, _ptrs(A_blocks), n, p, _ptrs(xs), _ptrs(ys), ws, wb))
        self._leave(sync)

    def vecmat(self, op: int, A_blocks: list, n: int, p: int, xs: list, zs: list, sync: bool = True) -> None:
        self._enter()
        rows = [shard_range(n, r, self.size) for r in range(self.size)]
        ws, wb = self._workspaces(capi.PRIM_VECMAT, op, [max(hi - lo, 1) for lo, hi in rows], [p] * self.size)
        check(self.lib.forge_sharded_vecmat(self.h, op, _ptrs(A_blocks), n, p, _ptrs(xs), _ptrs(zs), ws, wb))
        self._leave(sync)

    def scan_cyclic(self, op: int, inclusive: bool, src: list, dst: list, n: int, chunk: int,
                    sync: bool = True) -> None:
        """Scan of a block-cyclic array (chunk c on shard c mod G) with the
        cross-GPU decoupled look-back; src[r] / dst[r] hold shard r's chunks
        back to back (cyclic_split gives their global ranges)."""
        self._enter()
        ptrs, sizes = [], []
        for r in range(self.size):
            with torch.cuda.device(self.devices[r]):
                need = C.c_uint64()
                check(self.lib.forge_cyclic_workspace_bytes(op, cyclic_local_n(n, chunk, r, self.size),
                                                            C.byref(need)))
                b = self.ws[r].ensure(need.value, self.streams[r])
            ptrs.append(b.data_ptr())
            sizes.append(b.numel())
        check(self.lib.forge_sharded_scan_cyclic(self.h, op, 1 if inclusive else 0, _ptrs(src), _ptrs(dst), n, chunk,
                                                 _ptrs(ptrs), (C.c_uint64 * self.size)(*sizes)))
        self._leave(sync)
