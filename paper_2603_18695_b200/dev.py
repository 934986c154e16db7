"""Device-pointer layer over the C-ABI for torch-tensor callers.

torch provides HBM allocations and streams (plumbing); every computation is a
libforge.so sm_100a kernel launched on the given stream.  Tensors are passed by
data_ptr(); element types are the op's T / S (struct types travel as uint8
tensors of n * sizeof bytes).  All calls are asynchronous and stream-ordered.
"""
from __future__ import annotations

import ctypes as C
import functools

import torch

from . import capi
from .forge import ForgeError, check, op_info


def _lib():
    return capi.load()


_raw_stream = torch._C._cuda_getCurrentRawStream  # current stream handle without a Stream object
_cur_device = torch._C._cuda_getDevice


def _stream(stream) -> int:
    """cudaStream_t of `stream` (a torch Stream, a raw handle, or None = the
    current stream).  The raw accessors cost ~0.2 us; torch.cuda.current_stream()
    builds a Python object per call (~3 us — more than the kernel launch)."""
    if stream is None:
        return _raw_stream(_cur_device())
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _ptr(t) -> int:
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    if not t.is_cuda:
        raise ForgeError(capi.ERR_INVALID_ARGUMENT, "tensor must live on a CUDA device")
    return t.data_ptr()


@functools.lru_cache(maxsize=256)
def _workspace_bytes(device: int, prim: int, op: int, n: int, p_cols: int) -> int:
    out = C.c_uint64()
    check(_lib().forge_dev_workspace_bytes(prim, op, n, p_cols, C.byref(out)))
    return out.value


def workspace_bytes(prim: int, op: int, n: int, p_cols: int = 0) -> int:
    """Bytes of device workspace a call needs (cached per device and shape: a
    ctypes round trip per launch is host latency small launches would pay)."""
    return _workspace_bytes(_cur_device(), prim, op, n, p_cols)


class Workspace:
    """A zero-initialised device byte buffer, grown on demand.  The kernels
    leave it reusable (self-resetting tickets / epochs) and the library
    re-zeroes it when it moves to another primitive's layout, so one
    Workspace may serve every primitive in turn; it must not be used by two
    launches in flight at once."""

    def __init__(self, device=None):
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.buf = torch.zeros(256, dtype=torch.uint8, device=self.device)
        self._shapes: dict = {}  # (prim, op, n, p_cols) -> (ptr, bytes, buffer generation)
        self._gen = 0

    def ensure(self, nbytes: int, stream=None) -> torch.Tensor:
        """Grows the buffer to >= nbytes.  The new buffer is allocated and zeroed
        ON `stream` (the stream the next kernel runs on), and the old one is
        recorded on it so the caching allocator cannot hand its memory out
        while kernels queued there may still use it."""
        if self.buf.numel() < nbytes:
            s = torch.cuda.current_stream(self.device) if stream is None else stream
            if not isinstance(s, torch.cuda.Stream):
                s = torch.cuda.ExternalStream(int(s), device=self.device)
            old = self.buf
            with torch.cuda.stream(s):
                self.buf = torch.zeros(max(nbytes, 2 * old.numel()), dtype=torch.uint8, device=self.device)
            old.record_stream(s)
            self._gen += 1
        return self.buf

    def for_(self, prim: int, op: int, n: int, p_cols: int = 0, stream=None) -> tuple[int, int]:
        # (ptr, bytes) per shape while the buffer stays the same: small launches
        # are host-bound, and this is one dict lookup instead of four calls
        key = (prim, op, n, p_cols)
        hit = self._shapes.get(key)
        if hit is not None and hit[2] == self._gen:
            return hit[0], hit[1]
        need = workspace_bytes(prim, op, n, p_cols)
        b = self.buf if self.buf.numel() >= need else self.ensure(need, stream)
        if len(self._shapes) > 64:
            self._shapes.clear()
        self._shapes[key] = (b.data_ptr(), b.numel(), self._gen)
        return b.data_ptr(), b.numel()


def empty(op: int, n: int, which: str = "T", device=None) -> torch.Tensor:
    info = op_info(op)
    size = info["t_size"] if which == "T" else info["s_size"]
    return torch.empty(n * size, dtype=torch.uint8, device=device or "cuda")


def fill_synthetic(op: int, dst: torch.Tensor, n: int, seed: int, index_base: int = 0, variant: int = 0,
                   stream=None) -> None:
    check(_lib().forge_dev_fill_synthetic(op, _ptr(dst), n, seed, index_base, variant, _stream(stream)))


def mapreduce(op: int, src, n: int, out, ws: Workspace, stream=None) -> None:
    w, wb = ws.for_(capi.PRIM_MAPREDUCE, op, n, stream=stream)
    rc = _lib().forge_dev_mapreduce(op, _ptr(src), n, _ptr(out), w, wb, _stream(stream))
    if rc:
        check(rc)


def reduce_ordered(op: int, src, n: int, out, ws: Workspace, stream=None) -> None:
    w, wb = ws.for_(capi.PRIM_MAPREDUCE, op, n, stream=stream)
    check(_lib().forge_dev_reduce_ordered(op, _ptr(src), n, _ptr(out), w, wb, _stream(stream)))


def scan(op: int, inclusive: bool, src, dst, n: int, ws: Workspace, carry_in=None, total_out=None,
         stream=None) -> None:
    w, wb = ws.for_(capi.PRIM_SCAN, op, n, stream=stream)
    rc = _lib().forge_dev_scan(op, 1 if inclusive else 0, _ptr(src), _ptr(dst), n, _ptr(carry_in),
                               _ptr(total_out), w, wb, _stream(stream))
    if rc:
        check(rc)


def matvec(op: int, A, n: int, p_cols: int, x, y, ws: Workspace, stream=None, lda: int = 0) -> None:
    """y[j] = op_i f(x[i], A[i,j]) over an n x p column-major A whose columns are
    `lda` (0 = n) elements apart; A may be a pointer (int) into a larger matrix."""
    w, wb = ws.for_(capi.PRIM_MATVEC, op, n, p_cols, stream=stream)
    check(_lib().forge_dev_matvec_lda(op, _ptr(A), n, p_cols, lda, _ptr(x), _ptr(y), w, wb, _stream(stream)))


def vecmat(op: int, A, n: int, p_cols: int, x, z, ws: Workspace, stream=None, lda: int = 0) -> None:
    """z[i] = op_j f(A[i,j], x[j]); see matvec for `lda`."""
    w, wb = ws.for_(capi.PRIM_VECMAT, op, n, p_cols, stream=stream)
    check(_lib().forge_dev_vecmat_lda(op, _ptr(A), n, p_cols, lda, _ptr(x), _ptr(z), w, wb, _stream(stream)))


def fold(op: int, values, count: int, out, exclusive_upto: int = -1, has_out=None, stream=None) -> None:
    check(_lib().forge_dev_fold(op, _ptr(values), count, exclusive_upto, _ptr(out), _ptr(has_out),
                                _stream(stream)))


def copy(src, dst, nbytes: int, stream=None) -> None:
    check(_lib().forge_dev_copy(_ptr(src), _ptr(dst), nbytes, _stream(stream)))
