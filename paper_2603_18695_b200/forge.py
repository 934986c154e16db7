"""Python mirror of the reference primitive API over the C-ABI.

Reads like /root/reference/proj/include/forge/{machine,intrinsics,primitives}.hpp:
    m = Machine()
    a = create_buffer(m, F32_SUM, n); m.write(a, x)
    ws = make_scan_workspace(m, F32_SUM, n)
    rep = scan(m, make_semiring(F32_SUM), make_view(m, a), make_view(m, b), True, ws, ArchParams())
Errors raise ForgeError whose `.name` is the reference ErrorCode name
(error.hpp:10-19); device faults come back as LaunchReport(ok=False) plus a
ForgeError("DeviceFault") — the same split as the reference (error.hpp:8-9).
Every call goes through libforge.so's sm_100a kernels; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import capi
from .capi import (AFFINE_F32, ARGMAX_F32I32, F32_LOGSUMEXP, F32_MAX, F32_MIN, F32_SUM, F32_SUMSQ,  # noqa: F401
                   F64_SUM, I32_MAX, I32_MIN, I32_SUM, I64_SUM, MAT2_U32, MV_F32_MAX_PLUS,
                   MV_F32_MIN_PLUS, MV_F32_PLUS_TIMES, MV_F64_PLUS_TIMES, MV_I32_PLUS_TIMES,
                   MV_MAT2_U32, QUAT_F32, U32_SUM, UF8_F32_SUM)

AFFINE_DTYPE = np.dtype([("a", "<f4"), ("b", "<f4")])
ARGMAX_DTYPE = np.dtype([("v", "<f4"), ("i", "<i4")])
MAT2_DTYPE = np.dtype([("m", "<u4", (4,))])
QUAT_DTYPE = np.dtype([("w", "<f4"), ("x", "<f4"), ("y", "<f4"), ("z", "<f4")])

# op -> (T dtype, S dtype, T descriptor, S descriptor)
_TYPES = {
    F32_SUM: (np.float32, np.float32, "f32", "f32"),
    F32_SUMSQ: (np.float32, np.float32, "f32", "f32"),
    F32_MAX: (np.float32, np.float32, "f32", "f32"),
    F32_MIN: (np.float32, np.float32, "f32", "f32"),
    F64_SUM: (np.float64, np.float64, "f64", "f64"),
    I32_SUM: (np.int32, np.int32, "u32", "u32"),
    I32_MAX: (np.int32, np.int32, "u32", "u32"),
    I32_MIN: (np.int32, np.int32, "u32", "u32"),
    U32_SUM: (np.uint32, np.uint32, "u32", "u32"),
    I64_SUM: (np.int64, np.int64, "u64", "u64"),
    AFFINE_F32: (AFFINE_DTYPE, AFFINE_DTYPE, "tuple(f32,f32)", "tuple(f32,f32)"),
    ARGMAX_F32I32: (ARGMAX_DTYPE, ARGMAX_DTYPE, "tuple(f32,u32)", "tuple(f32,u32)"),
    MAT2_U32: (MAT2_DTYPE, MAT2_DTYPE, "tuple(u32,u32,u32,u32)", "tuple(u32,u32,u32,u32)"),
    QUAT_F32: (QUAT_DTYPE, QUAT_DTYPE, "tuple(f32,f32,f32,f32)", "tuple(f32,f32,f32,f32)"),
    UF8_F32_SUM: (np.uint8, np.float32, "u8", "f32"),
    F32_LOGSUMEXP: (np.float32, np.float32, "f32", "f32"),
    MV_F32_PLUS_TIMES: (np.float32, np.float32, "f32", "f32"),
    MV_F32_MIN_PLUS: (np.float32, np.float32, "f32", "f32"),
    MV_F32_MAX_PLUS: (np.float32, np.float32, "f32", "f32"),
    MV_I32_PLUS_TIMES: (np.int32, np.int32, "u32", "u32"),
    MV_F64_PLUS_TIMES: (np.float64, np.float64, "f64", "f64"),
    MV_MAT2_U32: (MAT2_DTYPE, MAT2_DTYPE, "tuple(u32,u32,u32,u32)", "tuple(u32,u32,u32,u32)"),
}


def t_dtype(op: int) -> np.dtype:
    return np.dtype(_TYPES[op][0])


def s_dtype(op: int) -> np.dtype:
    return np.dtype(_TYPES[op][1])


def t_descriptor(op: int) -> str:
    return _TYPES[op][2]


def s_descriptor(op: int) -> str:
    return _TYPES[op][3]


class ForgeError(RuntimeError):
    """Host-side error; `.name` is the reference ErrorCode name."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.name = capi.STATUS_NAMES.get(status, f"status{status}")
        super().__init__(f"{self.name}: {message}")


def _lib():
    return capi.load()


def check(rc: int) -> None:
    if rc != capi.OK:
        raise ForgeError(rc, _lib().forge_last_error().decode(errors="replace"))


# ---- reference value types ---------------------------------------------------

def ArchParams(**overrides) -> capi.ArchParams:  # noqa: N802 (mirrors the C++ type name)
    p = capi.ArchParams()
    _lib().forge_arch_params_default(C.byref(p))
    for k, v in overrides.items():
        setattr(p, k, v)
    return p


def View(buf: int, offset: int = 0, length: int = 0, stride: int = 1) -> capi.View:  # noqa: N802
    return capi.View(buf, offset, length, stride)


def subview(v: capi.View, first: int, count: int) -> capi.View:
    return capi.View(v.buf, v.offset + first * v.stride, count, v.stride)


def strided(v: capi.View, first: int, count: int, step: int) -> capi.View:
    return capi.View(v.buf, v.offset + first * v.stride, count, v.stride * step)


def make_semiring(op: int, identity: bool = True) -> capi.Semiring:
    """SemiringSpec for a menu op; identity=False drops the identity (nullopt)."""
    return capi.Semiring(op, 1 if identity else 0)


@dataclass
class LaunchReport:
    ok: bool
    fault_kind: int
    steps: int
    wall_seconds: float
    detail: str


def _report(r: capi.LaunchReport) -> LaunchReport:
    return LaunchReport(bool(r.ok), int(r.fault_kind), int(r.steps), float(r.wall_seconds),
                        bytes(r.detail).split(b"\0", 1)[0].decode(errors="replace"))


def op_info(op: int) -> dict:
    info = capi.OpInfo()
    check(_lib().forge_get_op_info(op, C.byref(info)))
    return {"t_size": info.t_size, "s_size": info.s_size, "commutative": bool(info.commutative),
            "binary": bool(info.binary), "name": info.name.decode()}


# ---- Machine (machine.hpp:142-184) -------------------------------------------

class Machine:
    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(_lib().forge_machine_create(device, C.byref(h)))
        self._h = h

    @property
    def handle(self) -> C.c_void_p:
        if self._h is None:
            raise ForgeError(capi.ERR_INVALID_ARGUMENT, "machine is closed")
        return self._h

    def close(self) -> None:
        if self._h is not None:
            _lib().forge_machine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def stream(self) -> int:
        s = C.c_void_p()
        check(_lib().forge_machine_stream(self.handle, C.byref(s)))
        return s.value or 0

    def synchronize(self) -> None:
        check(_lib().forge_machine_synchronize(self.handle))

    def create_buffer(self, descriptor: str, length: int, base_alignment: int = 0) -> int:
        out = C.c_int32()
        check(_lib().forge_create_buffer(self.handle, descriptor.encode(), length, base_alignment,
                                         C.byref(out)))
        return out.value

    def destroy_buffer(self, buf: int) -> None:
        check(_lib().forge_destroy_buffer(self.handle, buf))

    def buffer_length(self, buf: int) -> int:
        v = C.c_uint64()
        check(_lib().forge_buffer_length(self.handle, buf, C.byref(v)))
        return v.value

    def buffer_elem_size(self, buf: int) -> int:
        v = C.c_uint32()
        check(_lib().forge_buffer_elem_size(self.handle, buf, C.byref(v)))
        return v.value

    def buffer_alignment(self, buf: int) -> int:
        v = C.c_uint32()
        check(_lib().forge_buffer_alignment(self.handle, buf, C.byref(v)))
        return v.value

    def device_ptr(self, buf: int) -> int:
        v = C.c_void_p()
        check(_lib().forge_buffer_device_ptr(self.handle, buf, C.byref(v)))
        return v.value or 0

    def write(self, buf: int, values: np.ndarray, elem_offset: int = 0) -> None:
        a = np.ascontiguousarray(values)
        check(_lib().forge_write_bytes(self.handle, buf, elem_offset, a.ctypes.data_as(C.c_void_p),
                                       a.nbytes))

    def write_ptr(self, buf: int, host_ptr: int, nbytes: int, elem_offset: int = 0) -> None:
        check(_lib().forge_write_bytes(self.handle, buf, elem_offset, C.c_void_p(host_ptr), nbytes))

    def read(self, buf: int, count: int, dtype, elem_offset: int = 0) -> np.ndarray:
        out = np.empty(count, dtype=dtype)
        check(_lib().forge_read_bytes(self.handle, buf, elem_offset, out.ctypes.data_as(C.c_void_p),
                                      out.nbytes))
        return out

    def read_ptr(self, buf: int, host_ptr: int, nbytes: int, elem_offset: int = 0) -> None:
        """forge_read_bytes into caller host memory (e.g. a pinned buffer)."""
        check(_lib().forge_read_bytes(self.handle, buf, elem_offset, C.c_void_p(host_ptr), nbytes))

    def fill_zero(self, buf: int) -> None:
        check(_lib().forge_fill_zero(self.handle, buf))


def create_buffer(m: Machine, op_or_descriptor, length: int, base_alignment: int = 0,
                  which: str = "T") -> int:
    """intr::create_buffer: by descriptor literal, or by a menu op's T / S type."""
    if isinstance(op_or_descriptor, str):
        desc = op_or_descriptor
    else:
        desc = t_descriptor(op_or_descriptor) if which == "T" else s_descriptor(op_or_descriptor)
    return m.create_buffer(desc, length, base_alignment)


def make_view(m: Machine, buf: int) -> capi.View:
    return capi.View(buf, 0, m.buffer_length(buf), 1)


# ---- workspaces (primitives.hpp:246-300) ---------------------------------------

def required_workspace(prim: int, accum_size: int, n: int, p_cols: int = 0, params=None) -> int:
    out = C.c_uint64()
    p = params or ArchParams()
    check(_lib().forge_required_workspace(prim, accum_size, n, p_cols, C.byref(p), C.byref(out)))
    return out.value


def make_scan_workspace(m: Machine, op: int, n: int, params=None) -> capi.Workspace:
    ws = capi.Workspace()
    p = params or ArchParams()
    check(_lib().forge_make_scan_workspace(m.handle, op, n, C.byref(p), C.byref(ws)))
    return ws


def make_mapreduce_workspace(m: Machine, op: int, params=None) -> capi.Workspace:
    ws = capi.Workspace()
    p = params or ArchParams()
    check(_lib().forge_make_mapreduce_workspace(m.handle, op, C.byref(p), C.byref(ws)))
    return ws


def make_mat_workspace(m: Machine, op: int, reduce_len: int, outputs: int, params=None) -> capi.Workspace:
    ws = capi.Workspace()
    p = params or ArchParams()
    check(_lib().forge_make_mat_workspace(m.handle, op, reduce_len, outputs, C.byref(p), C.byref(ws)))
    return ws


def release(m: Machine, ws: capi.Workspace) -> None:
    check(_lib().forge_workspace_release(m.handle, C.byref(ws)))


# ---- primitives ----------------------------------------------------------------

def _run(rc: int, rep: capi.LaunchReport) -> LaunchReport:
    r = _report(rep)
    check(rc)
    return r


def scan(m, spec, src, dst, inclusive: bool, ws, params=None) -> LaunchReport:
    rep = capi.LaunchReport()
    p = params or ArchParams()
    rc = _lib().forge_scan(m.handle, spec, src, dst, 1 if inclusive else 0, C.byref(ws), C.byref(p),
                           C.byref(rep))
    return _run(rc, rep)


def mapreduce(m, spec, src, ws, params=None):
    """Returns (value, LaunchReport); the value is one S element (numpy scalar/record)."""
    rep = capi.LaunchReport()
    p = params or ArchParams()
    out = np.zeros(1, dtype=s_dtype(spec.op))
    rc = _lib().forge_mapreduce(m.handle, spec, src, C.byref(ws), C.byref(p),
                                out.ctypes.data_as(C.c_void_p), C.byref(rep))
    r = _run(rc, rep)
    return out[0], r


def matvec(m, spec, A, n, p_cols, x, y, ws, params=None, uses_vector=True) -> LaunchReport:
    rep = capi.LaunchReport()
    p = params or ArchParams()
    rc = _lib().forge_matvec(m.handle, spec, A, n, p_cols, x, y, C.byref(ws), C.byref(p), C.byref(rep),
                             1 if uses_vector else 0)
    return _run(rc, rep)


def vecmat(m, spec, A, n, p_cols, x, z, ws, params=None, uses_vector=True) -> LaunchReport:
    rep = capi.LaunchReport()
    p = params or ArchParams()
    rc = _lib().forge_vecmat(m.handle, spec, A, n, p_cols, x, z, C.byref(ws), C.byref(p), C.byref(rep),
                             1 if uses_vector else 0)
    return _run(rc, rep)


ROWS, COLS = capi.AXIS_ROWS, capi.AXIS_COLS


def mapreduce_2d(m, spec, A, n, p_cols, axis, out, ws, params=None) -> LaunchReport:
    rep = capi.LaunchReport()
    p = params or ArchParams()
    rc = _lib().forge_mapreduce_2d(m.handle, spec, A, n, p_cols, axis, out, C.byref(ws), C.byref(p),
                                   C.byref(rep))
    return _run(rc, rep)


def vcopy(m, src, dst, nitem: int = 4, params=None) -> LaunchReport:
    rep = capi.LaunchReport()
    p = params or ArchParams()
    rc = _lib().forge_vcopy(m.handle, src, dst, nitem, C.byref(p), C.byref(rep))
    return _run(rc, rep)


def vload_pattern(offset: int, nitem: int) -> list[int]:
    segs = (C.c_uint32 * 16)()
    cnt = C.c_uint32()
    check(_lib().forge_vload_pattern(offset, nitem, segs, C.byref(cnt)))
    return [segs[i] for i in range(cnt.value)]


def descriptor_info(text: str) -> tuple[int, int, str]:
    size, align = C.c_uint32(), C.c_uint32()
    buf = C.create_string_buffer(512)
    check(_lib().forge_descriptor_info(text.encode(), C.byref(size), C.byref(align), buf, 512))
    return size.value, align.value, buf.value.decode()


def value_bytes_equal(text: str, a: bytes, b: bytes) -> bool:
    eq = C.c_int32()
    check(_lib().forge_value_bytes_equal(text.encode(), a, b, C.byref(eq)))
    return bool(eq.value)


def device_count() -> int:
    c = C.c_int()
    _lib().forge_device_count(C.byref(c))
    return c.value


# ---- litmus (forge::lit: reference proj/include/forge/litmus.hpp) -------------

def parse_litmus(text: str) -> None:
    """Validates a litmus program (reference parse_litmus, litmus.cpp:169-253);
    raises ForgeError("ParseError") with the offending line."""
    check(_lib().forge_litmus_parse(text.encode()))


def run_litmus(text: str, seed_begin: int, seed_end: int) -> dict:
    """Runs instances seed_begin .. seed_end-1 of the program on the GPU
    (reference run_litmus, litmus.cpp:283-350; here each block is a CTA on
    its own SM).  Returns seeds_run, assert_violations, faults and the
    histogram {outcome string: count}."""
    res = capi.LitmusResult()
    buf = C.create_string_buffer(1 << 16)
    check(_lib().forge_litmus_run(text.encode(), seed_begin, seed_end, C.byref(res), buf, len(buf)))
    hist = {}
    for line in buf.value.decode().splitlines():
        count, outcome = line.split("\t", 1)
        hist[outcome] = int(count)
    return {"seeds_run": res.seeds_run, "assert_violations": res.assert_violations, "faults": res.faults,
            "distinct_outcomes": res.distinct_outcomes, "histogram": hist}

