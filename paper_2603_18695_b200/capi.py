"""ctypes declarations of include/forge.h (the C-ABI of libforge.so).

This is the reference-side binding a maintainer would add:
every struct and entry point mirrors include/forge.h one to one.  The shared
library is loaded from the package directory (built in-tree by
`make -C paper_2603_18695_b200/csrc`); a missing library is an ImportError —
there is no fallback implementation.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# FORGE_LIB=dev selects libforge_dev.so (`make DEV=1`: the same kernels plus the
# environment-read development knobs); the product is libforge.so.
_lib_env = os.environ.get("FORGE_LIB", "")
LIB_PATH = Path(__file__).resolve().parent / ("libforge_dev.so" if _lib_env == "dev"
                                              else _lib_env if _lib_env.endswith(".so") else "libforge.so")

# ---- status codes (forge_status) ------------------------------------------
OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_INVALID_DESCRIPTOR = 2
ERR_INVALID_NITEM = 3
ERR_MISSING_IDENTITY = 4
ERR_WORKSPACE_TOO_SMALL = 5
ERR_DIMENSION_MISMATCH = 6
ERR_PARSE_ERROR = 7
ERR_UNSUPPORTED = 8
ERR_DEVICE_FAULT = 100
ERR_NO_DEVICE = 101

STATUS_NAMES = {
    ERR_INVALID_ARGUMENT: "InvalidArgument",
    ERR_INVALID_DESCRIPTOR: "InvalidDescriptor",
    ERR_INVALID_NITEM: "InvalidNitem",
    ERR_MISSING_IDENTITY: "MissingIdentity",
    ERR_WORKSPACE_TOO_SMALL: "WorkspaceTooSmall",
    ERR_DIMENSION_MISMATCH: "DimensionMismatch",
    ERR_PARSE_ERROR: "ParseError",
    ERR_UNSUPPORTED: "Unsupported",
    ERR_DEVICE_FAULT: "DeviceFault",
    ERR_NO_DEVICE: "NoDevice",
}

# ---- forge_op ---------------------------------------------------------------
F32_SUM, F32_SUMSQ, F32_MAX, F32_MIN, F64_SUM = 0, 1, 2, 3, 4
I32_SUM, I32_MAX, I32_MIN, U32_SUM, I64_SUM = 5, 6, 7, 8, 9
AFFINE_F32, ARGMAX_F32I32, MAT2_U32, QUAT_F32, UF8_F32_SUM, F32_LOGSUMEXP = 10, 11, 12, 13, 14, 15
MV_F32_PLUS_TIMES, MV_F32_MIN_PLUS, MV_F32_MAX_PLUS = 32, 33, 34
MV_I32_PLUS_TIMES, MV_F64_PLUS_TIMES, MV_MAT2_U32 = 35, 36, 37

OPS_1D = list(range(16))
OPS_2D = list(range(32, 38))

# ---- forge_primitive / axis -------------------------------------------------
PRIM_SCAN, PRIM_MAPREDUCE, PRIM_MATVEC, PRIM_VECMAT, PRIM_VCOPY, PRIM_MAPREDUCE_2D = range(6)
AXIS_ROWS, AXIS_COLS = 0, 1


class OpInfo(C.Structure):
    _fields_ = [("t_size", C.c_uint32), ("s_size", C.c_uint32), ("commutative", C.c_uint32),
                ("binary", C.c_uint32), ("name", C.c_char_p)]


class Semiring(C.Structure):
    _fields_ = [("op", C.c_int), ("has_identity", C.c_int32)]


class ArchParams(C.Structure):
    _fields_ = [("warp_width", C.c_uint32), ("mapreduce_blocks", C.c_uint32),
                ("threads_per_block", C.c_uint32), ("nitem_scan", C.c_uint32),
                ("nitem_copy", C.c_uint32), ("lookback_window", C.c_uint32),
                ("matvec_wide_warp_cols", C.c_uint32), ("matvec_wide_block_threads", C.c_uint32),
                ("matvec_wide_min_outputs", C.c_uint64)]


class View(C.Structure):
    _fields_ = [("buf", C.c_int32), ("offset", C.c_uint64), ("length", C.c_uint64),
                ("stride", C.c_uint64)]


class Workspace(C.Structure):
    _fields_ = [("tile_aggregate", C.c_int32), ("tile_prefix", C.c_int32), ("tile_flag", C.c_int32),
                ("partials", C.c_int32), ("flags", C.c_int32), ("result", C.c_int32),
                ("tiles", C.c_uint64), ("slots", C.c_uint64)]


class LaunchReport(C.Structure):
    _fields_ = [("ok", C.c_int32), ("fault_kind", C.c_int32), ("steps", C.c_uint64),
                ("wall_seconds", C.c_double), ("detail", C.c_char * 240)]


# name -> (restype, argtypes); exactly the declarations of include/forge.h
_P = C.c_void_p
_u32, _u64, _i32 = C.c_uint32, C.c_uint64, C.c_int32
class LitmusResult(C.Structure):
    """forge_litmus_result (include/forge.h)."""
    _fields_ = [("seeds_run", C.c_uint64), ("assert_violations", C.c_uint64), ("faults", C.c_uint64),
                ("distinct_outcomes", C.c_uint64)]


_SIGNATURES = {
    "forge_last_error": (C.c_char_p, []),
    "forge_abi_version": (C.c_int, []),
    "forge_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "forge_get_op_info": (C.c_int, [C.c_int, C.POINTER(OpInfo)]),
    "forge_arch_params_default": (None, [C.POINTER(ArchParams)]),
    "forge_machine_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "forge_machine_destroy": (C.c_int, [_P]),
    "forge_machine_stream": (C.c_int, [_P, C.POINTER(_P)]),
    "forge_machine_synchronize": (C.c_int, [_P]),
    "forge_create_buffer": (C.c_int, [_P, C.c_char_p, _u64, _u32, C.POINTER(_i32)]),
    "forge_destroy_buffer": (C.c_int, [_P, _i32]),
    "forge_buffer_length": (C.c_int, [_P, _i32, C.POINTER(_u64)]),
    "forge_buffer_elem_size": (C.c_int, [_P, _i32, C.POINTER(_u32)]),
    "forge_buffer_alignment": (C.c_int, [_P, _i32, C.POINTER(_u32)]),
    "forge_buffer_device_ptr": (C.c_int, [_P, _i32, C.POINTER(_P)]),
    "forge_write_bytes": (C.c_int, [_P, _i32, _u64, _P, _u64]),
    "forge_read_bytes": (C.c_int, [_P, _i32, _u64, _P, _u64]),
    "forge_fill_zero": (C.c_int, [_P, _i32]),
    "forge_descriptor_info": (C.c_int, [C.c_char_p, C.POINTER(_u32), C.POINTER(_u32), C.c_char_p, _u64]),
    "forge_value_bytes_equal": (C.c_int, [C.c_char_p, _P, _P, C.POINTER(_i32)]),
    "forge_required_workspace": (C.c_int, [C.c_int, _u32, _u64, _u64, C.POINTER(ArchParams), C.POINTER(_u64)]),
    "forge_make_scan_workspace": (C.c_int, [_P, C.c_int, _u64, C.POINTER(ArchParams), C.POINTER(Workspace)]),
    "forge_make_mapreduce_workspace": (C.c_int, [_P, C.c_int, C.POINTER(ArchParams), C.POINTER(Workspace)]),
    "forge_make_mat_workspace": (C.c_int, [_P, C.c_int, _u64, _u64, C.POINTER(ArchParams), C.POINTER(Workspace)]),
    "forge_workspace_release": (C.c_int, [_P, C.POINTER(Workspace)]),
    "forge_scan": (C.c_int, [_P, Semiring, View, View, _i32, C.POINTER(Workspace), C.POINTER(ArchParams),
                             C.POINTER(LaunchReport)]),
    "forge_mapreduce": (C.c_int, [_P, Semiring, View, C.POINTER(Workspace), C.POINTER(ArchParams), _P,
                                  C.POINTER(LaunchReport)]),
    "forge_matvec": (C.c_int, [_P, Semiring, View, _u64, _u64, View, View, C.POINTER(Workspace),
                               C.POINTER(ArchParams), C.POINTER(LaunchReport), _i32]),
    "forge_vecmat": (C.c_int, [_P, Semiring, View, _u64, _u64, View, View, C.POINTER(Workspace),
                               C.POINTER(ArchParams), C.POINTER(LaunchReport), _i32]),
    "forge_mapreduce_2d": (C.c_int, [_P, Semiring, View, _u64, _u64, C.c_int, View, C.POINTER(Workspace),
                                     C.POINTER(ArchParams), C.POINTER(LaunchReport)]),
    "forge_vcopy": (C.c_int, [_P, View, View, _u32, C.POINTER(ArchParams), C.POINTER(LaunchReport)]),
    "forge_set_mutation_flags": (C.c_int, [_i32, _i32]),
    "forge_set_schedule_perturbation": (C.c_int, [_u64, _u32]),
    "forge_vload_pattern": (C.c_int, [_u64, _u32, C.POINTER(_u32), C.POINTER(_u32)]),
    "forge_litmus_parse": (C.c_int, [C.c_char_p]),
    "forge_litmus_run": (C.c_int, [C.c_char_p, _u64, _u64, C.POINTER(LitmusResult), C.c_char_p, _u64]),
    "forge_dev_workspace_bytes": (C.c_int, [C.c_int, C.c_int, _u64, _u64, C.POINTER(_u64)]),
    "forge_dev_mapreduce": (C.c_int, [C.c_int, _P, _u64, _P, _P, _u64, _P]),
    "forge_dev_reduce_ordered": (C.c_int, [C.c_int, _P, _u64, _P, _P, _u64, _P]),
    "forge_dev_scan": (C.c_int, [C.c_int, _i32, _P, _P, _u64, _P, _P, _P, _u64, _P]),
    "forge_dev_matvec": (C.c_int, [C.c_int, _P, _u64, _u64, _P, _P, _P, _u64, _P]),
    "forge_dev_vecmat": (C.c_int, [C.c_int, _P, _u64, _u64, _P, _P, _P, _u64, _P]),
    "forge_dev_matvec_lda": (C.c_int, [C.c_int, _P, _u64, _u64, _u64, _P, _P, _P, _u64, _P]),
    "forge_dev_vecmat_lda": (C.c_int, [C.c_int, _P, _u64, _u64, _u64, _P, _P, _P, _u64, _P]),
    "forge_dev_fold": (C.c_int, [C.c_int, _P, _u32, _i32, _P, _P, _P]),
    "forge_dev_copy": (C.c_int, [_P, _P, _u64, _P]),
    "forge_dev_fill_synthetic": (C.c_int, [C.c_int, _P, _u64, _u64, _u64, _i32, _P]),
    # single-process multi-GPU groups (group.cu)
    "forge_shard_range": (C.c_int, [_u64, _i32, _i32, C.POINTER(_u64), C.POINTER(_u64)]),
    "forge_group_create": (C.c_int, [C.POINTER(_i32), _i32, C.POINTER(_P)]),
    "forge_group_destroy": (C.c_int, [_P]),
    "forge_group_size": (C.c_int, [_P, C.POINTER(_i32), C.POINTER(_i32)]),
    "forge_group_stream": (C.c_int, [_P, _i32, C.POINTER(_P)]),
    "forge_group_synchronize": (C.c_int, [_P]),
    "forge_sharded_mapreduce": (C.c_int, [_P, C.c_int, C.POINTER(_P), C.POINTER(_u64), C.POINTER(_P),
                                          C.POINTER(_u64), _P]),
    "forge_sharded_result_dev": (C.c_int, [_P, _i32, C.POINTER(_P)]),
    "forge_sharded_scan": (C.c_int, [_P, C.c_int, _i32, C.POINTER(_P), C.POINTER(_P), C.POINTER(_u64),
                                     C.POINTER(_P), C.POINTER(_u64)]),
    "forge_sharded_matvec": (C.c_int, [_P, C.c_int, C.POINTER(_P), _u64, _u64, C.POINTER(_P), C.POINTER(_P),
                                       C.POINTER(_P), C.POINTER(_u64)]),
    "forge_sharded_vecmat": (C.c_int, [_P, C.c_int, C.POINTER(_P), _u64, _u64, C.POINTER(_P), C.POINTER(_P),
                                       C.POINTER(_P), C.POINTER(_u64)]),
    "forge_cyclic_chunk_quantum": (C.c_int, [C.c_int, C.POINTER(_u64)]),
    "forge_cyclic_local_n": (C.c_int, [_u64, _u64, _i32, _i32, C.POINTER(_u64)]),
    "forge_cyclic_workspace_bytes": (C.c_int, [C.c_int, _u64, C.POINTER(_u64)]),
    "forge_sharded_scan_cyclic": (C.c_int, [_P, C.c_int, _i32, C.POINTER(_P), C.POINTER(_P), _u64, _u64,
                                            C.POINTER(_P), C.POINTER(_u64)]),
}

_lib: C.CDLL | None = None


def load(path: str | os.PathLike | None = None) -> C.CDLL:
    """Loads libforge.so and declares every entry point.  Raises ImportError
    if the library was not built — the product never falls back."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(f"libforge.so not found at {p}; build it with "
                          f"`make -C paper_2603_18695_b200/csrc` (no CPU fallback exists)")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGNATURES.items():
        if _lib_env.endswith(".so") and not hasattr(lib, name):
            continue  # FORGE_LIB=<other build>.so: development comparisons against older builds
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.forge_abi_version() != 1:
        raise ImportError("libforge.so ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)
