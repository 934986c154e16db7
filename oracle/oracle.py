"""ctypes front-end of the CPU oracle (oracle/oracle.c) and of the reference VM
compiled from /root/reference (oracle/_ref/libforge_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  Never imported by the
paper_2603_18695_b200 package.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "build" / "liboracle.so"
REF_SO = HERE / "_ref" / "libforge_ref.so"

_P = C.c_void_p
_u64 = C.c_uint64


def build_oracle(force: bool = False) -> Path:
    src = HERE / "oracle.c"
    if force or not ORACLE_SO.exists() or ORACLE_SO.stat().st_mtime < max(
            src.stat().st_mtime, (HERE / "oracle.h").stat().st_mtime):
        ORACLE_SO.parent.mkdir(exist_ok=True)
        subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-fopenmp", "-o", str(ORACLE_SO), str(src),
                        "-lm"],
                       check=True)
    return ORACLE_SO


_orc = None
_ref = None


def lib() -> C.CDLL:
    global _orc
    if _orc is None:
        if not ORACLE_SO.exists():
            build_oracle()
        L = C.CDLL(str(ORACLE_SO))
        L.orc_mix.restype = C.c_uint64
        L.orc_mix.argtypes = [C.c_uint64]
        L.orc_fill_synthetic.argtypes = [C.c_int, _P, _u64, _u64, _u64, C.c_int32]
        L.orc_float_components.argtypes = [C.c_int]
        L.orc_mapreduce.argtypes = [C.c_int, _P, _u64, _u64, _P, _P, _P]
        L.orc_scan.argtypes = [C.c_int, C.c_int32, _P, _u64, _P, _P, _P, _P]
        L.orc_matvec.argtypes = [C.c_int, _P, _u64, _u64, _P, _P, _P, _P]
        L.orc_vecmat.argtypes = [C.c_int, _P, _u64, _u64, _P, _P, _P, _P]
        L.orc_vload_pattern.argtypes = [_u64, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.orc_mapreduce_synthetic.argtypes = [C.c_int, _u64, _u64, C.c_int32, _P, _P, _P]
        L.orc_check_scan_synthetic_at.restype = C.c_int64
        L.orc_check_scan_synthetic_at.argtypes = [C.c_int, C.c_int32, _u64, C.c_int32, _P, _u64, _P, C.c_double,
                                                  C.POINTER(C.c_double)]
        L.orc_check_scan_synthetic.restype = C.c_int64
        L.orc_check_scan_synthetic.argtypes = [C.c_int, C.c_int32, _u64, _u64, C.c_int32, _P, C.c_double,
                                               C.POINTER(C.c_double)]
        L.orc_uf8_decode.restype = C.c_float
        L.orc_uf8_decode.argtypes = [C.c_uint8]
        L.orc_uf8_encode.restype = C.c_uint8
        L.orc_uf8_encode.argtypes = [C.c_float]
        _orc = L
    return _orc


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        L = C.CDLL(str(REF_SO))
        L.ref_last_error.restype = C.c_char_p
        L.ref_scan.argtypes = [C.c_int, C.c_int, _P, _u64, _P, C.c_int, _u64, C.POINTER(C.c_double)]
        L.ref_mapreduce.argtypes = [C.c_int, _P, _u64, _P, C.c_int, _u64, C.POINTER(C.c_double)]
        L.ref_mat.argtypes = [C.c_int, C.c_int, _P, _u64, _u64, _P, _P, C.c_int, _u64, C.POINTER(C.c_double)]
        L.ref_vcopy.argtypes = [_P, _P, _u64, C.c_uint32, C.c_uint32, C.c_int, C.POINTER(C.c_double)]
        L.ref_vload_pattern.argtypes = [_u64, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.ref_required_workspace.argtypes = [C.c_int, C.c_uint32, _u64, _u64, C.POINTER(_u64)]
        L.ref_scan_tiles.restype = C.c_uint64
        L.ref_scan_tiles.argtypes = [_u64]
        L.ref_error_probe.argtypes = [C.c_int]
        _ref = L
    return _ref


def _ptr(a) -> C.c_void_p:
    if a is None:
        return C.c_void_p(0)
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("oracle inputs must be C-contiguous (use np.ascontiguousarray)")
    return a.ctypes.data_as(C.c_void_p)


def _c(a):
    return None if a is None else np.ascontiguousarray(a)


# ---- dtype table (mirrors paper_2603_18695_b200.forge._TYPES, kept separate so
# the oracle never imports the product) ------------------------------------------
AFFINE = np.dtype([("a", "<f4"), ("b", "<f4")])
ARGMAX = np.dtype([("v", "<f4"), ("i", "<i4")])
MAT2 = np.dtype([("m", "<u4", (4,))])
QUAT = np.dtype([("w", "<f4"), ("x", "<f4"), ("y", "<f4"), ("z", "<f4")])
T_DTYPES = {0: np.float32, 1: np.float32, 2: np.float32, 3: np.float32, 4: np.float64, 5: np.int32,
            6: np.int32, 7: np.int32, 8: np.uint32, 9: np.int64, 10: AFFINE, 11: ARGMAX, 12: MAT2, 13: QUAT,
            14: np.uint8, 15: np.float32, 32: np.float32, 33: np.float32, 34: np.float32, 35: np.int32,
            36: np.float64, 37: MAT2}


def t_dtype(op):
    return np.dtype(T_DTYPES[op])


def s_dtype(op):
    return np.dtype(np.float32) if op == 14 else t_dtype(op)


def ncomp(op) -> int:
    return lib().orc_float_components(op)


def fill(op, n, seed, variant=0, index_base=0) -> np.ndarray:
    a = np.empty(n, dtype=t_dtype(op))
    lib().orc_fill_synthetic(op, _ptr(a), n, seed, index_base, variant)
    return a


def mapreduce(op, src: np.ndarray, stride: int = 1):
    """Returns (S value, exact[ncomp], scale[ncomp])."""
    src = _c(src)
    nc = max(ncomp(op), 1)
    out = np.zeros(1, dtype=s_dtype(op))
    ex, sc = np.zeros(nc), np.zeros(nc)
    n = (len(src) + stride - 1) // stride if stride > 1 else len(src)
    lib().orc_mapreduce(op, _ptr(src), n, stride, _ptr(out), _ptr(ex), _ptr(sc))
    return out[0], ex, sc


def mapreduce_synthetic(op, n, seed, variant=0):
    nc = max(ncomp(op), 1)
    out = np.zeros(1, dtype=s_dtype(op))
    ex, sc = np.zeros(nc), np.zeros(nc)
    lib().orc_mapreduce_synthetic(op, n, seed, variant, _ptr(out), _ptr(ex), _ptr(sc))
    return out[0], ex, sc


def scan(op, inclusive: bool, src: np.ndarray, carry=None):
    """Returns (dst S array, exact[n, ncomp], scale[n, ncomp])."""
    src = _c(src)
    n = len(src)
    nc = max(ncomp(op), 1)
    dst = np.zeros(n, dtype=s_dtype(op))
    ex, sc = np.zeros((n, nc)), np.zeros((n, nc))
    c = None
    if carry is not None:
        c = np.array([carry], dtype=s_dtype(op))
    lib().orc_scan(op, 1 if inclusive else 0, _ptr(src), n, _ptr(c), _ptr(dst), _ptr(ex), _ptr(sc))
    return dst, ex, sc


def matvec(op, A: np.ndarray, n, p, x=None):
    A, x = _c(A), _c(x)
    nc = max(ncomp(op), 1)
    y = np.zeros(p, dtype=s_dtype(op))
    ex, sc = np.zeros((p, nc)), np.zeros((p, nc))
    lib().orc_matvec(op, _ptr(A), n, p, _ptr(x), _ptr(y), _ptr(ex), _ptr(sc))
    return y, ex, sc


def vecmat(op, A: np.ndarray, n, p, x=None):
    A, x = _c(A), _c(x)
    nc = max(ncomp(op), 1)
    z = np.zeros(n, dtype=s_dtype(op))
    ex, sc = np.zeros((n, nc)), np.zeros((n, nc))
    lib().orc_vecmat(op, _ptr(A), n, p, _ptr(x), _ptr(z), _ptr(ex), _ptr(sc))
    return z, ex, sc


def vload_pattern(offset, nitem):
    segs = (C.c_uint32 * 16)()
    cnt = C.c_uint32()
    rc = lib().orc_vload_pattern(offset, nitem, segs, C.byref(cnt))
    if rc:
        return rc
    return [segs[i] for i in range(cnt.value)]


def check_scan_synthetic(op, inclusive, n, seed, got: np.ndarray, tol: float, variant=0):
    got = _c(got)
    worst = C.c_double()
    bad = lib().orc_check_scan_synthetic(op, 1 if inclusive else 0, n, seed, variant, _ptr(got), tol,
                                         C.byref(worst))
    return int(bad), worst.value


def check_scan_synthetic_at(op, inclusive, seed, idx: np.ndarray, got_at: np.ndarray, tol: float, variant=0):
    """Streaming check of scan outputs at ascending positions `idx` only."""
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    assert np.all(np.diff(idx.astype(np.int64)) > 0), "positions must be strictly ascending"
    got_at = _c(got_at)
    worst = C.c_double()
    bad = lib().orc_check_scan_synthetic_at(op, 1 if inclusive else 0, seed, variant, _ptr(idx), len(idx),
                                            _ptr(got_at), tol, C.byref(worst))
    return int(bad), worst.value


def float_view(op, arr: np.ndarray) -> np.ndarray:
    """Float components of S values as an (n, ncomp) float64 array."""
    a = np.atleast_1d(arr)
    if a.dtype.names:
        return np.stack([a[f].astype(np.float64) for f in a.dtype.names], axis=-1)
    return a.astype(np.float64).reshape(-1, 1)


def within(op, got: np.ndarray, exact: np.ndarray, scale: np.ndarray, tol: float) -> tuple[bool, float]:
    """|got - exact| <= tol * scale component-wise (SURVEY.md §8(c) parity rule)."""
    g = float_view(op, got)
    e = exact.reshape(g.shape)
    with np.errstate(invalid="ignore"):
        err = np.where(g == e, 0.0, np.abs(g - e))  # equal infinities (identities) are exact
    sc = scale.reshape(g.shape)
    ok = np.all(err <= tol * sc) and np.all(np.isfinite(g) == np.isfinite(exact.reshape(g.shape)))
    rel = float(np.max(np.where(sc > 0, err / np.where(sc > 0, sc, 1), np.where(err > 0, np.inf, 0)))) if g.size else 0.0
    return bool(ok), rel


# ---- the reference VM --------------------------------------------------------------

SIM, THREADS = 0, 1


def _ref_check(rc):
    if rc:
        raise RuntimeError(f"reference VM status {rc}: {ref().ref_last_error().decode()}")


def ref_scan(op, inclusive, src: np.ndarray, backend=THREADS, seed=0):
    dst = np.zeros(len(src), dtype=s_dtype(op))
    w = C.c_double()
    _ref_check(ref().ref_scan(op, 1 if inclusive else 0, _ptr(src), len(src), _ptr(dst), backend, seed,
                              C.byref(w)))
    return dst, w.value


def ref_mapreduce(op, src: np.ndarray, backend=THREADS, seed=0):
    out = np.zeros(1, dtype=s_dtype(op))
    w = C.c_double()
    _ref_check(ref().ref_mapreduce(op, _ptr(src), len(src), _ptr(out), backend, seed, C.byref(w)))
    return out[0], w.value


def ref_matvec(op, A, n, p, x=None, backend=THREADS, seed=0):
    out = np.zeros(p, dtype=s_dtype(op))
    w = C.c_double()
    _ref_check(ref().ref_mat(0, op, _ptr(A), n, p, _ptr(x), _ptr(out), backend, seed, C.byref(w)))
    return out, w.value


def ref_vecmat(op, A, n, p, x=None, backend=THREADS, seed=0):
    out = np.zeros(n, dtype=s_dtype(op))
    w = C.c_double()
    _ref_check(ref().ref_mat(1, op, _ptr(A), n, p, _ptr(x), _ptr(out), backend, seed, C.byref(w)))
    return out, w.value


def ref_vload_pattern(offset, nitem):
    segs = (C.c_uint32 * 16)()
    cnt = C.c_uint32()
    rc = ref().ref_vload_pattern(offset, nitem, segs, C.byref(cnt))
    if rc:
        return rc
    return [segs[i] for i in range(cnt.value)]
