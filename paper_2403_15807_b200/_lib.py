"""ctypes binding of libvrs.so (include/vrs.h) -- argument marshalling only.

Every step of the search runs in the CUDA kernels of libvrs; this module only
turns torch tensors into pointers and status codes into exceptions.  There is
no fallback: if the shared library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvrs.so")
if os.environ.get("VRS_LIB"):   # experiment builds of the same sources (csrc/Makefile `exp`): libvrs_<VRS_LIB>.so
    LIB_PATH = os.path.join(_HERE, "libvrs_%s.so" % os.environ["VRS_LIB"])

OK, EINVAL, ENOTFOUND, EDEGENERATE, ENOMEM, ECUDA, ECOMM, EUNSUPPORTED, ERANGE = range(9)
STATUS_NAMES = ["VRS_OK", "VRS_EINVAL", "VRS_ENOTFOUND", "VRS_EDEGENERATE", "VRS_ENOMEM", "VRS_ECUDA",
                "VRS_ECOMM", "VRS_EUNSUPPORTED", "VRS_ERANGE"]
L2, IP, COSINE = 0, 1, 2
ATTR_I32, ATTR_U8 = 0, 1
PATH_AUTO, PATH_SCAN, PATH_GEMM = 0, 1, 2
ROWS_AUTO, ROWS_GATHER, ROWS_MASKED = 0, 1, 2
PREC_DEFAULT, PREC_TF32, PREC_BF16, PREC_FP16 = 0, 1, 2, 3
K_MAX = 240
MAX_CLAUSES = 8

# every symbol include/vrs.h declares (tests check the library exports them)
EXPORTS = ("vrs_load", "vrs_load_ex", "vrs_search", "vrs_range_search", "vrs_search_ex", "vrs_search_host", "vrs_host_fence", "vrs_select", "vrs_merge", "vrs_free",
           "vrs_merge_push", "vrs_push_buffer_bytes", "vrs_last_error", "vrs_last_path", "vrs_last_precision", "vrs_index_precision", "vrs_last_launches", "vrs_index_rows", "vrs_index_dim",
           "vrs_profile_enable", "vrs_profile_read", "vrs_profile_reset", "vrs_pool_reserved_bytes")


class VrsError(RuntimeError):
    def __init__(self, status: int, call: str, msg: str):
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{call} -> {name}: {msg}")
        self.status = status


class Attr(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("data", ctypes.c_void_p)]


class Clause(ctypes.Structure):
    _fields_ = [("attr", ctypes.c_int32), ("lo", ctypes.c_int64), ("hi", ctypes.c_int64)]


class Predicate(ctypes.Structure):
    _fields_ = [("n_clauses", ctypes.c_int32), ("clauses", ctypes.POINTER(Clause))]


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class Allocator(ctypes.Structure):
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("ctx", ctypes.c_void_p)]


class SearchOptions(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int32), ("rows", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("host_async", ctypes.c_int32), ("reserved0", ctypes.c_int32), ("stats", ctypes.c_void_p),
                ("reserved", ctypes.c_int32 * 2)]


class LoadOptions(ctypes.Structure):
    _fields_ = [("precision", ctypes.c_int32), ("reserved", ctypes.c_int32 * 7)]


_lib = None


def load_library():
    """Load libvrs.so (built by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (there is no non-CUDA fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    p, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.vrs_load.argtypes = [p, i64, i32, p, i32, i64, p, p, ctypes.POINTER(p)]
    lib.vrs_load_ex.argtypes = [p, i64, i32, p, i32, i64, p, p, p, ctypes.POINTER(p)]
    lib.vrs_search.argtypes = [p, p, i64, i32, p, i32, ctypes.c_int, p, p, p]
    lib.vrs_search_ex.argtypes = [p, p, i64, i32, p, i32, ctypes.c_int, p, p, p, p]
    lib.vrs_search_host.argtypes = [p, p, i64, i32, p, i32, ctypes.c_int, p, p, p, p]
    lib.vrs_range_search.argtypes = [p, p, i64, i32, p, ctypes.c_double, ctypes.c_int, i64, p, p, p,
                                     ctypes.POINTER(i64), p, p]
    lib.vrs_host_fence.argtypes = [p, p]
    lib.vrs_select.argtypes = [p, p, p, p, p, p]
    lib.vrs_merge.argtypes = [p, p, i32, i64, i32, ctypes.c_int, p, p, p]
    lib.vrs_merge_push.argtypes = [p, p, p, i64, i32, i32, i64, i32, ctypes.c_int, p, p, p, p]
    lib.vrs_merge_push.restype = ctypes.c_int
    lib.vrs_push_buffer_bytes.argtypes = [i32, i64, i32]
    lib.vrs_push_buffer_bytes.restype = i64
    lib.vrs_free.argtypes = [p]
    for f in ("vrs_load", "vrs_load_ex", "vrs_search", "vrs_range_search", "vrs_search_ex", "vrs_search_host", "vrs_host_fence",
              "vrs_select", "vrs_merge", "vrs_free"):
        getattr(lib, f).restype = ctypes.c_int
    lib.vrs_last_error.restype = ctypes.c_char_p
    lib.vrs_last_path.restype = i32
    lib.vrs_last_precision.restype = i32
    lib.vrs_index_precision.argtypes = [p]
    lib.vrs_index_precision.restype = i32
    lib.vrs_last_launches.restype = i32
    lib.vrs_index_rows.argtypes = [p]
    lib.vrs_index_rows.restype = i64
    lib.vrs_index_dim.argtypes = [p]
    lib.vrs_index_dim.restype = i32
    lib.vrs_profile_enable.argtypes = [i32]
    lib.vrs_profile_enable.restype = None
    lib.vrs_profile_reset.restype = None
    lib.vrs_profile_read.argtypes = [i32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(i64)]
    lib.vrs_profile_read.restype = i32
    lib.vrs_pool_reserved_bytes.restype = i64
    _lib = lib
    return lib


def check(status: int, call: str):
    if status != OK:
        msg = _lib.vrs_last_error().decode(errors="replace") if _lib else ""
        raise VrsError(status, call, msg)


_pred_cache = {}


def make_predicate(clauses):
    """[(attr, lo, hi), ...] -> (Predicate, keepalive); cached per clause tuple."""
    try:
        key = tuple((int(a), int(lo), int(hi)) for a, lo, hi in (clauses or []))
    except (TypeError, ValueError):
        key = None
    if key is not None and key in _pred_cache:
        return _pred_cache[key]
    clauses = list(clauses or [])
    arr = (Clause * max(len(clauses), 1))()
    for i, (a, lo, hi) in enumerate(clauses):
        arr[i].attr, arr[i].lo, arr[i].hi = int(a), int(lo), int(hi)
    pred = Predicate(len(clauses), ctypes.cast(arr, ctypes.POINTER(Clause)))
    if key is not None and len(_pred_cache) < 1024:
        _pred_cache[key] = (pred, arr)
    return pred, arr
