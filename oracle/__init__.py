"""CPU brute-force oracle for filtered exact top-k search -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product
(``paper_2403_15807_b200``) never imports it and shares no code with it.

The arithmetic lives in ``vrs_oracle.c`` (plain C, fp64, -ffp-contract=off);
this module only compiles it with gcc and marshals numpy arrays through ctypes.
Every function follows PAPER.md L285-L288 (Sec. 3, predicate pushdown
equation) and the readings R1-R5 listed in the C file header and DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "vrs_oracle.c")
_LIB = os.path.join(_HERE, "libvrs_oracle.so")

OK, EINVAL, ENOTFOUND, EDEGENERATE, ENOMEM = 0, 1, 2, 3, 4
ERANGE = 8
L2, IP, COS = 0, 1, 2
I32, U8 = 0, 1


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"oracle {what} failed with status {status}")
        self.status = status


class _Clause(ctypes.Structure):
    _fields_ = [("attr", ctypes.c_int32), ("lo", ctypes.c_int64), ("hi", ctypes.c_int64)]


def build(force: bool = False) -> str:
    """Compile the oracle shared library with gcc (-O2 -fopenmp -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c11",
             "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        p = ctypes.c_void_p
        lib.orc_select.argtypes = [p, p, ctypes.c_int32, ctypes.c_int64, p, ctypes.c_int32, p, p, p]
        lib.orc_search.argtypes = [p, ctypes.c_int64, ctypes.c_int32, p, p, ctypes.c_int32, p,
                                   ctypes.c_int32, p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                   ctypes.c_int64, p, p, p, ctypes.c_int32]
        lib.orc_score.argtypes = [p, ctypes.c_int32, p, p, ctypes.c_int64, ctypes.c_int32, p]
        lib.orc_range.argtypes = [p, ctypes.c_int64, ctypes.c_int32, p, p, ctypes.c_int32, p, ctypes.c_int32, p,
                                  ctypes.c_int64, ctypes.c_double, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                  p, p, p, p, ctypes.c_int32]
        lib.orc_merge.argtypes = [p, p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                  p, p]
        for f in ("orc_select", "orc_search", "orc_score", "orc_range", "orc_merge"):
            getattr(lib, f).restype = ctypes.c_int
        lib.orc_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _attrs(attrs):
    """attrs: list of numpy int32 / uint8 arrays -> (keepalive, ptr array, type array)."""
    cols = [np.ascontiguousarray(a) for a in attrs]
    types = []
    for a in cols:
        if a.dtype == np.int32:
            types.append(I32)
        elif a.dtype == np.uint8:
            types.append(U8)
        else:
            raise TypeError(f"attribute dtype {a.dtype} not supported (int32, uint8)")
    n = max(len(cols), 1)
    ptrs = (ctypes.c_void_p * n)(*[a.ctypes.data for a in cols]) if cols else (ctypes.c_void_p * 1)()
    tarr = np.asarray(types if types else [0], dtype=np.int32)
    return cols, ptrs, tarr


def _clauses(pred):
    """pred: list of (attr, lo, hi) -> ctypes array (or None)."""
    pred = list(pred or [])
    arr = (_Clause * max(len(pred), 1))()
    for i, (a, lo, hi) in enumerate(pred):
        arr[i].attr, arr[i].lo, arr[i].hi = int(a), int(lo), int(hi)
    return arr, len(pred)


def select(attrs, n: int, pred):
    """-> (bitmap uint32[ceil(n/32)], count, ids int64 ascending)."""
    lib = _load()
    cols, ptrs, tarr = _attrs(attrs)
    carr, nc = _clauses(pred)
    nwords = max((n + 31) // 32, 1)
    bitmap = np.zeros(nwords, dtype=np.uint32)
    ids = np.zeros(max(n, 1), dtype=np.int64)
    cnt = ctypes.c_int64(0)
    st = lib.orc_select(ptrs, _ptr(tarr), len(cols), n, carr, nc, _ptr(bitmap), ctypes.byref(cnt), _ptr(ids))
    if st != OK:
        raise OracleError(st, "select")
    return bitmap, int(cnt.value), ids[: cnt.value].copy()


def search(X: np.ndarray, attrs, pred, Q: np.ndarray, k: int, metric: int, row_offset: int = 0,
           nthreads: int = 0):
    """-> (ids int64[q,k], dists float32[q,k], scores float64[q,k])."""
    lib = _load()
    X = np.ascontiguousarray(X, dtype=np.float32)
    Q = np.ascontiguousarray(Q, dtype=np.float32)
    n, d = X.shape
    q = Q.shape[0]
    if q and Q.shape[1] != d:
        raise OracleError(EINVAL, "search (dimension mismatch)")
    cols, ptrs, tarr = _attrs(attrs)
    carr, nc = _clauses(pred)
    ids = np.zeros((q, k), dtype=np.int64)
    dists = np.zeros((q, k), dtype=np.float32)
    sc = np.zeros((q, k), dtype=np.float64)
    st = lib.orc_search(_ptr(X), n, d, ptrs, _ptr(tarr), len(cols), carr, nc, _ptr(Q), q, k, metric,
                        row_offset, _ptr(ids), _ptr(dists), _ptr(sc), nthreads)
    if st != OK:
        raise OracleError(st, "search")
    return ids, dists, sc


def score(X: np.ndarray, q: np.ndarray, local_ids, metric: int) -> np.ndarray:
    """fp64 eps(q, X[i]) for the given local row ids."""
    lib = _load()
    X = np.ascontiguousarray(X, dtype=np.float32)
    q = np.ascontiguousarray(q, dtype=np.float32)
    ids = np.ascontiguousarray(np.asarray(local_ids, dtype=np.int64))
    out = np.zeros(len(ids), dtype=np.float64)
    st = lib.orc_score(_ptr(X), X.shape[1], _ptr(q), _ptr(ids), len(ids), metric, _ptr(out))
    if st != OK:
        raise OracleError(st, "score")
    return out


def merge(cand_ids: np.ndarray, cand_dists: np.ndarray, k: int, metric: int):
    """cand_*: [parts, q, k] -> top-k of the union, (ids [q,k], dists [q,k])."""
    lib = _load()
    cand_ids = np.ascontiguousarray(cand_ids, dtype=np.int64)
    cand_dists = np.ascontiguousarray(cand_dists, dtype=np.float32)
    parts, q, kk = cand_ids.shape
    assert kk == k
    ids = np.zeros((q, k), dtype=np.int64)
    dists = np.zeros((q, k), dtype=np.float32)
    st = lib.orc_merge(_ptr(cand_ids), _ptr(cand_dists), parts, q, k, metric, _ptr(ids), _ptr(dists))
    if st != OK:
        raise OracleError(st, "merge")
    return ids, dists


def range_search(X: np.ndarray, attrs, pred, Q: np.ndarray, tau: float, metric: int, row_offset: int = 0,
                 nthreads: int = 0):
    """Threshold selection (orc_range): every qualifying row with score >= tau
    (IP, COS) / squared distance <= tau (L2), ascending id.
    -> (offsets int64[q+1], ids int64[total], dists float32[total], scores float64[total])."""
    lib = _load()
    X = np.ascontiguousarray(X, dtype=np.float32)
    Q = np.ascontiguousarray(Q, dtype=np.float32)
    n, d = X.shape
    q = Q.shape[0]
    if q and Q.shape[1] != d:
        raise OracleError(EINVAL, "range_search (dimension mismatch)")
    cols, ptrs, tarr = _attrs(attrs)
    carr, nc = _clauses(pred)
    offsets = np.zeros(q + 1, dtype=np.int64)
    cap = 0
    for _ in range(2):   # count, then fill with the exact capacity
        ids = np.zeros(max(cap, 1), dtype=np.int64)
        dists = np.zeros(max(cap, 1), dtype=np.float32)
        sc = np.zeros(max(cap, 1), dtype=np.float64)
        st = lib.orc_range(_ptr(X), n, d, ptrs, _ptr(tarr), len(cols), carr, nc, _ptr(Q), q, float(tau), metric,
                           row_offset, cap, _ptr(offsets), _ptr(ids), _ptr(dists), _ptr(sc), nthreads)
        if st == OK:
            t = int(offsets[q])
            return offsets, ids[:t].copy(), dists[:t].copy(), sc[:t].copy()
        if st != ERANGE:
            raise OracleError(st, "range_search")
        cap = int(offsets[q])
    raise OracleError(ERANGE, "range_search")


def num_threads() -> int:
    return int(_load().orc_num_threads())
