"""paper_2403_15807_b200 -- B200-native filtered exact top-k vector search.

The hot path of the scan-based access path of Sanca & Ailamaki,
"Efficient Data Access Paths for Mixed Vector-Relational Search"
(arxiv 2403.15807): sigma_{eps,v,theta_R}(R) <=> sigma_eps(v x sigma_{theta_R}(R))
 for a batch of queries, on hand-written sm_100a CUDA
kernels behind the C ABI in include/vrs.h.  This package is a thin binding:
torch supplies device memory, streams and process groups only.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import (ATTR_I32, ATTR_U8, COSINE, EXPORTS, IP, K_MAX, L2, PATH_AUTO, PATH_GEMM, PATH_SCAN,
                   PREC_BF16, PREC_DEFAULT, PREC_FP16, PREC_TF32, ROWS_AUTO, ROWS_GATHER, ROWS_MASKED, VrsError)

__all__ = ["Index", "merge", "VrsError", "L2", "IP", "COSINE", "PATH_AUTO", "PATH_SCAN", "PATH_GEMM",
           "ROWS_AUTO", "ROWS_GATHER", "ROWS_MASKED", "PREC_DEFAULT", "PREC_TF32", "PREC_BF16", "PREC_FP16", "K_MAX",
           "last_path", "new_stats", "read_stats", "pool_reserved_bytes",
           "last_precision", "last_launches", "library"]

METRICS = {"l2": L2, "ip": IP, "cos": COSINE, "cosine": COSINE}


def library():
    return _lib.load_library()


def _metric(m):
    return METRICS[m.lower()] if isinstance(m, str) else int(m)


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(stream=None):
    if stream is None and _raw_stream is not None:   # (no Stream object per call)
        return ctypes.c_void_p(_raw_stream(torch.cuda.current_device()))
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


_opt_cache = {}


def _options(path, rows, precision=None, host_async=False, stats=None):
    sp = 0
    if stats is not None:
        if stats.dtype != torch.int64 or stats.numel() < 4 or not stats.is_cuda or not stats.is_contiguous():
            raise ValueError("stats must be a contiguous CUDA int64 tensor of >= 4 entries (new_stats())")
        sp = stats.data_ptr()
    if path is None and rows is None and precision is None and not host_async and not sp:
        return None
    key = (path, rows, precision, int(host_async), sp)
    if key in _opt_cache:
        return _opt_cache[key][1]
    o = _lib.SearchOptions()
    o.path = PATH_AUTO if path is None else int(path)
    o.rows = ROWS_AUTO if rows is None else int(rows)
    o.precision = PREC_DEFAULT if precision is None else int(precision)
    o.host_async = int(host_async)   # False / True (1) / 2 = overlap (see vrs.h)
    o.stats = sp or None
    if len(_opt_cache) > 4096:
        _opt_cache.clear()
    _opt_cache[key] = (o, ctypes.byref(o))   # the struct stays alive with its reference
    return _opt_cache[key][1]


def new_stats(device=None) -> torch.Tensor:
    """A zeroed device counter block for search(..., stats=): [queries, queries whose fp16
    selection was not certified, max observed key error / bound (double bits), queries that
    reached the exact fp64 fallback (the rest were certified by the refine pass)]."""
    return torch.zeros(4, dtype=torch.int64, device=device or torch.device("cuda", torch.cuda.current_device()))


def read_stats(stats: torch.Tensor) -> dict:
    """Decode a stats block (synchronises): queries, uncertified, certified fraction, max key error / bound."""
    v = stats.cpu()
    q, u, fb = int(v[0]), int(v[1]), int(v[3])
    ratio = float(v[2:3].view(torch.float64)[0])
    return {"queries": q, "uncertified": u, "certified_fraction": (q - u) / q if q else 1.0,
            "refined": u - fb, "exact_fallback": fb, "max_key_error_over_bound": ratio}


def _torch_allocator():
    """vrs_allocator backed by torch's caching allocator (SURVEY 8(b) "Ownership": the index's
    derived data and every call's scratch come from torch's pool; a failed allocation makes the
    call return VRS_ENOMEM).  Blocks are tied to the stream they are allocated on, so a block
    freed right after the call's kernels were enqueued is reused only in stream order."""
    def alloc(nbytes, stream, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device(), stream or 0)
        except Exception:   # noqa: BLE001 -- out of memory: NULL -> VRS_ENOMEM
            return None

    def free(ptr, stream, ctx):
        if ptr:
            torch.cuda.caching_allocator_delete(ptr)

    a = _lib.Allocator(_lib.ALLOC_FN(alloc), _lib.FREE_FN(free), None)
    return a


def pool_reserved_bytes() -> int:
    """Bytes libvrs's own cudaMallocAsync pool reserves on the current device (0 when every
    index uses the torch allocator)."""
    return int(library().vrs_pool_reserved_bytes())


def _check_queries(queries: torch.Tensor, d: int, device, host: bool = False):
    if not isinstance(queries, torch.Tensor) or queries.dtype != torch.float32 or queries.dim() != 2:
        raise ValueError("queries must be a float32 [q, d] tensor")
    if queries.shape[0] and queries.shape[1] != d:
        raise ValueError(f"queries have {queries.shape[1]} columns, the index d = {d}")
    if not queries.is_contiguous():
        raise ValueError("queries must be contiguous (row-major)")
    if host:
        if queries.is_cuda:
            raise ValueError("search_host takes HOST queries (use search for device tensors)")
    elif queries.device != device:
        raise ValueError(f"queries are on {queries.device}, the index on {device}")


def _check_out(out, q, k, device):
    ids, dists = out
    for t, dt, nm in ((ids, torch.int64, "ids"), (dists, torch.float32, "dists")):
        if t.dtype != dt or tuple(t.shape) != (q, k) or not t.is_contiguous() or t.device != device:
            raise ValueError(f"out {nm} must be a contiguous {dt} [{q}, {k}] tensor on {device}")


def last_path() -> int:
    return int(library().vrs_last_path())


def last_precision() -> int:
    """Tensor-core selection precision of the last search on this thread (PREC_DEFAULT: scan path)."""
    return int(library().vrs_last_precision())


def last_launches() -> int:
    return int(library().vrs_last_launches())


def profile(on: bool = True):
    """Enable / disable per-kernel CUDA-event timing inside libvrs."""
    library().vrs_profile_enable(1 if on else 0)


def profile_reset():
    library().vrs_profile_reset()


def profile_read() -> dict:
    """{kernel: (total_ms, launches)} since the last reset (synchronises the recorded events)."""
    lib = library()
    out = {}
    n = lib.vrs_profile_read(-1, None, None, None)
    for i in range(n):
        name, ms, cnt = ctypes.c_char_p(), ctypes.c_double(), ctypes.c_int64()
        lib.vrs_profile_read(i, ctypes.byref(name), ctypes.byref(ms), ctypes.byref(cnt))
        out[name.value.decode()] = (ms.value, cnt.value)
    return out


class Index:
    """vrs_load over one (shard of a) relation: fp32 vectors [n, d] and
    int32 / uint8 attribute columns, all CUDA tensors (borrowed, kept alive here)."""

    def __init__(self, vectors: torch.Tensor, attrs=(), row_offset: int = 0, stream=None, precision=None,
                 allocator="torch"):
        """allocator: "torch" (default) -- the library's own memory (norms, 16-bit shadow, per-call
        scratch) comes from torch's caching allocator; None -- libvrs's bounded cudaMallocAsync
        pool; or a ready _lib.Allocator (tests)."""
        lib = library()
        if vectors.dtype != torch.float32 or vectors.dim() != 2 or not vectors.is_contiguous() or not vectors.is_cuda:
            raise ValueError("vectors must be a contiguous float32 [n, d] CUDA tensor")
        self.vectors = vectors
        self.attrs = [a.contiguous() for a in attrs]
        for i, a in enumerate(self.attrs):
            if a.dim() != 1 or a.numel() != vectors.shape[0] or a.device != vectors.device:
                raise ValueError(f"attribute {i}: a 1-D tensor of n = {vectors.shape[0]} entries on {vectors.device} "
                                 f"is required (got {tuple(a.shape)} on {a.device})")
        carr = (_lib.Attr * max(len(self.attrs), 1))()
        for i, a in enumerate(self.attrs):
            if a.dtype == torch.int32:
                carr[i].type = ATTR_I32
            elif a.dtype == torch.uint8:
                carr[i].type = ATTR_U8
            else:
                raise ValueError(f"attribute {i}: dtype {a.dtype} (int32 or uint8 expected)")
            carr[i].data = a.data_ptr()
        h = ctypes.c_void_p()
        n, d = vectors.shape
        opts = _lib.LoadOptions()
        opts.precision = PREC_DEFAULT if precision is None else int(precision)
        if allocator == "torch":
            allocator = _torch_allocator()
        self._alloc = allocator   # (the callbacks must outlive the index)
        st = lib.vrs_load_ex(_ptr(vectors), n, d, carr, len(self.attrs), int(row_offset),
                             ctypes.byref(allocator) if allocator is not None else None, ctypes.byref(opts),
                             _stream(stream), ctypes.byref(h))
        _lib.check(st, "vrs_load_ex")
        self.precision = int(lib.vrs_index_precision(h))
        self._h = h
        self.n, self.d, self.row_offset = int(n), int(d), int(row_offset)

    def close(self):
        if getattr(self, "_h", None):
            library().vrs_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def search(self, queries: torch.Tensor, pred=None, k: int = 10, metric="l2", path=None, rows=None,
               out=None, stream=None, precision=None, stats=None):
        """-> (ids int64 [q, k], dists float32 [q, k]) on the device (async on `stream`).
        stats: optional new_stats() block the call accumulates into (certificate counters)."""
        lib = library()
        dev = self.vectors.device
        _check_queries(queries, self.d, dev)
        q, d = queries.shape[0], self.d
        if out is None:
            ids = torch.empty((q, k), dtype=torch.int64, device=dev)
            dists = torch.empty((q, k), dtype=torch.float32, device=dev)
        else:
            _check_out(out, q, k, dev)
            ids, dists = out
        pr, keep = _lib.make_predicate(pred)
        st = lib.vrs_search_ex(self._h, _ptr(queries) if q else None, q, d, ctypes.byref(pr), int(k),
                               _metric(metric), _ptr(ids) if q else None, _ptr(dists) if q else None,
                               _options(path, rows, precision, stats=stats), _stream(stream))
        _lib.check(st, "vrs_search")
        return ids, dists

    def search_host(self, queries_h: torch.Tensor, pred=None, k: int = 10, metric="l2", path=None, rows=None,
                    out=None, stream=None, precision=None, host_async=False):
        """End-to-end call on host buffers (H2D + search + D2H inside libvrs).  Synchronous,
        unless host_async: True -> the caller synchronises the stream (pinned buffers);
        2 -> overlap: results are complete after host_fence(stream) + a stream sync."""
        lib = library()
        _check_queries(queries_h, self.d, None, host=True)
        q, d = queries_h.shape
        if out is None:
            ids = torch.empty((q, k), dtype=torch.int64, pin_memory=True)
            dists = torch.empty((q, k), dtype=torch.float32, pin_memory=True)
        else:
            _check_out(out, q, k, torch.device("cpu"))
            ids, dists = out
        pr, keep = _lib.make_predicate(pred)
        st = lib.vrs_search_host(self._h, _ptr(queries_h), q, d, ctypes.byref(pr), int(k), _metric(metric),
                                 _ptr(ids), _ptr(dists), _options(path, rows, precision, host_async),
                                 _stream(stream))
        _lib.check(st, "vrs_search_host")
        return ids, dists

    def host_fence(self, stream=None):
        """vrs_host_fence: order `stream` after every result download search_host issued."""
        _lib.check(library().vrs_host_fence(self._h, _stream(stream)), "vrs_host_fence")

    def range_search(self, queries: torch.Tensor, pred=None, tau: float = 0.9, metric="cos", capacity=None,
                     rows=None, precision=None, stream=None):
        """vrs_range_search: every qualifying row with score >= tau (ip / cos) or squared
        distance <= tau (l2), ascending global id.  -> (offsets int64 [q+1], ids int64 [total],
        dists float32 [total]) on the device.  Synchronises the stream (the result size is
        data-dependent); grows the output and calls again if `capacity` is too small."""
        lib = library()
        dev = self.vectors.device
        _check_queries(queries, self.d, dev)
        q, d = queries.shape[0], self.d
        offsets = torch.empty(q + 1, dtype=torch.int64, device=dev)
        cap = int(capacity) if capacity is not None else max(1024, 64 * q)
        pr, keep = _lib.make_predicate(pred)
        for _ in range(2):
            ids = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
            dists = torch.empty(max(cap, 1), dtype=torch.float32, device=dev)
            total = ctypes.c_int64(0)
            st = lib.vrs_range_search(self._h, _ptr(queries) if q else None, q, d, ctypes.byref(pr), float(tau),
                                      _metric(metric), cap, _ptr(offsets), _ptr(ids), _ptr(dists),
                                      ctypes.byref(total), _options(None, rows, precision), _stream(stream))
            if st == _lib.ERANGE:
                cap = int(total.value)
                continue
            _lib.check(st, "vrs_range_search")
            t = int(total.value)
            return offsets, ids[:t], dists[:t]
        _lib.check(st, "vrs_range_search")

    def select(self, pred=None, with_ids: bool = False, stream=None):
        """-> (bitmap uint32-as-int32 [ceil(n/32)], count int64 [1], ids int32 [n] or None); device tensors."""
        lib = library()
        dev = self.vectors.device
        words = (self.n + 31) // 32
        bitmap = torch.empty(words, dtype=torch.int32, device=dev)
        count = torch.empty(1, dtype=torch.int64, device=dev)
        ids = torch.empty(self.n, dtype=torch.int32, device=dev) if with_ids else None
        pr, keep = _lib.make_predicate(pred)
        st = lib.vrs_select(self._h, ctypes.byref(pr), _ptr(bitmap), _ptr(count), _ptr(ids), _stream(stream))
        _lib.check(st, "vrs_select")
        return bitmap, count, ids


def merge(cand_ids: torch.Tensor, cand_dists: torch.Tensor, k: int, metric="l2", stream=None):
    """vrs_merge: cand_* [parts, q, k] device tensors -> (ids [q, k], dists [q, k])."""
    lib = library()
    parts, q, kk = cand_ids.shape
    if kk != k:
        raise ValueError("candidate lists must have k entries")
    ids = torch.empty((q, k), dtype=torch.int64, device=cand_ids.device)
    dists = torch.empty((q, k), dtype=torch.float32, device=cand_ids.device)
    ci, cd = cand_ids.contiguous(), cand_dists.contiguous()
    st = lib.vrs_merge(_ptr(ci), _ptr(cd), parts, q, int(k), _metric(metric), _ptr(ids), _ptr(dists),
                       _stream(stream))
    _lib.check(st, "vrs_merge")
    return ids, dists
