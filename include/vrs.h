/*
 * vrs.h -- C ABI of libvrs: batched, relationally filtered, exact k-NN search
 * on NVIDIA B200 (sm_100a).
 *
 * The operation is the paper's selection with a query vector, a similarity
 * predicate and a relational predicate, evaluated predicate-first:
 *
 *   PAPER.md L285-L288 (Sec. 3):  sigma_{eps,v,theta_R}(R) <=> sigma_eps(v x sigma_{theta_R}(R))
 *
 * for a whole batch of query vectors at once ("batching both
 * the data and query vectors"), one relational predicate per batch
 * (late materialization), and eps = "the k best under a
 * metric" (PAPER.md L350 top-k; result contract SPEC.md L141-L147).
 *
 * Conventions shared by every call
 *  - Device pointers are CUDA device (or managed) memory of the current
 *    device; host pointers are rejected with VRS_EINVAL unless the call says
 *    otherwise.  Integers are little-endian, arrays are dense row-major.
 *  - Every call that takes `cuda_stream` (a cudaStream_t; NULL = legacy
 *    default stream) validates its arguments synchronously, enqueues all
 *    device work on that stream and returns without synchronising.  Device
 *    faults surface as VRS_ECUDA on a later call.
 *  - On any error nothing is enqueued and vrs_last_error() describes it.
 *  - Metrics (reading R1 in DESIGN.md):
 *      VRS_L2      squared Euclidean distance sum_t (q_t - x_t)^2, best = smallest
 *      VRS_IP      inner product sum_t q_t x_t, best = largest
 *      VRS_COSINE  cosine SIMILARITY <q,x>/(|q||x|), best = largest
 *                  ("dot product of two normalized input matrices")
 *  - Results: row j of ids/dists holds the m = min(k, N_sel) best qualifying
 *    rows of query j, best first, ties broken by the lower global row id
 *    (SPEC.md L145, L177); entries m..k-1 are padding id = -1 and
 *    dist = +inf (L2) or -inf (IP, COSINE).  ids are GLOBAL: row_offset + local row.
 *    dists are computed exactly in fp32 from the fp32 inputs (the tensor-core
 *    selection pass is re-scored).
 *  - Exactness (Table 1 "Accuracy: Exact"; L26): the returned
 *    rows ARE the top-k of the definition, not an approximation.  The fast
 *    selection pass (16-bit / TF32 tensor-core keys, or fp32 FFMA keys) carries
 *    a per-query error bound E; a query is CERTIFIED when the k-th exact score
 *    of the re-scored candidates beats every unselected row's key + E.
 *    Uncertified queries are recomputed on the device by an exact fp64 scan of
 *    the qualifying rows.  No host synchronisation.
 */
#ifndef VRS_H
#define VRS_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define VRS_API __attribute__((visibility("default")))
#else
#define VRS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define VRS_ABI_VERSION 2
/* Largest k vrs_search accepts (the selection pass over-fetches k' = the power of two >= k + 16). */
#define VRS_K_MAX 240
/* Largest number of AND-ed clauses in one predicate. */
#define VRS_MAX_CLAUSES 8

typedef enum {
  VRS_OK = 0,
  VRS_EINVAL = 1,        /* bad argument: sizes, null / host pointer, enum value, d mismatch */
  VRS_ENOTFOUND = 2,     /* a clause names an attribute index >= n_attrs */
  VRS_EDEGENERATE = 3,   /* VRS_COSINE over a corpus holding a zero-norm row */
  VRS_ENOMEM = 4,        /* the allocator returned NULL */
  VRS_ECUDA = 5,         /* a CUDA runtime error (including asynchronous faults) */
  VRS_ECOMM = 6,         /* reserved for collective errors raised by callers of vrs_merge */
  VRS_EUNSUPPORTED = 7,  /* k > VRS_K_MAX, too many clauses, or a device that is not sm_100 */
  VRS_ERANGE = 8         /* vrs_range_search: more results than `capacity` (*total = the size needed) */
} vrs_status;

typedef enum { VRS_L2 = 0, VRS_IP = 1, VRS_COSINE = 2 } vrs_metric;

typedef enum { VRS_ATTR_I32 = 0, VRS_ATTR_U8 = 1 } vrs_attr_type;

/* One relational column: `data` is a device array of n entries (int32 or uint8). */
typedef struct {
  vrs_attr_type type;
  const void *data;
} vrs_attr;

/* One clause of theta_R: lo <= attr[i] <= hi, compared as exact integers
 * (uint8 as unsigned).  lo > hi selects nothing.  (reading R4;
 * SPEC.md L48-L52 LT/LE/GT/GE/BETWEEN all map to one closed interval.) */
typedef struct {
  int32_t attr;
  int64_t lo;
  int64_t hi;
} vrs_clause;

/* theta_R = AND of the clauses; n_clauses == 0 (clauses may be NULL) selects every row. */
typedef struct {
  int32_t n_clauses;
  const vrs_clause *clauses;
} vrs_predicate;

/* Optional stream-ordered allocator for ALL of the library's own device memory (norms and
 * shadow at load, per-call scratch on the call's stream, vrs_search_host staging with
 * stream NULL).  NULL => cudaMalloc / cudaMallocAsync + cudaFreeAsync.  alloc returning
 * NULL makes the call fail with VRS_ENOMEM.  The Python binding passes torch's caching
 * allocator. */
typedef struct {
  void *(*alloc)(size_t bytes, void *cuda_stream, void *ctx);
  void (*free)(void *ptr, void *cuda_stream, void *ctx);
  void *ctx;
} vrs_allocator;

typedef struct vrs_index vrs_index;

/* Operand precision of the tensor-core SELECTION pass.
 * Returned distances are always re-scored exactly from the fp32 inputs and the
 * result is certified exact whatever the precision; the precision decides the
 * pass's speed and how often its certificate holds without the exact fallback. */
typedef enum {
  VRS_PREC_DEFAULT = 0,  /* load: fp16 shadow when d % 8 == 0; search: the index's own */
  VRS_PREC_TF32 = 1,     /* tcgen05 kind::tf32 on the fp32 corpus (no extra memory) */
  VRS_PREC_BF16 = 2,     /* tcgen05 kind::f16 on a bf16 shadow copy built at load (+2 bytes / element) */
  VRS_PREC_FP16 = 3      /* tcgen05 kind::f16 on an fp16 shadow (+2 bytes / element): the corpus scaled by one
                            power of two 2^e_x at load, each query by its own 2^e_q, so the 11-bit significand
                            is used in full (8x tighter selection keys than bf16 at the same cost) */
} vrs_precision;

typedef struct {
  int32_t precision;     /* vrs_precision */
  int32_t reserved[7];
} vrs_load_options;

/*
 * vrs_load -- build an index over one (shard of a) relation R (PAPER.md L269,
 * "column-store layout that stores both vector and relational data").
 *   vectors : device fp32 [n x d], row-major, BORROWED: must stay valid and
 *             unmodified until vrs_free.  16-byte aligned rows (d % 4 == 0 and a
 *             16-byte aligned base) enable the vectorised / TMA paths; other
 *             layouts run on the scalar-load scan path.
 *   attrs   : n_attrs relational columns (device, n entries each), BORROWED.
 *   row_offset : global id of local row 0 (row sharding).
 *   alloc   : optional allocator (copied; its ctx must outlive the index).
 * Computes per-row |x|^2 and 1/|x| once (the norm terms of PAPER.md L305, L790)
 * on `cuda_stream` and waits for them (load is not on the search path).
 * Errors: EINVAL (n < 1, n >= 2^31, d < 1, n_attrs < 0, null / host pointers,
 * bad attr type), ENOMEM, ECUDA, EUNSUPPORTED (device is not sm_100).
 */
VRS_API vrs_status vrs_load(const float *vectors, int64_t n, int32_t d, const vrs_attr *attrs, int32_t n_attrs,
                    int64_t row_offset, const vrs_allocator *alloc, void *cuda_stream, vrs_index **out);

/*
 * vrs_load_ex -- vrs_load with options (opts == NULL => defaults).  precision:
 * DEFAULT builds the fp16 shadow when d % 8 == 0 and the base is 16-byte aligned;
 * TF32 never builds one; FP16 / BF16 require it (else VRS_EUNSUPPORTED).  The
 * shadow is index-owned memory (n * d * 2 bytes, through `alloc`), converted on
 * `cuda_stream` with round-to-nearest-even; the load also measures the shadow's
 * per-row rounding residual |x~ - x| exactly (fp64) -- the certificate's bound.
 */
VRS_API vrs_status vrs_load_ex(const float *vectors, int64_t n, int32_t d, const vrs_attr *attrs, int32_t n_attrs,
                               int64_t row_offset, const vrs_allocator *alloc, const vrs_load_options *opts,
                               void *cuda_stream, vrs_index **out);

/*
 * vrs_search -- sigma_{eps,v,theta_R}(R) for a batch of q query vectors.
 *   queries : device fp32 [q x d] row-major (d must equal the loaded d).
 *   pred    : theta_R (NULL => every row).
 *   k       : 1..VRS_K_MAX.
 *   ids     : device int64 [q x k] (output), dists: device fp32 [q x k] (output).
 * q == 0 is a successful no-op.  A zero-norm COSINE query yields an all-padding
 * row (documented deviation from SPEC.md L95: detecting it would need a host sync).
 * Errors: EINVAL, ENOTFOUND, EDEGENERATE, EUNSUPPORTED, ENOMEM, ECUDA.
 */
VRS_API vrs_status vrs_search(vrs_index *ix, const float *queries, int64_t q, int32_t d, const vrs_predicate *pred,
                      int32_t k, vrs_metric metric, int64_t *ids, float *dists, void *cuda_stream);

/* Path control for tests and the bench (vrs_search uses VRS_PATH_AUTO). */
typedef enum {
  VRS_PATH_AUTO = 0,  /* dispatch on (q, d): scan for small batches, tensor cores above */
  VRS_PATH_SCAN = 1,  /* per-tuple fp32 FFMA scan over the selection */
  VRS_PATH_GEMM = 2   /* batched tcgen05 tensor-core formulation */
} vrs_path;

typedef enum {
  VRS_ROWS_AUTO = 0,    /* selectivity-driven choice between the two below */
  VRS_ROWS_GATHER = 1,  /* compact the selection, deliver only qualifying rows (late materialization) */
  VRS_ROWS_MASKED = 2   /* stream full row tiles, unqualified rows masked out by the bitmap */
} vrs_rows;

typedef struct {
  int32_t path;      /* vrs_path */
  int32_t rows;      /* vrs_rows */
  int32_t precision; /* vrs_precision of the tensor-core selection (DEFAULT: the index's shadow if it has one, else TF32) */
  int32_t host_async; /* vrs_search_host only (the host buffers must then be pinned):
                         0 = synchronise cuda_stream before returning;
                         1 = do not synchronise; cuda_stream is ordered after the device->host copies,
                             the caller synchronises it before reading h_ids / h_dists;
                         2 = overlap: cuda_stream is NOT ordered after the copies (the next call's
                             kernels overlap this call's download); h_ids / h_dists are complete once
                             vrs_host_fence(ix, s) has been enqueued on a stream s and s has synchronised */
  int32_t reserved0;
  /* Optional DEVICE uint64 [4] the call accumulates into (NULL: nothing is recorded):
   *   [0] += queries answered, [1] += queries whose first selection was NOT certified
   *   (re-selected by the refine pass when it runs, else recomputed exactly), [2] =
   *   max(previous, the largest observed |selection key - exact key| / E over all
   *   re-scored candidates) as IEEE-754 double bits (< 1 confirms the bound on this data),
   *   [3] += queries recomputed by the exact fp64 fallback. */
  uint64_t *stats;
  int32_t reserved[2];
} vrs_search_options;

/* vrs_search with explicit options (opts == NULL => defaults). */
VRS_API vrs_status vrs_search_ex(vrs_index *ix, const float *queries, int64_t q, int32_t d, const vrs_predicate *pred,
                         int32_t k, vrs_metric metric, int64_t *ids, float *dists,
                         const vrs_search_options *opts, void *cuda_stream);

/*
 * vrs_search_host -- end-to-end call on HOST buffers: copies the queries
 * host->device, runs vrs_search_ex, copies ids/dists device->host, and
 * synchronises `cuda_stream` before returning (unless opts->host_async, then
 * the caller synchronises).  h_queries / h_ids / h_dists are host memory
 * (pinned memory makes the copies asynchronous DMA; required with host_async).
 */
VRS_API vrs_status vrs_search_host(vrs_index *ix, const float *h_queries, int64_t q, int32_t d,
                           const vrs_predicate *pred, int32_t k, vrs_metric metric, int64_t *h_ids,
                           float *h_dists, const vrs_search_options *opts, void *cuda_stream);

/*
 * vrs_host_fence -- orders cuda_stream after every device->host result copy that
 * vrs_search_host has issued on `ix` so far (for host_async = 2).  Enqueues a
 * wait only; never blocks the host.  Errors: VRS_EINVAL (ix NULL), VRS_ECUDA.
 */
VRS_API vrs_status vrs_host_fence(vrs_index *ix, void *cuda_stream);

/*
 * vrs_range_search -- threshold selection instead of top-k: eps = "the score
 * satisfies tau" (Sec. 5: "We use cosine similarity > 0.9";
 * L1436, Sec. 6: "range instead of top-k search").
 * For each query j, every qualifying row with score >= tau (VRS_IP, VRS_COSINE)
 * or squared distance <= tau (VRS_L2), in ascending global row id, with its
 * exact score (fp64 from the fp32 inputs, rounded once to fp32); the decision
 * score-vs-tau is taken on that fp64 score.
 *   offsets : device int64 [q + 1] (output): query j's results are
 *             ids[offsets[j] .. offsets[j+1]), offsets[q] = total.
 *   ids     : device int64 [capacity], dists: device fp32 [capacity] (outputs).
 *   total   : HOST int64 (output): the number of results.
 * The call SYNCHRONISES `cuda_stream` twice (once to size the candidate buffer,
 * once to check `capacity`); the final writes stay enqueued.  If total >
 * capacity it returns VRS_ERANGE with *total and the device offsets valid and
 * ids / dists untouched: call again with capacity >= *total.
 * Runs on the tensor-core path (d % 4 == 0, 16-byte aligned rows and queries);
 * other shapes get VRS_EUNSUPPORTED.  opts: precision / rows as in vrs_search_ex
 * (path is ignored).  Errors: as vrs_search, plus EINVAL for a NaN tau or a
 * negative capacity, ERANGE.
 */
VRS_API vrs_status vrs_range_search(vrs_index *ix, const float *queries, int64_t q, int32_t d,
                                    const vrs_predicate *pred, double tau, vrs_metric metric, int64_t capacity,
                                    int64_t *offsets, int64_t *ids, float *dists, int64_t *total,
                                    const vrs_search_options *opts, void *cuda_stream);

/*
 * vrs_select -- the relational step alone, sigma_{theta_R}(R):
 *   bitmap : device uint32 [ceil(n/32)], word w bit b <-> local row 32w+b,
 *            LSB first, bits past n zero (output).
 *   count  : device int64 [1], the number of qualifying rows (output).
 *   ids    : optional device int32 [n] (NULL allowed): ascending qualifying local row ids.
 * Bit-exact by construction (integer work).  Errors: EINVAL, ENOTFOUND, ECUDA.
 */
VRS_API vrs_status vrs_select(vrs_index *ix, const vrs_predicate *pred, uint32_t *bitmap, int64_t *count, int32_t *ids,
                      void *cuda_stream);

/*
 * vrs_merge -- final step of a row-sharded search (north_star (4)): the top-k
 * of the union of n_parts candidate lists, each the vrs_search output of one
 * shard (same q, k, metric), as gathered by an all-gather.
 *   cand_ids   : device int64 [n_parts x q x k] (padding id = -1 ignored)
 *   cand_dists : device fp32  [n_parts x q x k]
 *   ids, dists : device [q x k] outputs, same ordering / tie / padding rules.
 * Exact: top-k(A u B) = top-k(top-k(A) u top-k(B)) under the total order (dist, id).
 */
VRS_API vrs_status vrs_merge(const int64_t *cand_ids, const float *cand_dists, int32_t n_parts, int64_t q, int32_t k,
                     vrs_metric metric, int64_t *ids, float *dists, void *cuda_stream);

/*
 * vrs_merge_push -- the multi-GPU exchange and merge in ONE kernel over peer memory
 * (north_star (4); SURVEY 8(e) mitigation 2: one-shot P2P stores, a device-side wait, the
 * merge): every rank calls it on its own stream with its exact local vrs_search output; the
 * kernel stores that [q x k] into this rank's slot of every rank's receive buffer (NVLink
 * P2P), counts the push there with a system-scope atomic, waits until every rank's push of
 * this call has arrived in its own buffer, and writes the top-k of the union -- the same
 * result as vrs_merge over an all-gather.  No host synchronisation; CUDA-graph capturable
 * (the call counter lives in `state`).
 *   local_ids, local_dists : device [q x k], this rank's vrs_search output (global ids)
 *   peer_bufs  : DEVICE array of n_parts pointers, rank p's receive buffer as mapped on this
 *                GPU (e.g. torch symmetric memory's buffer_ptrs_dev); each buffer holds
 *                buf_bytes >= vrs_push_buffer_bytes(n_parts, q, k) bytes, its first 256 bytes
 *                zeroed before the first call (ownership: the caller's)
 *   n_parts    : ranks, 1..64;  my_part : this rank, 0..n_parts-1
 *   state      : this rank's device uint32[4], zeroed before the first call, then owned by
 *                the calls (every rank must make the same sequence of calls); state[3] != 0
 *                after a call: a peer's push did not arrive within the wait bound (20 s,
 *                VRS_PUSH_TIMEOUT_MS) -- that call's and every later call's output is invalid
 *   ids, dists : device [q x k] outputs (may not alias the inputs)
 * Errors: VRS_EINVAL (bad sizes, host pointers, buffer too small), VRS_EUNSUPPORTED
 * (k > VRS_K_MAX, n_parts > 64).  All ranks' kernels must be able to run concurrently
 * (one process per GPU): a rank whose peers never call gives up after the wait bound and
 * sets state[3] (the status of the launch is still VRS_OK: the host reads the flag).
 */
VRS_API vrs_status vrs_merge_push(const int64_t *local_ids, const float *local_dists, void *const *peer_bufs,
                                  int64_t buf_bytes, int32_t n_parts, int32_t my_part, int64_t q, int32_t k,
                                  vrs_metric metric, uint32_t *state, int64_t *ids, float *dists, void *cuda_stream);
/* Bytes each rank's receive buffer needs for vrs_merge_push(n_parts, q, k). */
VRS_API int64_t vrs_push_buffer_bytes(int32_t n_parts, int64_t q, int32_t k);

/* Release the index's own memory (borrowed vectors / attrs are untouched). NULL is a no-op. */
VRS_API vrs_status vrs_free(vrs_index *ix);

/* Thread-local description of the last failure on this thread; valid until the next vrs_* call. */
VRS_API const char *vrs_last_error(void);

/* Introspection for tests / bench: which path the last vrs_search_ex on this
 * thread took (vrs_path value) and how many kernels it enqueued. */
VRS_API int32_t vrs_last_path(void);
/* vrs_precision of the last vrs_search_ex's tensor-core pass on this thread (DEFAULT when it took the scan path). */
VRS_API int32_t vrs_last_precision(void);
/* VRS_PREC_FP16 / VRS_PREC_BF16 if the index holds that shadow, else VRS_PREC_TF32. */
VRS_API int32_t vrs_index_precision(const vrs_index *ix);
VRS_API int32_t vrs_last_launches(void);

/*
 * Kernel timing for the bench (bench.py "roofline"): while enabled, every
 * kernel libvrs enqueues is bracketed by CUDA events recorded on its launch
 * stream; vrs_profile_read(i, ...) resolves them (synchronising those events)
 * and reports per-kernel totals since the last reset.  Returns the number of
 * kernel names (i past the end leaves the outputs untouched).
 */
VRS_API void vrs_profile_enable(int32_t on);
VRS_API int32_t vrs_profile_read(int32_t i, const char **name, double *total_ms, int64_t *launches);
VRS_API void vrs_profile_reset(void);

/* Bytes the library's own stream-ordered pool (cudaMallocAsync, used for per-call scratch
 * when the index has no allocator) currently reserves on the current device; it keeps at
 * most 2 GiB of freed scratch cached and releases the rest at synchronisation.  -1 on error. */
VRS_API int64_t vrs_pool_reserved_bytes(void);

/* Loaded index properties. */
VRS_API int64_t vrs_index_rows(const vrs_index *ix);
VRS_API int32_t vrs_index_dim(const vrs_index *ix);

#ifdef __cplusplus
}
#endif
#endif /* VRS_H */
