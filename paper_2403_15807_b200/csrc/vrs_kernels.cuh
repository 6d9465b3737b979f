// vrs_kernels.cuh -- launch interfaces of the libvrs kernels (host side).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "vrs_internal.cuh"

namespace vrs {

// Kernel timing scope (vrs_profile_enable): CUDA events recorded on the launch
// stream around the enclosed launches, resolved by vrs_profile_read.
struct ProfScope {
  const char *name;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  ProfScope(const char *n, cudaStream_t st);
  ~ProfScope();
  ProfScope(const ProfScope &) = delete;
  ProfScope &operator=(const ProfScope &) = delete;
};

// The per-search 16-bit query operand of the tensor-core pass (convert16.cuh
// query_row_to16: per-row power-of-two exponent, 16-bit row, exact residual):
// folded into select_count_kernel (select.cu; saves a launch), or its own
// launch (launch_query16) when there is no predicate.
struct QueryFuse {
  const float *q_in;       // fp32 queries [q x d] (nullptr: no conversion)
  void *q_out;             // 16-bit [rows x d]; rows q..rows-1 are zero (whole 128-row tiles)
  int64_t q, rows;
  int32_t d;
  int32_t fmt;             // 0 fp16, 1 bf16
  int32_t *qexp;           // [q] out: the row's exponent e_q (q~ = 16-bit(q * 2^e_q))
  float *rq;               // [q] out: |q~ 2^-e_q - q| (fp64, rounded up)
};
using SelectFuse = QueryFuse;
cudaError_t launch_query16(const QueryFuse &f, cudaStream_t s);
// the fp16 / bf16 shadow at load (and with out_lo, fp16 only, the refine pass's low half); res
// (device u64[4], zeroed): max |x~ - x|, max |x~ - x| / |x|, and the same after hi + lo, as double bits
cudaError_t launch_shadow(const float *X, int64_t n, int32_t d, int32_t e, int32_t fmt, void *out, void *out_lo,
                          const float *nx2, unsigned long long *res, cudaStream_t s);
// select.cu -- K4'/K5' (the query conversion rides along when `fuse` is given)
cudaError_t launch_select(const PredDev &pred, int64_t n, uint32_t *bitmap, int32_t *ids, int64_t *count,
                          void *scratch, cudaStream_t stream, int *launches, const SelectFuse *fuse = nullptr);
size_t select_scratch_bytes(int64_t n);
// One-kernel selection for the tensor-core path: bitmap, per-chunk counts (scratch,
// select_scratch_bytes) and chunk-local ids (ids_local[c * kSelChunkRows + j], the
// j-th selected row of chunk c); select_finish (gemm_tc.cu) turns them into the
// count, the dense ids and -- in gathered mode -- the copied rows.
constexpr int kSelChunkRows = 8192;
constexpr int kSelFinishMaxChunks = 56 * 1024;   // prefix table in <= 224 KB of shared memory
inline int64_t select_chunks(int64_t n) { return (n + kSelChunkRows - 1) / kSelChunkRows; }
cudaError_t launch_select_local(const PredDev &pred, int64_t n, uint32_t *bitmap, int32_t *ids_local, void *scratch,
                                cudaStream_t stream, int *launches, const SelectFuse *fuse = nullptr);

// scan.cu -- K6' norms, K2' scan + fused top-k
cudaError_t launch_norms(const float *X, int64_t n, int32_t d, float *nx2, float *inv_nx, int32_t *flags,
                         cudaStream_t stream);

struct ScanArgs {
  const float *X;
  int64_t n;
  int32_t d;
  const int32_t *ids;     // compacted ascending local ids, or nullptr => identity over n rows
  const int64_t *count;   // device count of ids (ignored for identity)
  const float *Q;
  int64_t q;
  const float *nx2;
  const float *inv_nx;
  int32_t metric;
  int32_t kprime;         // entries per output list
  float *part_key;        // [P][q][kprime]
  int32_t *part_id;       // [P][q][kprime], -1 = padding
  int32_t P;
  int64_t q_base = 0;     // first query of this launch (launch_scan splits batches over grid.y's limit)
  const void *Xh = nullptr;   // the 16-bit shadow: rows read from it (half the bytes) when set
  int32_t fmt16 = 0;          // 0 fp16, 1 bf16
  int32_t xexp = 0;           // the shadow's exponent e_x
};
int scan_query_group(int64_t q, int d, int kpe);
cudaError_t launch_scan(const ScanArgs &a, int qg, int kpe, cudaStream_t s, int *launches);

// gemm_tc.cu -- K3' tcgen05 GEMM + fused top-k epilogue
// Candidate lists per row split of the tensor-core pass: each of the epilogue's
// 4 x kListsPerSplit warps (4 TMEM lane quadrants) owns BN / kListsPerSplit
// columns of every tile and one (list, query) buffer per query.
#ifndef VRS_LPS
#define VRS_LPS 2
#endif
constexpr int kListsPerSplit = VRS_LPS;

struct GemmPlan {
  int32_t P;        // row splits = candidate lists per query
  int32_t qtiles;   // query tiles of 128
  int32_t ok;       // shape supported
  int32_t min_p;    // splits that keep ~every SM busy over the query tiles (used_splits)
};
GemmPlan gemm_plan(int64_t q, int32_t d, int64_t n_upper, int32_t kprime, int num_sms, bool h16);
bool pair_main(int64_t qtiles, int32_t d, bool h16);

struct GemmArgs {
  const float *X;
  int64_t n;
  int32_t d;
  const int32_t *ids;       // compacted ids (gather) or nullptr (identity)
  const int64_t *count;
  const uint32_t *bitmap;   // selection bitmap (masked mode) or nullptr
  int32_t masked;           // 0 auto (device-side selectivity switch), 1 force masked, 2 force gathered
  void *xsel;               // materialised-selection buffer [xsel_cap x d] fp32 / bf16 (gathered mode)
  int64_t xsel_cap;
  float *xsel_norm;         // [xsel_cap] the gathered rows' norm terms
  const float *Q;
  int64_t q;
  const float *nx2;
  const float *inv_nx;
  int32_t metric;
  int32_t kprime;
  float *part_key;          // [P][q][kprime]
  int32_t *part_id;
  int32_t P;
  int32_t bf16;             // select on the 16-bit shadow (kind::f16) instead of fp32 (kind::tf32)
  const void *Xb;           // 16-bit shadow corpus [n x d] (16-bit only)
  void *Qb;                 // scratch [qtiles * 128 x d] 16-bit queries (16-bit only)
  int32_t prepped;          // 1: the select kernels already converted the queries
  int32_t fmt16 = 0;        // 16-bit format: 0 fp16, 1 bf16
  int32_t xexp = 0;         // the shadow's exponent e_x
  int32_t *qexp = nullptr;  // [q] per-query exponents e_q (written by the conversion)
  float *rq = nullptr;      // [q] per-query residuals |q~ - q|
  int64_t cp_min_bytes = INT64_MAX;   // gathered selections of >= this many row bytes: cp.async by id (vrs_api row_plan)
  int64_t cp_min_rows = INT64_MAX;    // ... or of >= this many rows (cp_fetch)
  int32_t xsel_ready = 0;   // the refine pass: X_sel already holds the gathered rows (no copy launch)
  // launch_select_local's output (nullptr: ids / count were written by launch_select):
  // the tensor-core pass first runs select_finish -> count, dense ids, gathered rows
  const int32_t *ids_local = nullptr;
  const uint32_t *chunk_count = nullptr;
};
size_t gemm_scratch_bytes(const GemmPlan &plan, int64_t q, int32_t kprime);
cudaError_t launch_gemm(const GemmArgs &a, const GemmPlan &plan, void *scratch, cudaStream_t s, int *launches);
// the tensor-core pass's candidate lists, as finalize reads them
struct GemmLists {
  const float *key;        // [lists][q][stride]
  const int32_t *id;
  const int32_t *cnt;      // [lists][q] entries per list
  int32_t lists;
  int32_t stride;
  const uint32_t *gtau;    // [q] ordered-u32 lower bound of the k'-th best key (0 = none)
  SplitInfo split;         // lists 2s, 2s+1 belong to split s; only splits_used() carry entries
};
GemmLists gemm_lists(const GemmArgs &a, const GemmPlan &plan, void *scratch);

// finalize.cu -- K7'/K12' candidate selection + exact re-score; K10' shard merge
struct FinalizeArgs {
  const float *key;        // candidate lists [lists][q][stride] (ranking keys, larger = better)
  const int32_t *id;       // local row ids, -1 = padding
  const int32_t *cnt;      // [lists][q] entries per list, or nullptr: kread entries per list
  int32_t lists;
  int32_t stride;          // list stride in entries
  int32_t kread;           // entries per list when cnt == nullptr
  int32_t sorted;          // lists sorted best-first (scan path): their kprime-th entries bound the result
  const uint32_t *gtau;    // optional [q] ordered-u32 lower bound of the kprime-th best key (0 = none)
  SplitInfo split;         // tensor-core lists: 2 per split, only splits_used() carry entries (bn 0: all)
  int32_t kprime;          // candidates selected for the exact re-score
  int64_t q;
  const float *X;
  int32_t d;
  const float *Q;
  int32_t metric;
  int32_t k;
  int64_t row_offset;
  int64_t *ids;            // [q][k]
  float *dists;            // [q][k]
  // certificate: computed when cert != nullptr
  KeyBound kb{};                   // error-bound constants of the selection pass that produced the keys
  const int32_t *qexp = nullptr;   // [q] 16-bit operand exponents: IP / COS keys are in the domain 2^(e_q + xexp)
  const float *rq = nullptr;       // [q] query residuals |q~ - q| (KEY_H16)
  int32_t xexp = 0;
  uint8_t *cert = nullptr;         // [q] out: 1 = the selection is certified exact
  double *sk = nullptr;            // [q] out: exact sort key of the k-th result (L2: -dist, IP / COS: score)
  int32_t *gcnt = nullptr;         // [q] out: zeroed (the exact fallback's per-group completion counters)
  unsigned long long *stats = nullptr;   // optional vrs_search_options.stats
  // the refine pass's finalize: row j of the lists is compacted query qmap[j] (its Q row, result
  // row and certificate); rows j >= *qcount return at once; rq = |q_lo|, rq2 = the residual after lo
  const int32_t *qmap = nullptr;
  const int32_t *qcount = nullptr;
  int32_t fold_qtiles = 0;         // the refine's finalize: level 0's query tiles (refine_fold)
  const float *rq2 = nullptr;
  int32_t *uncert_seen = nullptr;   // (mapped host flag) set to 1 when a level-0 certificate fails
  // (A/B and tests only, VRS_FIN_STAGE: the small-batch finalize stages at most this many
  // candidates (> 0), or skips its histogram selection for the radix select (< 0); 0 = default)
  int32_t stage_cap = 0;
};
cudaError_t launch_finalize(const FinalizeArgs &a, cudaStream_t s, int *launches);

// probe slot maxima -> per-query threshold: the kth largest of a query's values
// (each the key of a distinct row) bounds the kth best key over all rows from below
struct ThresholdArgs {
  const float *vals;       // [q][nvals]
  int32_t nvals;
  int64_t q;
  int32_t kth;
  uint32_t *gtau;          // [q] ordered-u32 out (0 = fewer than kth finite values)
  SplitInfo split;         // values [list][32] per query: only lists < kListsPerSplit * splits_used() are read
};
cudaError_t launch_threshold(const ThresholdArgs &a, cudaStream_t s);

// gemm_range.cu -- range (threshold) selection on the tensor-core pass
struct TcLaunch;   // tc_kernel.cuh
struct RangeState {
  TcLaunch *tc;            // from range_tc_alloc (tensor maps + parameters shared by the passes)
  double tau;              // the caller's threshold (score >= tau; squared L2 <= tau)
  KeyBound kb;             // the selection pass's key error bound constants
  uint32_t *gtau;          // [q] key thresholds (ordered u32)
  int32_t *cand_cnt;       // [2P][q] candidate counts
  int64_t *coff;           // [q * 2P + 1] candidate segment offsets, query-major; coff[q*2P] = C
  int32_t *cand;           // [C] candidate local row ids
  double *score;           // [C] exact scores
  uint8_t *keep;           // [C] 1 iff the exact score satisfies tau
  int32_t *kept;           // [q]
  int64_t *offsets;        // [q + 1] (the caller's) result offsets; offsets[q] = R
  int64_t *ids;            // [capacity] (the caller's)
  float *dists;
  int64_t row_offset;
};
TcLaunch *range_tc_alloc();
void range_tc_free(TcLaunch *t);
cudaError_t launch_range_count(const GemmArgs &a, const GemmPlan &plan, RangeState &r, cudaStream_t s, int *launches);
cudaError_t launch_range_fill(const GemmArgs &a, const GemmPlan &plan, RangeState &r, cudaStream_t s, int *launches);
cudaError_t launch_range_write(const GemmArgs &a, const GemmPlan &plan, RangeState &r, cudaStream_t s, int *launches);

// exact.cu -- the certificate's fallback: exact fp64 top-k of the queries whose
// selection was not certified (finalize wrote cert = 0), over every qualifying row.
struct ExactArgs {
  const uint8_t *cert;     // [q] from finalize
  const double *sk;        // [q] sort key of finalize's k-th result: rows below it cannot enter
  int32_t *gcnt;           // [q] group completion counters (zeroed by finalize)
  const float *X;
  int32_t d;
  int64_t n;
  const int32_t *ids;      // selection (nullptr: all n rows)
  const int64_t *count;
  const float *Q;
  int64_t q;
  int32_t metric;
  int32_t k;
  int64_t row_offset;
  double xmax;
  const float *nx2;        // the index's |x|^2 and 1/|x| (the fp32 filter keys)
  const float *inv_nx;
  int64_t *out_ids;        // [q][k] (overwritten for the uncertified queries)
  float *out_dists;
  double *slot_key;        // [items_max][qg][k]
  int64_t *slot_id;
  int32_t *slot_cnt;       // [items_max][qg]
  int32_t qg;              // queries per group (1, 2, 4, 8 or 16)
  unsigned long long *stats = nullptr;   // [3] += the queries recomputed here
};
int exact_group_size(int32_t d, int32_t k);
int64_t exact_items_max(int64_t q, int qg);
cudaError_t launch_exact(const ExactArgs &a, cudaStream_t s, int *launches);

// refine.cu -- the refine pass: the uncertified queries, compacted, re-selected
// with three 16-bit products per dot (q_hi.x_hi + q_hi.x_lo + q_lo.x_hi), then finalized again.
struct RefineArgs {
  const uint8_t *cert;     // [q] level-0 certificates
  const double *sk;        // [q] level-0 k-th sort keys
  const float *Q;
  int64_t q;
  int32_t d, dpad;         // dpad: d rounded up to whole 64-element K blocks
  int32_t metric;
  KeyBound kb;             // KEY_H16X3
  int32_t xexp;
  int64_t rows;            // rows of qr (whole 128-row tiles of q)
  int32_t *qlist;          // [q] out: compacted -> original query
  int32_t *ucount;         // [1] out: the number of uncertified queries
  uint16_t *qr;            // [rows x 2 dpad] out: fp16 [q_hi | q_lo] per compacted query
  int32_t *qexp;           // [q] out
  float *rqa, *rq2;        // [q] out: |q_lo|, |(q_hi + q_lo) 2^-e - q|
  uint32_t *gtau;          // [q] out: the refine pass's provable key threshold (ordered u32)
  int64_t gather_cap = 0;  // no xsel_lo: gathered (cp.async by id) iff N_sel <= this, else masked
  void *xsel_lo = nullptr; // [xsel_cap x d] x_lo rows of the level-0 selection: the refine delivers its rows
                           // like level 0 (X_sel copies + TMA, cp.async, or masked; the same device decision)
};
cudaError_t launch_refine(const RefineArgs &r, const GemmArgs &a, const GemmPlan &plan, void *gemm_scratch,
                          const void *x_lo, cudaStream_t s, int *launches);

struct MergeArgs {
  const int64_t *cand_ids;
  const float *cand_dists;
  int32_t parts;
  int64_t q;
  int32_t k;
  int32_t metric;
  int64_t *ids;
  float *dists;
};
cudaError_t launch_merge(const MergeArgs &a, cudaStream_t s, int *launches);

// the multi-GPU exchange + merge in one kernel over peer (symmetric) memory (finalize.cu)
constexpr int64_t kPushHeader = 256;   // bytes before the slots: uint32 counts[64]
constexpr int kPushMaxParts = 64;
inline int64_t push_buffer_bytes(int32_t parts, int64_t q, int32_t k) { return kPushHeader + 2 * (int64_t)parts * q * k * 12; }
struct PushMergeArgs {
  const int64_t *local_ids;   // this rank's exact results [q][k] (device)
  const float *local_dists;
  void *const *peer_bufs;     // device array [parts]: every rank's receive buffer (peer-mapped)
  int32_t parts, my_part;
  int64_t q;
  int32_t k, metric;
  uint32_t *state;            // this rank's device state [4]: epoch, ticket, pushes expected so far, timed-out flag
  int64_t *ids;               // merged [q][k]
  float *dists;
  uint64_t wait_ns;           // bound of the wait for the peers' pushes (state[3] = 1 when it expires)
};
cudaError_t launch_push_merge(const PushMergeArgs &a, cudaStream_t s, int *launches);

}  // namespace vrs
