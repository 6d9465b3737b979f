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

// select.cu -- K4'/K5'.  Optional work folded into the count kernel (saves a
// launch on the tensor-core path): the bf16 conversion of the queries.  (Folding
// the row gather into the 1-CTA-per-8192-rows scatter kernel was measured slower
// than the separate gather_copy_kernel.)
struct SelectFuse {
  const float *q_in;       // fp32 queries (nullptr: no conversion)
  void *q_out;             // bf16 [q_total]: q_count converted values, zero padding after
  int64_t q_count, q_total;
};
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
cudaError_t launch_norms(const float *X, int64_t n, int32_t d, float *nx2, float *inv_nx, int32_t *zero_flag,
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
GemmPlan gemm_plan(int64_t q, int32_t d, int64_t n_upper, int32_t kprime, int num_sms);

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
  int32_t bf16;             // select on the bf16 shadow (kind::f16) instead of fp32 (kind::tf32)
  const void *Xb;           // bf16 shadow corpus [n x d] (bf16 only)
  void *Qb;                 // scratch [q x d] bf16 queries (bf16 only)
  int32_t prepped;          // 1: the select kernels already converted the queries
  // launch_select_local's output (nullptr: ids / count were written by launch_select):
  // the tensor-core pass first runs select_finish -> count, dense ids, gathered rows
  const int32_t *ids_local = nullptr;
  const uint32_t *chunk_count = nullptr;
};
size_t gemm_scratch_bytes(const GemmPlan &plan, int64_t q, int32_t kprime);
cudaError_t launch_to_bf16(const float *in, void *out, int64_t count, int64_t total, cudaStream_t s);
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
  double xmax;             // max row norm of the index
  double gamma;            // tensor-core product error bound / (|q| |x|)
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

}  // namespace vrs
