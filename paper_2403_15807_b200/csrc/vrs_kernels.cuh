// vrs_kernels.cuh -- launch interfaces of the libvrs kernels (host side).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "vrs_internal.cuh"

namespace vrs {

// select.cu -- K4'/K5'
cudaError_t launch_select(const PredDev &pred, int64_t n, uint32_t *bitmap, int32_t *ids, int64_t *count,
                          void *scratch, cudaStream_t stream, int *launches);
size_t select_scratch_bytes(int64_t n);

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
struct GemmPlan {
  int32_t P;        // row splits = candidate lists per query
  int32_t qtiles;   // query tiles of 128
  int32_t ok;       // shape supported
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
  float *xsel;              // materialised-selection buffer [xsel_cap x d] (gathered mode)
  int64_t xsel_cap;
  const float *Q;
  int64_t q;
  const float *nx2;
  const float *inv_nx;
  int32_t metric;
  int32_t kprime;
  float *part_key;          // [P][q][kprime]
  int32_t *part_id;
  int32_t P;
};
size_t gemm_scratch_bytes(const GemmPlan &plan, int64_t q, int32_t kprime);
cudaError_t launch_gemm(const GemmArgs &a, const GemmPlan &plan, void *scratch, cudaStream_t s, int *launches);
void gemm_lists(const GemmArgs &a, const GemmPlan &plan, void *scratch, const float **key, const int32_t **id,
                int32_t *stride, int32_t *kread, int32_t *nlists, const float **list_tau);

// finalize.cu -- K7'/K12' merge + exact re-score; K10' shard merge
struct FinalizeArgs {
  const float *part_key;   // [P][q][kprime]
  const int32_t *part_id;
  int32_t P;
  int32_t kprime;          // entries selected for the exact re-score
  int32_t stride;          // list stride in entries
  int32_t kread;           // entries read per list (<= stride)
  int32_t sorted;          // lists sorted best-first with >= kprime entries (scan path)
  const float *list_tau;   // [P][q] per-list KP-th best key (-inf if unknown), or nullptr
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

struct ProbeArgs {
  const float *key;        // probe pass lists [lists][q][stride]
  const int32_t *id;
  int32_t lists;
  int32_t stride;
  int32_t kread;
  int64_t q;
  int32_t kp;
  uint32_t *gtau;          // [q] ordered-u32 shared thresholds (raised with atomicMax)
};
cudaError_t launch_probe_threshold(const ProbeArgs &a, cudaStream_t s);

struct SampleArgs {
  const float *dense;      // [q][ldd] raw keys of the sample pass (NaN / -inf = no row)
  int32_t ldd;
  int64_t q;
  int32_t kp;
  uint32_t *gtau;
};
cudaError_t launch_sample_threshold(const SampleArgs &a, cudaStream_t s);

struct RefineArgs {
  const float *key;        // main-pass lists [lists][q][cap]
  const int32_t *id;
  const int32_t *cnt;      // [lists][q] entries so far
  int32_t lists;
  int32_t cap;
  int64_t q;
  int32_t kp;
  uint32_t *gtau;
};
cudaError_t launch_refine_threshold(const RefineArgs &a, cudaStream_t s);

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
