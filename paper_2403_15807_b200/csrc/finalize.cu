// finalize.cu -- K7'/K12' cross-CTA merge + exact re-score, and K10' vrs_merge.
//
// finalize_kernel (one CTA per query): the per-(CTA, query) candidate lists
// written by the distance kernels (scan.cu, gemm_tc.cu) are reduced to the
// k' best by ranking key with a radix select (ties -> lower id), each of the
// k' rows is re-scored exactly (fp64 accumulation of the fp32 inputs, rounded
// once to fp32 -- DESIGN.md "Precision"), and the k best by exact score are
// written best-first with padding (reading R3).
//
// merge_kernel (one CTA per query): top-k of n_parts shard results by
// (dist, global id), the final step of the row-sharded search (north_star (4)).
#include <float.h>

#include "vrs_kernels.cuh"

namespace vrs {

constexpr int kFinThreads = 256;
constexpr int kFinMaxSel = 256;   // k' <= 256 (VRS_K_MAX + 16)
constexpr int kTieCap = 512;

// Exactly the m best (key desc, id asc) valid candidates -> out (unordered).
// get(c, &key, &id) returns false for padding.  Block-wide (kFinThreads).
template <typename IdT, typename Get>
__device__ int block_select_top(Get get, int64_t C, int m_want, IdT *out_id, float *out_key) {
  __shared__ uint32_t hist[256];
  __shared__ int s_n, s_out, s_ties, s_bin, s_above;
  __shared__ IdT s_tie[kTieCap];
  __shared__ IdT s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) { s_n = 0; s_out = 0; s_ties = 0; }
  __syncthreads();
  int local = 0;
  for (int64_t c = tid; c < C; c += kFinThreads) {
    float k; IdT i;
    local += get(c, k, i) ? 1 : 0;
  }
  atomicAdd(&s_n, local);
  __syncthreads();
  const int nvalid = s_n;
  if (nvalid <= m_want) {
    for (int64_t c = tid; c < C; c += kFinThreads) {
      float k; IdT i;
      if (get(c, k, i)) {
        const int p = atomicAdd(&s_out, 1);
        out_id[p] = i; out_key[p] = k;
      }
    }
    __syncthreads();
    return nvalid;
  }
  const int m = m_want;
  // radix select of the m-th largest ordered key, 8 bits per pass
  uint32_t prefix = 0, mask = 0;
  int rem = m;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = tid; b < 256; b += kFinThreads) hist[b] = 0;
    __syncthreads();
    for (int64_t c = tid; c < C; c += kFinThreads) {
      float k; IdT i;
      if (get(c, k, i)) {
        const uint32_t ok = ordered_u32(k);
        if ((ok & mask) == prefix) atomicAdd(&hist[(ok >> shift) & 255u], 1u);
      }
    }
    __syncthreads();
    if (warp == 0) {
      // lane l owns bins [255-8l-7, 255-8l] (descending); suffix sums from the top
      uint32_t v[8], s = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) { v[t] = hist[255 - 8 * lane - t]; s += v[t]; }
      uint32_t incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      uint32_t before = incl - s;  // count in bins above this lane's range
      const bool hit = before < (uint32_t)rem && (uint32_t)rem <= incl;
      if (hit) {
        uint32_t run = before;
        for (int t = 0; t < 8; ++t) {
          if ((uint32_t)rem <= run + v[t]) { s_bin = 255 - 8 * lane - t; s_above = (int)run; break; }
          run += v[t];
        }
      }
    }
    __syncthreads();
    prefix |= (uint32_t)s_bin << shift;
    mask |= 255u << shift;
    rem -= s_above;
    __syncthreads();
  }
  // strictly better keys are all in; `rem` of the ties at `prefix` go by lowest id
  for (int64_t c = tid; c < C; c += kFinThreads) {
    float k; IdT i;
    if (get(c, k, i)) {
      const uint32_t ok = ordered_u32(k);
      if (ok > prefix) {
        const int p = atomicAdd(&s_out, 1);
        out_id[p] = i; out_key[p] = k;
      } else if (ok == prefix) {
        const int p = atomicAdd(&s_ties, 1);
        if (p < kTieCap) s_tie[p] = i;
      }
    }
  }
  __syncthreads();
  const int gt = s_out;
  const float tkey = [&] { uint32_t u = (prefix & 0x80000000u) ? (prefix & 0x7fffffffu) : ~prefix; return __uint_as_float(u); }();
  if (s_ties <= kTieCap) {
    if (tid == 0) {  // few ties in practice: simple selection by id
      const int nt = s_ties;
      for (int r = 0; r < rem; ++r) {
        int best = r;
        for (int t = r + 1; t < nt; ++t) if (s_tie[t] < s_tie[best]) best = t;
        IdT tmp = s_tie[r]; s_tie[r] = s_tie[best]; s_tie[best] = tmp;
        out_id[gt + r] = s_tie[r]; out_key[gt + r] = tkey;
      }
    }
  } else {
    // many exact ties: repeated block-wide minimum over ids above the last taken
    if (tid == 0) s_last = (IdT)-1;
    __syncthreads();
    for (int r = 0; r < rem; ++r) {
      IdT best = (IdT)0x7fffffffffffffffLL;
      if (sizeof(IdT) == 4) best = (IdT)0x7fffffff;
      for (int64_t c = tid; c < C; c += kFinThreads) {
        float k; IdT i;
        if (get(c, k, i) && ordered_u32(k) == prefix && i > s_last && i < best) best = i;
      }
      __shared__ IdT s_red[kFinThreads / 32];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        IdT y = __shfl_xor_sync(0xffffffffu, best, o);
        best = y < best ? y : best;
      }
      if (lane == 0) s_red[warp] = best;
      __syncthreads();
      if (tid == 0) {
        IdT b = s_red[0];
        for (int w = 1; w < kFinThreads / 32; ++w) b = s_red[w] < b ? s_red[w] : b;
        out_id[gt + r] = b; out_key[gt + r] = tkey; s_last = b;
      }
      __syncthreads();
    }
  }
  __syncthreads();
  return m;
}

// Warp bitonic sort of n = 2^p (double key, int64 id) pairs: key desc, id asc.
__device__ void warp_sort_desc_d(double *key, int64_t *id, int n) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= n; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncwarp();
      for (int t = lane; t < (n >> 1); t += 32) {
        const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const double ka = key[lo], kb = key[hi];
        const int64_t ia = id[lo], ib = id[hi];
        const bool b_better = (kb > ka) || (kb == ka && ib < ia);
        const bool a_better = (ka > kb) || (ka == kb && ia < ib);
        if (desc ? b_better : a_better) { key[lo] = kb; key[hi] = ka; id[lo] = ib; id[hi] = ia; }
      }
    }
  __syncwarp();
}


constexpr int kFinMaxStage = 3072;   // candidates staged in shared memory after pruning

__global__ void __launch_bounds__(kFinThreads) finalize_kernel(FinalizeArgs a) {
  __shared__ int32_t s_id[kFinMaxSel];
  __shared__ float s_key[kFinMaxSel];
  __shared__ double s_score[kFinMaxSel];
  __shared__ int64_t s_sid[kFinMaxSel];
  __shared__ double s_nq;
  __shared__ float s_ck[kFinMaxStage];
  __shared__ int32_t s_ci[kFinMaxStage];
  __shared__ float s_red[kFinThreads / 32];
  __shared__ int s_nc;
  const int64_t j = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float *q = a.Q + j * a.d;

  // 1. a provable lower bound T0 of the k'-th best key: every list holding >= k'
  //    entries at or above its own k'-th (scan: sorted lists) / KP-th (tensor
  //    path: list_tau) best key bounds the union's k'-th best from below
  float t0 = -INFINITY;
  for (int l = tid; l < a.P; l += kFinThreads) {
    if (a.list_tau) {
      t0 = fmaxf(t0, a.list_tau[(int64_t)l * a.q + j]);
    } else if (a.sorted) {
      const int64_t o = ((int64_t)l * a.q + j) * a.stride + (a.kprime - 1);
      if (a.part_id[o] >= 0) t0 = fmaxf(t0, a.part_key[o]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t0 = fmaxf(t0, __shfl_xor_sync(0xffffffffu, t0, o));
  if (lane == 0) s_red[warp] = t0;
  if (tid == 0) s_nc = 0;
  __syncthreads();
  t0 = s_red[0];
#pragma unroll
  for (int w = 1; w < kFinThreads / 32; ++w) t0 = fmaxf(t0, s_red[w]);

  // 2. stage the candidates >= T0 in shared memory (one pass over the lists)
  const int64_t C = (int64_t)a.P * a.kread;
  for (int64_t c0 = 0; c0 < C; c0 += kFinThreads) {
    const int64_t c = c0 + tid;
    float key = -INFINITY;
    int32_t id = -1;
    if (c < C) {
      const int64_t p = c / a.kread, r = c - p * a.kread;
      const int64_t o = (p * a.q + j) * a.stride + r;
      id = a.part_id[o];
      key = a.part_key[o];
    }
    const bool keep = id >= 0 && key >= t0;
    const uint32_t m = __ballot_sync(0xffffffffu, keep);
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(&s_nc, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (keep) {
      const int pos = base + __popc(m & lanemask_lt());
      if (pos < kFinMaxStage) { s_ck[pos] = key; s_ci[pos] = id; }
    }
  }
  __syncthreads();
  const int nc = s_nc;
  int m;
  if (nc <= kFinMaxStage) {
    auto get_s = [&](int64_t c, float &key, int32_t &id) -> bool {
      key = s_ck[c];
      id = s_ci[c];
      return true;
    };
    m = block_select_top<int32_t>(get_s, nc, a.kprime, s_id, s_key);
  } else {
    auto get = [&](int64_t c, float &key, int32_t &id) -> bool {
      const int64_t p = c / a.kread, r = c - p * a.kread;
      const int64_t o = (p * a.q + j) * a.stride + r;
      id = a.part_id[o];
      key = a.part_key[o];
      return id >= 0 && key >= t0;
    };
    m = block_select_top<int32_t>(get, C, a.kprime, s_id, s_key);
  }

  // |q|^2 in fp64 (COSINE only)
  if (warp == 0) {
    double s = 0.0;
    if (a.metric == VRS_COSINE)
      for (int t = lane; t < a.d; t += 32) s += (double)q[t] * (double)q[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) s_nq = s;
  }
  __syncthreads();
  const bool zero_cos = (a.metric == VRS_COSINE) && !(s_nq > 0.0);

  // exact re-score, one warp per candidate
  for (int c = warp; c < m; c += kFinThreads / 32) {
    const float *x = a.X + (int64_t)s_id[c] * a.d;
    double s = 0.0, xx = 0.0;
    if (a.metric == VRS_L2) {
      for (int t = lane; t < a.d; t += 32) { const double df = (double)q[t] - (double)x[t]; s += df * df; }
    } else {
      for (int t = lane; t < a.d; t += 32) {
        const double xv = (double)x[t];
        s += (double)q[t] * xv;
        xx += xv * xv;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      xx += __shfl_xor_sync(0xffffffffu, xx, o);
    }
    if (lane == 0) {
      double sc = s;
      if (a.metric == VRS_COSINE) sc = s / (sqrt(s_nq) * sqrt(xx));
      s_score[c] = (a.metric == VRS_L2) ? -sc : sc;  // sort key: larger is better
      s_sid[c] = s_id[c];
    }
  }
  __syncthreads();
  int np = 1;
  while (np < m) np <<= 1;
  for (int c = m + tid; c < np; c += kFinThreads) { s_score[c] = -INFINITY; s_sid[c] = INT64_MAX; }
  __syncthreads();
  if (warp == 0 && m > 1) warp_sort_desc_d(s_score, s_sid, np);
  __syncthreads();
  const int mv = zero_cos ? 0 : min(m, a.k);
  const float pad = a.metric == VRS_L2 ? INFINITY : -INFINITY;
  for (int r = tid; r < a.k; r += kFinThreads) {
    const int64_t o = j * a.k + r;
    if (r < mv) {
      a.ids[o] = a.row_offset + s_sid[r];
      const double sc = s_score[r];
      a.dists[o] = (float)(a.metric == VRS_L2 ? -sc : sc);
    } else {
      a.ids[o] = -1;
      a.dists[o] = pad;
    }
  }
}

// ---------------------------------------------------------- probe threshold
// Per query: the kp-th best key among the probe pass's lists (a subset of the
// rows) -- a provable lower bound of the kp-th best over all rows -- raises the
// query's shared threshold for the main pass (gemm_tc.cu).
__global__ void __launch_bounds__(kFinThreads) probe_threshold_kernel(ProbeArgs a) {
  __shared__ int32_t s_id[kFinMaxSel];
  __shared__ float s_key[kFinMaxSel];
  __shared__ float s_red[kFinThreads / 32];
  const int64_t j = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto get = [&](int64_t c, float &key, int32_t &id) -> bool {
    const int64_t p = c / a.kread, r = c - p * a.kread;
    const int64_t o = (p * a.q + j) * a.stride + r;
    id = a.id[o];
    key = a.key[o];
    return id >= 0;
  };
  const int m = block_select_top<int32_t>(get, (int64_t)a.lists * a.kread, a.kp, s_id, s_key);
  if (m < a.kp) return;   // fewer than kp candidates sampled: no bound
  float mn = INFINITY;
  for (int i = tid; i < m; i += kFinThreads) mn = fminf(mn, s_key[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if (lane == 0) s_red[warp] = mn;
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kFinThreads / 32; ++w) mn = fminf(mn, s_red[w]);
    mn = fminf(mn, s_red[0]);
    atomicMax(a.gtau + j, ordered_u32(mn));
  }
}

constexpr int kSampleMax = 4096;   // sample keys per query (SAMPLE_TILES x 256 in gemm_tc.cu)

// Per query: the kp-th best raw key of the sample pass (-inf / NaN = no row).
__global__ void __launch_bounds__(kFinThreads) sample_threshold_kernel(SampleArgs a) {
  __shared__ int32_t s_id[kFinMaxSel];
  __shared__ float s_key[kFinMaxSel];
  __shared__ float s_red[kFinThreads / 32];
  const int64_t j = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ float s_row[kSampleMax];
  const float *row = a.dense + j * a.ldd;
  for (int c = tid; c < a.ldd; c += kFinThreads) s_row[c] = row[c];   // one coalesced pass
  __syncthreads();
  auto get = [&](int64_t c, float &key, int32_t &id) -> bool {
    key = s_row[c];
    id = (int32_t)c;
    return key > -INFINITY;   // false for -inf padding and NaN fill
  };
  const int m = block_select_top<int32_t>(get, a.ldd, a.kp, s_id, s_key);
  if (m < a.kp) return;
  float mn = INFINITY;
  for (int i = tid; i < m; i += kFinThreads) mn = fminf(mn, s_key[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if (lane == 0) s_red[warp] = mn;
  __syncthreads();
  if (tid == 0) {
    for (int w = 0; w < kFinThreads / 32; ++w) mn = fminf(mn, s_red[w]);
    atomicMax(a.gtau + j, ordered_u32(mn));
  }
}

cudaError_t launch_sample_threshold(const SampleArgs &a, cudaStream_t s) {
  sample_threshold_kernel<<<(unsigned)a.q, kFinThreads, 0, s>>>(a);
  return cudaGetLastError();
}

// Per query: the kp-th best key over every list's entries so far (part 1 of the
// main pass) -- a lower bound of the final kp-th best -- raises the shared threshold.
__global__ void __launch_bounds__(kFinThreads) refine_threshold_kernel(RefineArgs a) {
  __shared__ int32_t s_id[kFinMaxSel];
  __shared__ float s_key[kFinMaxSel];
  __shared__ float s_red[kFinThreads / 32];
  const int64_t j = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto get = [&](int64_t c, float &key, int32_t &id) -> bool {
    const int64_t l = c / a.cap, r = c - l * a.cap;
    if (r >= a.cnt[l * a.q + j]) return false;
    const int64_t o = (l * a.q + j) * a.cap + r;
    id = a.id[o];
    key = a.key[o];
    return true;
  };
  const int m = block_select_top<int32_t>(get, (int64_t)a.lists * a.cap, a.kp, s_id, s_key);
  if (m < a.kp) return;
  float mn = INFINITY;
  for (int i = tid; i < m; i += kFinThreads) mn = fminf(mn, s_key[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if (lane == 0) s_red[warp] = mn;
  __syncthreads();
  if (tid == 0) {
    for (int w = 0; w < kFinThreads / 32; ++w) mn = fminf(mn, s_red[w]);
    atomicMax(a.gtau + j, ordered_u32(mn));
  }
}

cudaError_t launch_refine_threshold(const RefineArgs &a, cudaStream_t s) {
  refine_threshold_kernel<<<(unsigned)a.q, kFinThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_probe_threshold(const ProbeArgs &a, cudaStream_t s) {
  probe_threshold_kernel<<<(unsigned)a.q, kFinThreads, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const FinalizeArgs &a, cudaStream_t s, int *launches) {
  if (launches) *launches += 1;
  finalize_kernel<<<(unsigned)a.q, kFinThreads, 0, s>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K10' merge

__global__ void __launch_bounds__(kFinThreads) merge_kernel(MergeArgs a) {
  __shared__ int64_t s_id[kFinMaxSel];
  __shared__ float s_key[kFinMaxSel];
  __shared__ double s_k2[kFinMaxSel];
  __shared__ int64_t s_i2[kFinMaxSel];
  const int64_t j = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5;
  auto get = [&](int64_t c, float &key, int64_t &id) -> bool {
    const int64_t p = c / a.k, r = c - p * a.k;
    const int64_t o = (p * a.q + j) * a.k + r;
    id = a.cand_ids[o];
    const float dv = a.cand_dists[o];
    key = a.metric == VRS_L2 ? -dv : dv;
    return id >= 0;
  };
  const int m = block_select_top<int64_t>(get, (int64_t)a.parts * a.k, a.k, s_id, s_key);
  int np = 1;
  while (np < m) np <<= 1;
  for (int c = tid; c < np; c += kFinThreads) {
    s_k2[c] = c < m ? (double)s_key[c] : -INFINITY;
    s_i2[c] = c < m ? s_id[c] : INT64_MAX;
  }
  __syncthreads();
  if (warp == 0 && m > 1) warp_sort_desc_d(s_k2, s_i2, np);
  __syncthreads();
  const float pad = a.metric == VRS_L2 ? INFINITY : -INFINITY;
  for (int r = tid; r < a.k; r += kFinThreads) {
    const int64_t o = j * a.k + r;
    if (r < m) {
      a.ids[o] = s_i2[r];
      const float kv = (float)s_k2[r];
      a.dists[o] = a.metric == VRS_L2 ? -kv : kv;
    } else {
      a.ids[o] = -1;
      a.dists[o] = pad;
    }
  }
}

cudaError_t launch_merge(const MergeArgs &a, cudaStream_t s, int *launches) {
  if (launches) *launches += 1;
  merge_kernel<<<(unsigned)a.q, kFinThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace vrs
