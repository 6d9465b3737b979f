// finalize.cu -- K7'/K12' cross-CTA merge + exact re-score, and K10' vrs_merge.
//
// finalize_kernel (one warp per query): the per-(CTA, query) candidate lists
// written by the distance kernels (scan.cu, gemm_tc.cu) are reduced to the
// k' best by ranking key with a radix select (ties -> lower id), each of the
// k' rows is re-scored exactly (fp64 accumulation of the fp32 inputs, rounded
// once to fp32 -- DESIGN.md "Precision"), and the k best by exact score are
// written best-first with padding (reading R3).
//
// threshold_kernel (one warp per query): the k'-th largest probe slot maximum
// of the tensor-core path -> the shared threshold of the main pass.
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
template <typename IdT, int NT = kFinThreads, typename Get>
__device__ int block_select_top(Get get, int64_t C, int m_want, IdT *out_id, float *out_key) {
  __shared__ uint32_t hist[256];
  __shared__ int s_n, s_out, s_ties, s_bin, s_above;
  __shared__ IdT s_tie[kTieCap];
  __shared__ IdT s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) { s_n = 0; s_out = 0; s_ties = 0; }
  __syncthreads();
  int local = 0;
  for (int64_t c = tid; c < C; c += NT) {
    float k; IdT i;
    local += get(c, k, i) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if (lane == 0) atomicAdd(&s_n, local);
  __syncthreads();
  const int nvalid = s_n;
  if (nvalid <= m_want) {
    for (int64_t c = tid; c < C; c += NT) {
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
    for (int b = tid; b < 256; b += NT) hist[b] = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < C; c0 += NT) {
      const int64_t c = c0 + tid;
      float k; IdT i;
      uint32_t bin = 256u;
      if (c < C && get(c, k, i)) {
        const uint32_t ok = ordered_u32(k);
        if ((ok & mask) == prefix) bin = (ok >> shift) & 255u;
      }
      hist_add_warp(hist, bin);
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
  for (int64_t c = tid; c < C; c += NT) {
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
      for (int64_t c = tid; c < C; c += NT) {
        float k; IdT i;
        if (get(c, k, i) && ordered_u32(k) == prefix && i > s_last && i < best) best = i;
      }
      __shared__ IdT s_red[NT / 32];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        IdT y = __shfl_xor_sync(0xffffffffu, best, o);
        best = y < best ? y : best;
      }
      if (lane == 0) s_red[warp] = best;
      __syncthreads();
      if (tid == 0) {
        IdT b = s_red[0];
        for (int w = 1; w < NT / 32; ++w) b = s_red[w] < b ? s_red[w] : b;
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


// ------------------------------------------------------ warp-level selection
constexpr int kBufCap = 512;     // per-warp candidate buffer (>= 2 k' for every k' <= 256)

// The K-th largest of the u32 values get(i, u) (i < n, only those for which get
// returns true), by a warp-cooperative radix select (8 bits per pass, histogram
// in shared memory).  *above = how many values are strictly larger; returns
// false (and *above = the number of values) when there are fewer than K.
template <typename Get>
__device__ bool warp_kth_largest(Get get, int n, int K, uint32_t *hist, uint32_t *out, int *above_out) {
  const int lane = threadIdx.x & 31;
  uint32_t prefix = 0, mask = 0;
  int rem = K, above_total = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = lane; b < 256; b += 32) hist[b] = 0;
    __syncwarp();
#pragma unroll 4
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + lane;
      uint32_t u, bin = 256u;
      if (i < n && get(i, u) && (u & mask) == prefix) bin = (u >> shift) & 255u;
      hist_add_warp(hist, bin);
    }
    __syncwarp();
    // lane l owns bins [255-8l-7, 255-8l] (descending); suffix sums from the top
    uint32_t v[8], s = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) { v[t] = hist[255 - 8 * lane - t]; s += v[t]; }
    uint32_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (total < (uint32_t)rem) {   // only on the first pass: fewer than K values
      *above_out = (int)total;
      return false;
    }
    const uint32_t before = incl - s;
    int bin = -1, above = 0;
    if (before < (uint32_t)rem && (uint32_t)rem <= incl) {
      uint32_t run = before;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        if (bin < 0 && (uint32_t)rem <= run + v[t]) { bin = 255 - 8 * lane - t; above = (int)run; }
        if (bin < 0) run += v[t];
      }
    }
    const int src = __ffs(__ballot_sync(0xffffffffu, bin >= 0)) - 1;
    bin = __shfl_sync(0xffffffffu, bin, src);
    above = __shfl_sync(0xffffffffu, above, src);
    prefix |= (uint32_t)bin << shift;
    mask |= 255u << shift;
    rem -= above;
    above_total += above;
    __syncwarp();
  }
  *out = prefix;
  *above_out = above_total;
  return true;
}

// Keep exactly the K best of the warp's buffer (key desc, then id asc), in place
// (requires n >= K).  Returns the ordered key of the K-th best.
__device__ __noinline__ uint32_t warp_keep_best(float *bk, int32_t *bi, int &n, int K, uint32_t *hist) {
  const int lane = threadIdx.x & 31;
  uint32_t v = 0, idv = 0xffffffffu;
  int above = 0;
  warp_kth_largest([&](int i, uint32_t &u) { u = ordered_u32(bk[i]); return true; }, n, K, hist, &v, &above);
  // ties at v: keep the (K - above) smallest ids (row ids are unique per query)
  int ties = 0;
  for (int i = lane; i < n; i += 32) ties += ordered_u32(bk[i]) == v ? 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ties += __shfl_xor_sync(0xffffffffu, ties, o);
  if (ties > K - above) {
    uint32_t x = 0;
    int ab2 = 0;
    warp_kth_largest([&](int i, uint32_t &u) { u = ~(uint32_t)bi[i]; return ordered_u32(bk[i]) == v; }, n, K - above,
                     hist, &x, &ab2);
    idv = ~x;
  }
  int out = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    float kv = 0.f;
    int32_t iv = 0;
    bool keep = false;
    if (i < n) {
      kv = bk[i];
      iv = bi[i];
      const uint32_t ok = ordered_u32(kv);
      keep = ok > v || (ok == v && (uint32_t)iv <= idv);
    }
    const uint32_t km = __ballot_sync(0xffffffffu, keep);
    const int pos = out + __popc(km & lanemask_lt());
    __syncwarp();
    if (keep) { bk[pos] = kv; bi[pos] = iv; }
    out += __popc(km);
    __syncwarp();
  }
  n = out;
  return v;
}

// Bitonic sort of 64 (key, id) pairs, two per lane (element lane and lane + 32):
// best first (key descending, then id ascending).
__device__ __forceinline__ bool pair_first(float ka, int32_t ia, float kb, int32_t ib) {
  return ka > kb || (ka == kb && ia < ib);
}
__device__ __forceinline__ void warp_reg_sort64(float &ka, int32_t &ia, float &kb, int32_t &ib) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      if (jj == 32) {   // partners are the lane's two elements; k == 64: one ascending block
        if (pair_first(kb, ib, ka, ia)) {
          const float tk = ka; ka = kb; kb = tk;
          const int32_t ti = ia; ia = ib; ib = ti;
        }
        continue;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float &key = h ? kb : ka;
        int32_t &id = h ? ib : ia;
        const int i = lane + 32 * h;
        const float pk = __shfl_xor_sync(0xffffffffu, key, jj);
        const int32_t pid = __shfl_xor_sync(0xffffffffu, id, jj);
        const bool partner_first = pair_first(pk, pid, key, id);
        const bool keep_first = ((i & k) == 0) == ((i & jj) == 0);
        if (keep_first == partner_first) { key = pk; id = pid; }
      }
    }
  }
}

// ---- register bitonic networks over 32 * E (key, id) pairs, E per lane ----------
// Element e = h * 32 + lane sits in slot h of lane `lane`.  Order: best first
// (key descending, then id ascending).
template <int E>
__device__ __forceinline__ void warp_cmpx_e(float (&k)[E], int32_t (&id)[E], int kk, int jj) {
  const int lane = threadIdx.x & 31;
  if (jj >= 32) {   // partners in the same lane
    const int hj = jj >> 5;
#pragma unroll
    for (int h = 0; h < E; ++h) {
      if (h & hj) continue;
      const int hi = h | hj;
      const bool lo_first = ((h * 32 + lane) & kk) == 0;   // the lower element takes the better
      if (pair_first(k[hi], id[hi], k[h], id[h]) == lo_first) {
        const float tk = k[h]; k[h] = k[hi]; k[hi] = tk;
        const int32_t ti = id[h]; id[h] = id[hi]; id[hi] = ti;
      }
    }
  } else {
#pragma unroll
    for (int h = 0; h < E; ++h) {
      const int i = h * 32 + lane;
      const float pk = __shfl_xor_sync(0xffffffffu, k[h], jj);
      const int32_t pid = __shfl_xor_sync(0xffffffffu, id[h], jj);
      const bool keep_first = ((i & kk) == 0) == ((i & jj) == 0);
      if (keep_first == pair_first(pk, pid, k[h], id[h])) { k[h] = pk; id[h] = pid; }
    }
  }
}
// Full sort.
template <int E>
__device__ __forceinline__ void warp_sort_e(float (&k)[E], int32_t (&id)[E]) {
#pragma unroll
  for (int kk = 2; kk <= 32 * E; kk <<= 1)
#pragma unroll
    for (int jj = kk >> 1; jj > 0; jj >>= 1) warp_cmpx_e<E>(k, id, kk, jj);
}
// Sort of a bitonic sequence (the last stage of the network).
template <int E>
__device__ __forceinline__ void warp_merge_e(float (&k)[E], int32_t (&id)[E]) {
#pragma unroll
  for (int jj = 16 * E; jj > 0; jj >>= 1) warp_cmpx_e<E>(k, id, 32 * E, jj);
}
// Best 32E of two sorted 32E-lists: mine (registers) and other (smem, element e at
// ok[e] / oi[e]): the better of mine[e] and other[32E-1-e] is bitonic, then merged.
template <int E>
__device__ __forceinline__ void warp_merge_with_e(float (&k)[E], int32_t (&id)[E], const float *ok, const int32_t *oi) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int h = 0; h < E; ++h) {
    const int e = 32 * E - 1 - (h * 32 + lane);
    const float pk = ok[e];
    const int32_t pid = oi[e];
    if (pair_first(pk, pid, k[h], id[h])) { k[h] = pk; id[h] = pid; }
  }
  warp_merge_e<E>(k, id);
}
// Insert f into the descending per-lane list t[0] >= t[1] >= ... (keys only).
template <int E>
__device__ __forceinline__ void top_insert_e(float (&t)[E], float f) {
#pragma unroll
  for (int h = E - 1; h > 0; --h) t[h] = fmaxf(t[h], fminf(t[h - 1], f));
  t[0] = fmaxf(t[0], f);
}
template <int E>
__device__ __forceinline__ float elem_e(const float (&k)[E], int e) {   // element e (warp-uniform e)
  float v = k[0];
#pragma unroll
  for (int h = 1; h < E; ++h) if ((e >> 5) == h) v = k[h];
  return __shfl_sync(0xffffffffu, v, e & 31);
}

// Keep exactly the K best of the warp's buffer (K <= 128), usually in one
// histogram pass: keys bucketed linearly over [min, max] (a monotone map), the
// bucket holding the K-th best found from the top, every entry from that bucket
// up collected (<= 32E of them in the common case, E = 2 for K <= 64, else 4) and
// sorted in registers.  Falls back to the radix select when the collected set is
// larger (ties, spikes).
template <int E>
__device__ __noinline__ uint32_t warp_keep_best_fast_e(float *bk, int32_t *bi, int &n, int K, uint32_t *hist) {
  const int lane = threadIdx.x & 31;
  float lo = INFINITY, hi = -INFINITY;
  for (int i = lane; i < n; i += 32) { lo = fminf(lo, bk[i]); hi = fmaxf(hi, bk[i]); }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const float range = hi - lo;
  if (!(range > 0.f) || !(range < INFINITY)) return warp_keep_best(bk, bi, n, K, hist);
  const float scale = 255.5f / range;
  auto bucket = [&](float key) { return (uint32_t)min(255, (int)((key - lo) * scale)); };
  for (int b = lane; b < 256; b += 32) hist[b] = 0;
  __syncwarp();
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    hist_add_warp(hist, i < n ? bucket(bk[i]) : 256u);
  }
  __syncwarp();
  // lane l owns buckets [255-8l-7, 255-8l]; find the bucket where the count from the top reaches K
  uint32_t v[8], sum = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) { v[t] = hist[255 - 8 * lane - t]; sum += v[t]; }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int bstar = -1, upto = 0;   // upto: entries in buckets >= bstar
  const uint32_t before = incl - sum;
  if (before < (uint32_t)K && (uint32_t)K <= incl) {
    uint32_t run = before;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (bstar < 0 && (uint32_t)K <= run + v[t]) { bstar = 255 - 8 * lane - t; upto = (int)(run + v[t]); }
      if (bstar < 0) run += v[t];
    }
  }
  const int src = __ffs(__ballot_sync(0xffffffffu, bstar >= 0)) - 1;
  bstar = __shfl_sync(0xffffffffu, bstar, src);
  upto = __shfl_sync(0xffffffffu, upto, src);
  if (upto > 32 * E) return warp_keep_best(bk, bi, n, K, hist);
  // collect the candidates from bucket bstar up into the (no longer needed)
  // histogram space (32E keys, 32E ids <= 256 words), then E per lane into registers
  float *ck = reinterpret_cast<float *>(hist);
  int32_t *ci = reinterpret_cast<int32_t *>(hist + 32 * E);
  __syncwarp();
  int got = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const bool take = i < n && (int)bucket(bk[i]) >= bstar;
    const uint32_t m = __ballot_sync(0xffffffffu, take);
    if (take) {
      const int pos = got + __popc(m & lanemask_lt());
      ck[pos] = bk[i];
      ci[pos] = bi[i];
    }
    got += __popc(m);
  }
  __syncwarp();
  float kk[E];
  int32_t ii[E];
#pragma unroll
  for (int h = 0; h < E; ++h) {
    const int e = h * 32 + lane;
    kk[h] = e < got ? ck[e] : -INFINITY;
    ii[h] = e < got ? ci[e] : INT32_MAX;
  }
  warp_sort_e<E>(kk, ii);
  // the K best: elements 0..K-1
  __syncwarp();
#pragma unroll
  for (int h = 0; h < E; ++h) {
    const int e = h * 32 + lane;
    if (e < K) { bk[e] = kk[h]; bi[e] = ii[h]; }
  }
  __syncwarp();
  n = K;
  return ordered_u32(elem_e<E>(kk, K - 1));
}
// (collection capacity 32E >= 2K, else the K-th best's bucket would almost never fit
// and every compaction would take the radix path; E = 8 collects 2 x 256 words, so it
// needs a 512-word histogram area)
template <int HIST>
__device__ __forceinline__ uint32_t warp_keep_best_fast(float *bk, int32_t *bi, int &n, int K, uint32_t *hist) {
  if (K <= 32) return warp_keep_best_fast_e<2>(bk, bi, n, K, hist);
  if (K <= 64) return warp_keep_best_fast_e<4>(bk, bi, n, K, hist);
  if (HIST >= 512 && K <= 128) return warp_keep_best_fast_e<8>(bk, bi, n, K, hist);
  return warp_keep_best(bk, bi, n, K, hist);
}

// The K-th largest (K <= 64) of the nonzero ordered-u32 values v[0..n) (0 = no
// value), warp-cooperative, usually in one histogram pass: values bucketed
// linearly over [min, max] (monotone), the bucket holding the K-th largest found
// from the top, everything from it up (<= 64) sorted in registers.  Falls back
// to the radix select.  Returns false when fewer than K values exist.
__device__ bool warp_kth_value_fast(const uint32_t *v, int n, int K, uint32_t *hist, uint32_t *out) {
  const int lane = threadIdx.x & 31;
  auto radix = [&]() {
    int above = 0;
    return warp_kth_largest([&](int i, uint32_t &u) { u = v[i]; return u != 0u; }, n, K, hist, out, &above);
  };
  if (K > 64) return radix();
  uint32_t lo = 0xffffffffu, hi = 0u;
  int cnt = 0;
  for (int i = lane; i < n; i += 32) {
    const uint32_t u = v[i];
    if (u) { lo = min(lo, u); hi = max(hi, u); ++cnt; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if (cnt < K) return false;
  if (hi == lo) { *out = hi; return true; }
  const float scale = 255.5f / (float)(hi - lo);
  auto bucket = [&](uint32_t u) { return (uint32_t)min(255, (int)((float)(u - lo) * scale)); };
  for (int b = lane; b < 256; b += 32) hist[b] = 0;
  __syncwarp();
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const uint32_t u = i < n ? v[i] : 0u;
    hist_add_warp(hist, u ? bucket(u) : 256u);
  }
  __syncwarp();
  uint32_t c[8], sum = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t] = hist[255 - 8 * lane - t]; sum += c[t]; }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int bstar = -1, upto = 0;
  const uint32_t before = incl - sum;
  if (before < (uint32_t)K && (uint32_t)K <= incl) {
    uint32_t run = before;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (bstar < 0 && (uint32_t)K <= run + c[t]) { bstar = 255 - 8 * lane - t; upto = (int)(run + c[t]); }
      if (bstar < 0) run += c[t];
    }
  }
  const int src = __ffs(__ballot_sync(0xffffffffu, bstar >= 0)) - 1;
  bstar = __shfl_sync(0xffffffffu, bstar, src);
  upto = __shfl_sync(0xffffffffu, upto, src);
  if (upto > 64) return radix();
  __syncwarp();
  uint32_t *cv = hist;   // reuse: the collected values
  int got = 0;
  for (int i0 = 0; i0 < n; i0 += 32) {
    const int i = i0 + lane;
    const uint32_t u = i < n ? v[i] : 0u;
    const bool take = u != 0u && (int)bucket(u) >= bstar;
    const uint32_t m = __ballot_sync(0xffffffffu, take);
    if (take) cv[got + __popc(m & lanemask_lt())] = u;
    got += __popc(m);
  }
  __syncwarp();
  // ordered u32 -> float keys for the shared register sort (ids: position, irrelevant)
  auto to_f = [](uint32_t o) { return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o); };
  float ka = lane < got ? to_f(cv[lane]) : -INFINITY, kb = lane + 32 < got ? to_f(cv[lane + 32]) : -INFINITY;
  int32_t ia = lane, ib = lane + 32;
  warp_reg_sort64(ka, ia, kb, ib);
  const float kth = __shfl_sync(0xffffffffu, K - 1 < 32 ? ka : kb, (K - 1) & 31);
  *out = ordered_u32(kth);
  return true;
}

// ------------------------------------------------------------------ finalize
// Per query: (1) a provable lower bound of the k'-th best ranking key (the
// shared probe threshold, or for sorted scan lists the best of their k'-th
// entries); (2) stream every list entry at or above it into a shared-memory
// buffer, compacting to the k' best by radix select whenever it fills; (3) keep
// exactly the k' best (ties -> lower id); (4) re-score those rows exactly (fp64
// accumulation of the fp32 inputs); (5) sort by exact score (ties -> lower id)
// and write the k best with padding.
// W = 1: one warp per query (4 queries per CTA) for large batches; W = 8: the
// 8 warps of a CTA share one query (lists and re-score split between them, the
// per-warp survivors merged by warp 0) so small batches are not latency-bound.
constexpr int kFinGroup = 4;   // queries per CTA when W == 1

template <int CAP, int HIST = 256>
struct FinBufsT {
  static constexpr int kHist = HIST;
  float key[CAP];
  int32_t id[CAP];
  uint32_t hist[HIST];
};
using FinBufs = FinBufsT<kBufCap, 512>;

// Steps 1-2 for one warp over lists l = first, first + step, ... (in groups of
// 32): the warp's buffer ends with at most K entries (or all it saw).
// (keep: the buffer is cut to the k' best only when it holds more than `keep`
// entries -- the CTA tree merge takes up to 32E unsorted survivors per warp)
template <bool FOLD, int CAP, int HIST>
__device__ int fin_stream_impl(const FinalizeArgs &a, int64_t j, int first_group, int group_step, FinBufsT<CAP, HIST> &B,
                               int keep) {
  const int lane = threadIdx.x & 31;
  const int K = a.kprime;
  // (every list's count is written -- lists of unused splits as 0 -- so all a.lists
  // are read without waiting on the selection count)
  // (the refine pass's lists: F groups of a.lists at list rows f Qa + j, refine_fold)
  const int lists0 = a.lists;
  int lists = lists0;
  int64_t Qa = 0;
  if (FOLD) {
    const RefineFold rf = refine_fold(__ldg(a.qcount), a.fold_qtiles, a.q);
    lists = lists0 * rf.F;
    Qa = rf.Qa;
  }
  auto lrow = [&](int l) -> int64_t {
    return !FOLD ? (int64_t)l * a.q + j : (int64_t)(l % lists0) * a.q + (int64_t)(l / lists0) * Qa + j;
  };
  uint32_t thr = a.gtau ? __ldg(a.gtau + j) : 0u;
  if (a.sorted && K <= a.kread) {
    for (int l = lane; l < lists; l += 32) {
      const int64_t o = lrow(l) * a.stride + (K - 1);
      if (__ldg(a.id + o) >= 0) thr = max(thr, ordered_u32(__ldg(a.key + o)));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) thr = max(thr, __shfl_xor_sync(0xffffffffu, thr, o));
  }
  int n = 0;
  auto count_of = [&](int l) { return l < lists ? (a.cnt ? __ldg(a.cnt + lrow(l)) : a.kread) : 0; };
  int c_next = count_of(first_group * 32 + lane);   // (the next group's counts load under this group's keys)
  for (int l0 = first_group * 32; l0 < lists; l0 += group_step * 32) {
    const int l = l0 + lane;
    const int c = c_next;
    c_next = count_of(l0 + group_step * 32 + lane);
    const int64_t base = lrow(l < lists ? l : 0) * a.stride;
    for (int r0 = 0; __any_sync(0xffffffffu, r0 < c); r0 += 8) {
      float kv[8];
      int32_t iv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        kv[u] = -INFINITY;
        iv[u] = -1;
        if (r0 + u < c) { kv[u] = __ldg(a.key + base + r0 + u); iv[u] = __ldg(a.id + base + r0 + u); }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        bool keep = iv[u] >= 0 && ordered_u32(kv[u]) >= thr;
        uint32_t m = __ballot_sync(0xffffffffu, keep);
        if (m == 0) continue;
        if (n + __popc(m) > CAP) {
          thr = max(thr, warp_keep_best_fast<HIST>(B.key, B.id, n, K, B.hist));
          keep = keep && ordered_u32(kv[u]) >= thr;
          m = __ballot_sync(0xffffffffu, keep);
        }
        if (keep) {
          const int pos = n + __popc(m & lanemask_lt());
          B.key[pos] = kv[u];
          B.id[pos] = iv[u];
        }
        n += __popc(m);
      }
      __syncwarp();
      if (a.sorted && !__any_sync(0xffffffffu, r0 + 8 < c && ordered_u32(kv[7]) >= thr)) break;
    }
  }
  __syncwarp();
  if (n > (keep < 0 ? K : keep)) warp_keep_best_fast<HIST>(B.key, B.id, n, K, B.hist);
  return n;
}
template <int CAP, int HIST>
__device__ __forceinline__ int fin_stream(const FinalizeArgs &a, int64_t j, int first_group, int group_step,
                                          FinBufsT<CAP, HIST> &B, int keep = -1) {
  if (a.qcount != nullptr && a.fold_qtiles > 0) return fin_stream_impl<true>(a, j, first_group, group_step, B, keep);
  return fin_stream_impl<false>(a, j, first_group, group_step, B, keep);
}

// Step 4 for candidates c0, c0 + cstep*U ... of ids[0..m): the warp reads each
// row coalesced, U rows in flight, fp64 accumulation, one transposing reduction
// per U rows.
// Per-query certificate constants: |q|, the key error bound E (natural units) and
// 1 / D, D = the key domain's scale (IP / COS on 16-bit operands: 2^(e_q + e_x)).
struct CertQ {
  double qn, E, dinv;
};
__device__ CertQ cert_setup(const FinalizeArgs &a, int64_t j, double qq) {
  CertQ c;
  c.qn = sqrt(qq);
  const double rq = a.rq ? (double)__ldg(a.rq + j) : 0.0;
  c.E = a.kb.kind == KEY_H16X3 ? key_error_bound_x3(a.kb, a.metric, c.qn, rq, a.rq2 ? (double)__ldg(a.rq2 + j) : 0.0)
                               : key_error_bound(a.kb, a.metric, c.qn, rq);
  const int e = (a.qexp && a.metric != VRS_L2) ? __ldg(a.qexp + j) + a.xexp : 0;
  c.dinv = ldexp(1.0, -e);
  return c;
}
// exact natural key (rank_key units) from a re-scored sort key v (L2: -|q-x|^2, IP: <q,x>, COS: cos)
__device__ __forceinline__ double natural_key(int metric, double v, double qq, double qn) {
  return metric == VRS_L2 ? qq + v : (metric == VRS_COSINE ? v * qn : v);
}

template <int U>
__device__ void fin_rescore(const FinalizeArgs &a, int64_t j, const int32_t *ids, int m, int cfirst, int cstep,
                            double qq, double *sc_out, int64_t *sid_out, const float *keys = nullptr,
                            const CertQ *cq = nullptr) {
  const int lane = threadIdx.x & 31;
  double ratio = 0.0;   // stats: largest observed |key / D - exact key| / E
  const float *q = a.Q + j * a.d;
  const bool vec = (a.d & 3) == 0 && ((reinterpret_cast<uintptr_t>(a.X) | reinterpret_cast<uintptr_t>(a.Q)) & 15) == 0;
  for (int c0 = cfirst * U; c0 < m; c0 += cstep * U) {
    const float *xr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xr[u] = a.X + (int64_t)ids[min(c0 + u, m - 1)] * a.d;
    double sc[U], xx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { sc[u] = 0.0; xx[u] = 0.0; }
    if (vec) {
      for (int t = lane * 4; t < a.d; t += 128) {
        const float4 qv = __ldg(reinterpret_cast<const float4 *>(q + t));
        float4 xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) xv[u] = __ldg(reinterpret_cast<const float4 *>(xr[u] + t));
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (a.metric == VRS_L2) {
            const double d0 = (double)qv.x - xv[u].x, d1 = (double)qv.y - xv[u].y, d2 = (double)qv.z - xv[u].z,
                         d3 = (double)qv.w - xv[u].w;
            sc[u] += d0 * d0; sc[u] += d1 * d1; sc[u] += d2 * d2; sc[u] += d3 * d3;
          } else {
            sc[u] += (double)qv.x * xv[u].x; sc[u] += (double)qv.y * xv[u].y;
            sc[u] += (double)qv.z * xv[u].z; sc[u] += (double)qv.w * xv[u].w;
            if (a.metric == VRS_COSINE) {   // |x|^2 only for the cosine
              xx[u] += (double)xv[u].x * xv[u].x; xx[u] += (double)xv[u].y * xv[u].y;
              xx[u] += (double)xv[u].z * xv[u].z; xx[u] += (double)xv[u].w * xv[u].w;
            }
          }
        }
      }
    } else {
      for (int t = lane; t < a.d; t += 32) {
        const double qv = __ldg(q + t);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const double xv = __ldg(xr[u] + t);
          if (a.metric == VRS_L2) { const double df = qv - xv; sc[u] += df * df; }
          else { sc[u] += qv * xv; if (a.metric == VRS_COSINE) xx[u] += xv * xv; }
        }
      }
    }
    // the U = 8 per-lane partial sums -> row (lane >> 2) & 7's total on every lane,
    // by a transposing butterfly (9 exchanges instead of 8 x 5)
    const double tot = warp_sum_transpose<U>(sc);
    const double xtot = a.metric == VRS_COSINE ? warp_sum_transpose<U>(xx) : 0.0;
    const int u = (lane >> (5 - log2u<U>())) & (U - 1);
    const int c = c0 + u;
    if ((lane & ((32 / U) - 1)) == 0 && c < m) {
      double v = tot;
      if (a.metric == VRS_L2) v = -v;   // sort key: larger is better
      else if (a.metric == VRS_COSINE) v = v / (sqrt(qq) * sqrt(xtot));
      sc_out[c] = v;
      sid_out[c] = ids[c];
      if (keys && cq && cq->E > 0.0 && v == v)
        ratio = fmax(ratio, fabs((double)keys[c] * cq->dinv - natural_key(a.metric, v, qq, cq->qn)) / cq->E);
    }
  }
  if (keys && cq) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ratio = fmax(ratio, __shfl_xor_sync(0xffffffffu, ratio, o));
    if (lane == 0 && ratio > 0.0) atomicMax(a.stats + 2, (unsigned long long)__double_as_longlong(ratio));
  }
}

__device__ double fin_qq(const FinalizeArgs &a, int64_t j) {
  const int lane = threadIdx.x & 31;
  double qq = 0.0;
  if (a.metric == VRS_COSINE || a.cert) {
    const float *q = a.Q + j * a.d;
    for (int t = lane; t < a.d; t += 32) qq += (double)q[t] * (double)q[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) qq += __shfl_xor_sync(0xffffffffu, qq, o);
  }
  return qq;
}

// Step 5 (one warp).
// Bitonic sort of <= 32 (score, id) pairs held one per lane: best first (score
// descending, then id ascending -- ids are unique, so the order is strict).
__device__ __forceinline__ void warp_reg_sort_desc(double &key, int32_t &id) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      const double pk = __shfl_xor_sync(0xffffffffu, key, jj);
      const int32_t pid = __shfl_xor_sync(0xffffffffu, id, jj);
      const bool partner_first = pk > key || (pk == key && pid < id);
      const bool keep_first = ((lane & k) == 0) == ((lane & jj) == 0);   // this slot holds the better of the pair
      if (keep_first == partner_first) { key = pk; id = pid; }
    }
  }
}

// Certificate, lane 0: every row outside the m = k' re-scored
// candidates has a selection key <= kmin (the k'-th kept key: the lists, their
// compactions and the probe threshold only ever drop keys below a kept one), so its
// exact key is <= kmin / D + E; if that is below the k-th exact key s_k, no such row
// can enter the top k and the result is exact.  Fewer than k' candidates: every
// qualifying row was re-scored.  Writes cert / sk / gcnt and the stats.
__device__ void fin_certify(const FinalizeArgs &a, int64_t j, int m, double qq, double skv, float kmin,
                            const CertQ &cq) {
  const bool zero_cos = a.metric == VRS_COSINE && !(qq > 0.0);
  bool ok = true;
  if (!zero_cos && m >= a.kprime) {
    const double s_nat = natural_key(a.metric, skv, qq, cq.qn);
    ok = (double)kmin * cq.dinv + cq.E < s_nat;
  }
  a.cert[j] = ok ? 1 : 0;
  a.sk[j] = skv;
  a.gcnt[j] = 0;
  if (!ok && a.uncert_seen && !a.qmap) *reinterpret_cast<volatile int32_t *>(a.uncert_seen) = 1;
  if (a.stats && !a.qmap) {   // (the refine's finalize re-certifies queries already counted)
    atomicAdd(a.stats, 1ull);
    if (!ok) atomicAdd(a.stats + 1, 1ull);
  }
}

__device__ void fin_sort_write(const FinalizeArgs &a, int64_t j, int m, double qq, double *sc, int64_t *sid,
                               float kmin = -INFINITY, const CertQ *cq = nullptr) {
  const int lane = threadIdx.x & 31;
  const bool zero_cos = a.metric == VRS_COSINE && !(qq > 0.0);
  const int mv = zero_cos ? 0 : min(m, a.k);
  const float pad = a.metric == VRS_L2 ? INFINITY : -INFINITY;
  const int kk = max(1, min(m, a.k));   // rank of the k-th result (or the last)
  if (m <= 32) {   // registers: one candidate per lane (local row ids fit 32 bits)
    double key = lane < m ? sc[lane] : -INFINITY;
    int32_t id = lane < m ? (int32_t)sid[lane] : INT32_MAX;
    warp_reg_sort_desc(key, id);
    if (a.cert) {
      const double skv = __shfl_sync(0xffffffffu, key, kk - 1);
      if (lane == 0) fin_certify(a, j, m, qq, skv, kmin, *cq);
    }
    if (a.k <= 32) {   // lane r holds rank r: write straight from registers
      if (lane < a.k) {
        const int64_t o = j * a.k + lane;
        if (lane < mv) {
          a.ids[o] = a.row_offset + id;
          a.dists[o] = (float)(a.metric == VRS_L2 ? -key : key);
        } else {
          a.ids[o] = -1;
          a.dists[o] = pad;
        }
      }
      return;
    }
    __syncwarp();
    sc[lane] = key;
    sid[lane] = id;
    __syncwarp();
  } else {
    int np = 1;
    while (np < m) np <<= 1;
    for (int c = m + lane; c < np; c += 32) { sc[c] = -INFINITY; sid[c] = INT64_MAX; }
    __syncwarp();
    warp_sort_desc_d(sc, sid, np);
    if (a.cert && lane == 0) fin_certify(a, j, m, qq, sc[kk - 1], kmin, *cq);
  }
  for (int r = lane; r < a.k; r += 32) {
    const int64_t o = j * a.k + r;
    if (r < mv) {
      a.ids[o] = a.row_offset + sid[r];
      const double v = sc[r];
      a.dists[o] = (float)(a.metric == VRS_L2 ? -v : v);
    } else {
      a.ids[o] = -1;
      a.dists[o] = pad;
    }
  }
}

// (CAP: candidate buffer per warp, >= 2 k'; SEL: re-scored rows per warp, >= k'.
// The k' <= 64 variant needs 4 KB of shared memory per warp instead of 9 KB, so
// a 4096-query batch runs in one wave.)
// (the k' <= 64 variant is held to 64 registers: 8 CTAs of 4 warps per SM, so a
// 4096-query batch is one wave -- at 96 registers it was 1.4 waves)
// resident CTAs per SM the <256, 64> variant is register-limited to (A/B: -DVRS_FIN_MINB)
#ifndef VRS_FIN_MINB
#define VRS_FIN_MINB 8
#endif
template <int CAP, int SEL>
__global__ void __launch_bounds__(kFinGroup * 32, SEL <= 64 ? VRS_FIN_MINB : 1) finalize_warp_kernel(FinalizeArgs a) {
  TL_SCOPE(1);
  __shared__ FinBufsT<CAP, SEL <= 64 ? 256 : 512> s_buf[kFinGroup];
  __shared__ double s_sc[kFinGroup][SEL];
  __shared__ int64_t s_sid[kFinGroup][SEL];
  const int w = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * kFinGroup + w;
  pdl_wait();
  TL_WAITED(1);
  pdl_trigger();
  if (j >= a.q) return;   // whole warps only; no block-wide synchronisation below
  if (a.qcount && j >= __ldg(a.qcount)) return;
  const int64_t jq = a.qmap ? __ldg(a.qmap + j) : j;   // (the refine: compacted row -> query)
  const int m = fin_stream_impl<false>(a, j, 0, 1, s_buf[w], -1);   // (the refine's finalize runs the CTA kernel)
  const double qq = fin_qq(a, jq);
  CertQ cq{0.0, 0.0, 1.0};
  float kmin = -INFINITY;
  if (a.cert) {
    cq = cert_setup(a, j, qq);
    kmin = INFINITY;
    for (int i = threadIdx.x & 31; i < m; i += 32) kmin = fminf(kmin, s_buf[w].key[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) kmin = fminf(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
  }
  fin_rescore<SEL <= 64 ? 4 : 8>(a, jq, s_buf[w].id, m, 0, 1, qq, s_sc[w], s_sid[w],
                                 a.stats ? s_buf[w].key : nullptr, &cq);
  __syncwarp();
  fin_sort_write(a, jq, m, qq, s_sc[w], s_sid[w], kmin, &cq);
}

#ifndef VRS_FIN_W
#define VRS_FIN_W 8
#endif
constexpr int kFinW = VRS_FIN_W;   // warps per query in the small-batch variant (16 measured: q = 16 -4 us, q = 256 +10 us)
// k' <= 32E: each warp of the CTA sorts its <= k' survivors, a tree of bitonic
// merges (best 32E of two sorted lists) leaves the 32E best of all warps, sorted,
// in warp 0, which writes the k' best ids to s_buf[0] and their count to s_n[0].
// Exact; ties -> lower id.  (Exchange through the free tail of each warp's buffer:
// its survivors sit at [0, nw <= k').)
template <int E, int W>
__device__ __forceinline__ void fin_tree_merge(const FinalizeArgs &a, FinBufs *s_buf, int nw, int *s_n, float *s_kmin) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float k[E];
  int32_t id[E];
#pragma unroll
  for (int h = 0; h < E; ++h) {
    const int e = h * 32 + lane;
    k[h] = e < nw ? s_buf[w].key[e] : -INFINITY;
    id[h] = e < nw ? s_buf[w].id[e] : INT32_MAX;
  }
  warp_sort_e<E>(k, id);
  constexpr int X0 = kBufCap - 32 * E;
#pragma unroll 1
  for (int stride = W / 2; stride >= 1; stride >>= 1) {
    if (w < 2 * stride) {
#pragma unroll
      for (int h = 0; h < E; ++h) { s_buf[w].key[X0 + h * 32 + lane] = k[h]; s_buf[w].id[X0 + h * 32 + lane] = id[h]; }
    }
    __syncthreads();
    if (w < stride) warp_merge_with_e<E>(k, id, s_buf[w + stride].key + X0, s_buf[w + stride].id + X0);
    __syncthreads();
  }
  if (w == 0) {
    const int K = a.kprime;
    int cnt = 0;
#pragma unroll
    for (int h = 0; h < E; ++h) {
      const int e = h * 32 + lane;
      cnt += __popc(__ballot_sync(0xffffffffu, e < K && id[h] != INT32_MAX));
      if (e < K) { s_buf[0].id[e] = id[h]; s_buf[0].key[e] = k[h]; }
    }
    const float kth = elem_e<E>(k, K - 1);   // the k'-th best (sorted), valid when cnt == K
    if (lane == 0) { s_n[0] = cnt; *s_kmin = kth; }
  }
}


// W warps per query: 8, or 32 for tiny batches (each warp then sees few enough
// candidates to skip the buffer compactions, and the re-score is 4x as wide: C4
// s = 5 %, Q = 1 spent 104 us in the 8-warp kernel, most of it in compactions)
template <int W>
__global__ void __launch_bounds__(W * 32) finalize_cta_kernel(FinalizeArgs a) {
  TL_SCOPE(1);
  extern __shared__ __align__(16) uint8_t fin_dyn[];
  FinBufs *s_buf = reinterpret_cast<FinBufs *>(fin_dyn);   // [W]
  __shared__ double s_sc[kFinMaxSel];
  __shared__ int64_t s_sid[kFinMaxSel];
  __shared__ int s_n[W];
  __shared__ float s_kmin;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = blockIdx.x;
  pdl_wait();
  TL_WAITED(1);
  pdl_trigger();
  if (a.qcount && j >= __ldg(a.qcount)) return;   // (whole CTA)
  const int64_t jq = a.qmap ? __ldg(a.qmap + j) : j;
  // each warp: its share of the lists -> its survivors (<= k', or <= 32E unsorted when
  // the tree merge follows: it sorts them anyway)
  const int keep = a.kprime <= 64 ? 64 : (a.kprime <= 128 ? 128 : -1);
  const int nw = fin_stream(a, j, w, W, s_buf[w], keep);
  if (lane == 0) s_n[w] = nw;
  __syncthreads();
  TL_STAMP(1, 2);
  if (a.kprime <= 64) {
    fin_tree_merge<2, W>(a, s_buf, nw, s_n, &s_kmin);
  } else if (a.kprime <= 128) {
    fin_tree_merge<4, W>(a, s_buf, nw, s_n, &s_kmin);
  } else if (w == 0) {
    // warp 0 merges the survivors of all warps into its own buffer
    const int K = a.kprime;
    FinBufs &B = s_buf[0];
    int n = nw;
    uint32_t thr = 0u;
    for (int v = 1; v < W; ++v) {
      const int nv = s_n[v];
      for (int i0 = 0; i0 < nv; i0 += 32) {
        const int i = i0 + lane;
        float kv = -INFINITY;
        int32_t iv = -1;
        if (i < nv) { kv = s_buf[v].key[i]; iv = s_buf[v].id[i]; }
        bool keep = i < nv && ordered_u32(kv) >= thr;
        uint32_t m = __ballot_sync(0xffffffffu, keep);
        if (n + __popc(m) > kBufCap) {
          thr = max(thr, warp_keep_best_fast<FinBufs::kHist>(B.key, B.id, n, K, B.hist));
          keep = keep && ordered_u32(kv) >= thr;
          m = __ballot_sync(0xffffffffu, keep);
        }
        if (keep) {
          const int pos = n + __popc(m & lanemask_lt());
          B.key[pos] = kv;
          B.id[pos] = iv;
        }
        n += __popc(m);
        __syncwarp();
      }
    }
    if (n > K) warp_keep_best_fast<FinBufs::kHist>(B.key, B.id, n, K, B.hist);
    float km = INFINITY;
    for (int i = lane; i < n; i += 32) km = fminf(km, B.key[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) km = fminf(km, __shfl_xor_sync(0xffffffffu, km, o));
    if (lane == 0) { s_n[0] = n; s_kmin = km; }
  }
  __syncthreads();
  TL_STAMP(1, 3);
  const int m = s_n[0];
  const double qq = fin_qq(a, jq);
  CertQ cq{0.0, 0.0, 1.0};
  if (a.cert) cq = cert_setup(a, j, qq);
  fin_rescore<8>(a, jq, s_buf[0].id, m, w, W, qq, s_sc, s_sid, a.stats ? s_buf[0].key : nullptr, &cq);
  __syncthreads();
  TL_STAMP(1, 4);
  if (w == 0) fin_sort_write(a, jq, m, qq, s_sc, s_sid, s_kmin, &cq);
}

// Small batches (tensor-core lists, q <= VRS_FIN_BLOCK_Q): one CTA of kFinBT threads per
// query, few block-wide steps (a Q = 1 finalize is a latency chain on one SM):
//  (1) the per-(split, list) counts, prefix-summed block-wide (a thread per list);
//  (2) every candidate at or above the probe threshold staged in shared memory;
//  (3) the k' best (key desc, id asc): min / max, one 2048-bucket histogram over a
//      monotone linear map of the keys, the bucket holding the k'-th best found from the
//      top, everything above it taken, the boundary bucket resolved by ranking;
//  (4) exact re-score (every warp, U rows in flight);
//  (5) rank sort of the <= k' exact scores, the certificate, the k best written.
// Replaces the per-warp buffer compactions and tree merge of finalize_cta_kernel
// (r02_small_q_chain_timeline.txt: 40-90 us at Q = 1).  More than kFinStage candidates,
// a single-valued key range or a crowded boundary bucket: the radix select
// (block_select_top) over the lists instead -- the same result.
constexpr int kFinBT = 512;
constexpr int kFinStage = 16384;      // staged candidates (128 KB of key + id)
constexpr int kFinBlockMaxLists = 4096;
constexpr int kFinNB = 2048;          // histogram buckets
constexpr int kFinBnd = 1024;         // boundary-bucket capacity of the ranking step
static size_t finalize_block_smem(int lists) { return (size_t)kFinStage * 8 + (size_t)(lists + 1) * 4; }

struct FinBlockShared {
  uint32_t hist[kFinNB];
  float bkey[kFinBnd];
  int32_t bid[kFinBnd];
  double sc[kFinMaxSel], sc2[kFinMaxSel];
  int64_t sid[kFinMaxSel], sid2[kFinMaxSel];
  int32_t sel[kFinMaxSel];
  float selk[kFinMaxSel];
  int32_t wsum[kFinBT / 32];
  uint32_t wlo[kFinBT / 32], whi[kFinBT / 32], wcnt[kFinBT / 32];
  float wkmin[kFinBT / 32];
  int n_out, n_bnd, bstar, above;
};

// (3) on the staged set: exactly the K best valid (id >= 0) entries -> out (unordered);
// returns their number, or -1 when the caller must fall back to the radix select.
template <int NT>
__device__ int block_select_staged(const float *key, const int32_t *id, int T, int K, FinBlockShared &S) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t lo = 0xffffffffu, hi = 0u, cnt = 0;
  for (int c = tid; c < T; c += NT)
    if (id[c] >= 0) {
      const uint32_t u = ordered_u32(key[c]);
      lo = min(lo, u); hi = max(hi, u); ++cnt;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if (lane == 0) { S.wlo[w] = lo; S.whi[w] = hi; S.wcnt[w] = cnt; }
  for (int b = tid; b < kFinNB; b += NT) S.hist[b] = 0;
  if (tid == 0) { S.n_out = 0; S.n_bnd = 0; }
  __syncthreads();
  lo = 0xffffffffu; hi = 0u; cnt = 0;
#pragma unroll
  for (int v = 0; v < NT / 32; ++v) { lo = min(lo, S.wlo[v]); hi = max(hi, S.whi[v]); cnt += S.wcnt[v]; }
  if ((int)cnt <= K) {   // every valid entry
    for (int c = tid; c < T; c += NT)
      if (id[c] >= 0) {
        const int p = atomicAdd(&S.n_out, 1);
        S.sel[p] = id[c]; S.selk[p] = key[c];
      }
    __syncthreads();
    return (int)cnt;
  }
  if (hi == lo) return -1;   // (block-uniform) one key value: ties by id -> the radix path
  const float scale = ((float)kFinNB - 0.5f) / (float)(hi - lo);
  auto bucket = [&](uint32_t u) { return min(kFinNB - 1, (int)((float)(u - lo) * scale)); };   // monotone
  for (int c = tid; c < T; c += NT)
    if (id[c] >= 0) atomicAdd(&S.hist[bucket(ordered_u32(key[c]))], 1u);
  __syncthreads();
  // bucket of the K-th best: thread t sums buckets [NB-1-4t-3, NB-1-4t] (descending)
  constexpr int PB = kFinNB / NT;
  uint32_t v[PB], s = 0;
#pragma unroll
  for (int t = 0; t < PB; ++t) { v[t] = S.hist[kFinNB - 1 - PB * tid - t]; s += v[t]; }
  uint32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) S.wcnt[w] = incl;
  __syncthreads();
  uint32_t wbefore = 0;
  for (int u = 0; u < w; ++u) wbefore += S.wcnt[u];
  const uint32_t before = wbefore + incl - s;
  if (before < (uint32_t)K && (uint32_t)K <= before + s) {
    uint32_t run = before;
#pragma unroll
    for (int t = 0; t < PB; ++t) {
      if ((uint32_t)K <= run + v[t]) { S.bstar = kFinNB - 1 - PB * tid - t; S.above = (int)run; break; }
      run += v[t];
    }
  }
  __syncthreads();
  const int bstar = S.bstar, above = S.above;
  for (int c = tid; c < T; c += NT)
    if (id[c] >= 0) {
      const int b = bucket(ordered_u32(key[c]));
      if (b > bstar) {
        const int p = atomicAdd(&S.n_out, 1);
        S.sel[p] = id[c]; S.selk[p] = key[c];
      } else if (b == bstar) {
        const int p = atomicAdd(&S.n_bnd, 1);
        if (p < kFinBnd) { S.bkey[p] = key[c]; S.bid[p] = id[c]; }
      }
    }
  __syncthreads();
  const int nb = S.n_bnd;
  if (nb > kFinBnd) return -1;   // (block-uniform)
  const int rem = K - above;
  for (int i = tid; i < nb; i += NT) {   // rank in the boundary bucket (key desc, id asc)
    const float ki = S.bkey[i];
    const int32_t ii = S.bid[i];
    int r = 0;
    for (int t = 0; t < nb; ++t) {
      const float kt = S.bkey[t];
      r += (kt > ki || (kt == ki && S.bid[t] < ii)) ? 1 : 0;
    }
    if (r < rem) { S.sel[above + r] = ii; S.selk[above + r] = ki; }
  }
  __syncthreads();
  return K;
}

__global__ void __launch_bounds__(kFinBT, 1) finalize_block_kernel(FinalizeArgs a) {
  TL_SCOPE(1);
  extern __shared__ __align__(16) uint8_t fin_dyn[];
  float *s_key = reinterpret_cast<float *>(fin_dyn);                 // [kFinStage]
  int32_t *s_id = reinterpret_cast<int32_t *>(s_key + kFinStage);    // [kFinStage]; -1 = dropped
  int32_t *s_off = s_id + kFinStage;                                 // [lists + 1] list offsets
  __shared__ FinBlockShared S;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  constexpr int NW = kFinBT / 32;
  const int64_t j = blockIdx.x;
  pdl_wait();
  TL_WAITED(1);
  pdl_trigger();
  const int L = a.lists;
  const uint32_t thr = a.gtau ? __ldg(a.gtau + j) : 0u;
  constexpr int PL = kFinBlockMaxLists / kFinBT;   // lists per thread (at most)
  const int per = (L + kFinBT - 1) / kFinBT;
  const int l0 = min(L, tid * per);
  auto lbase = [&](int l) { return ((int64_t)l * a.q + j) * a.stride; };
  // (1) counts (registers) -> block-wide exclusive prefix -> s_off
  int cl[PL];
  int mine = 0;
#pragma unroll
  for (int i = 0; i < PL; ++i) {
    const int l = l0 + i;
    cl[i] = (i < per && l < L) ? (a.cnt ? __ldg(a.cnt + (int64_t)l * a.q + j) : a.kread) : 0;
    mine += cl[i];
  }
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) S.wsum[w] = incl;
  __syncthreads();
  int off = incl - mine, total = 0;
#pragma unroll
  for (int v = 0; v < NW; ++v) {
    const int x = S.wsum[v];
    off += v < w ? x : 0;
    total += x;
  }
  const bool staged = total <= (a.stage_cap > 0 ? min(a.stage_cap, kFinStage) : kFinStage);
  // (2) stage (a thread per list, 8 loads in flight); s_off for the fallback's lookups
#pragma unroll
  for (int i = 0; i < PL; ++i) {
    const int l = l0 + i;
    if (i < per && l < L) {
      s_off[l] = off;
      if (staged) {
        const int c = cl[i];
        const int64_t b = lbase(l);
        for (int r0 = 0; r0 < c; r0 += 8) {
          float kv[8];
          int32_t iv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (r0 + u < c) { kv[u] = __ldg(a.key + b + r0 + u); iv[u] = __ldg(a.id + b + r0 + u); }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (r0 + u < c) {
              s_key[off + r0 + u] = kv[u];
              s_id[off + r0 + u] = (iv[u] >= 0 && ordered_u32(kv[u]) >= thr) ? iv[u] : -1;
            }
        }
      }
      off += cl[i];
    }
  }
  if (tid == 0) s_off[L] = total;
  __syncthreads();
  TL_STAMP(1, 2);
  // (3) the k' best by key (ties -> lower id), unordered, in S.sel / S.selk
  int m = staged && a.stage_cap >= 0 ? block_select_staged<kFinBT>(s_key, s_id, total, a.kprime, S) : -1;
  if (m < 0) {
    auto get = [&](int64_t c, float &k, int32_t &i) -> bool {
      if (staged) {
        i = s_id[c];
        k = s_key[c];
        return i >= 0;
      }
      int lo = 0, hi = L;   // the list holding entry c: s_off[lo] <= c < s_off[lo + 1]
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_off[mid] <= c) lo = mid; else hi = mid;
      }
      const int64_t o = lbase(lo) + (c - s_off[lo]);
      k = __ldg(a.key + o);
      i = __ldg(a.id + o);
      return i >= 0 && ordered_u32(k) >= thr;
    };
    m = block_select_top<int32_t, kFinBT>(get, total, a.kprime, S.sel, S.selk);
  }
  TL_STAMP(1, 3);
  // (4) exact re-score: every warp, 8 rows in flight
  const double qq = fin_qq(a, j);
  CertQ cq{0.0, 0.0, 1.0};
  if (a.cert) cq = cert_setup(a, j, qq);
  fin_rescore<8>(a, j, S.sel, m, w, NW, qq, S.sc, S.sid, a.stats ? S.selk : nullptr, &cq);
  __syncthreads();
  TL_STAMP(1, 4);
  // (5) rank sort by exact score (ids unique: a strict order; NaN ranks as -inf), the
  // certificate (thread 0), the k best written best-first with padding
  for (int i = tid; i < m; i += kFinBT) {
    const double ki = S.sc[i] == S.sc[i] ? S.sc[i] : -INFINITY;
    const int64_t ii = S.sid[i];
    int r = 0;
    for (int t = 0; t < m; ++t) {
      const double kt = S.sc[t] == S.sc[t] ? S.sc[t] : -INFINITY;
      r += (kt > ki || (kt == ki && S.sid[t] < ii)) ? 1 : 0;
    }
    S.sc2[r] = ki;
    S.sid2[r] = ii;
  }
  float km = INFINITY;
  for (int i = tid; i < m; i += kFinBT) km = fminf(km, S.selk[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) km = fminf(km, __shfl_xor_sync(0xffffffffu, km, o));
  if (lane == 0) S.wkmin[w] = km;
  __syncthreads();
  const bool zero_cos = a.metric == VRS_COSINE && !(qq > 0.0);
  if (a.cert && tid == 0) {
    float kmin = INFINITY;
    for (int v = 0; v < NW; ++v) kmin = fminf(kmin, S.wkmin[v]);
    fin_certify(a, j, m, qq, S.sc2[max(1, min(m, a.k)) - 1], kmin, cq);
  }
  const int mv = zero_cos ? 0 : min(m, a.k);
  const float pad = a.metric == VRS_L2 ? INFINITY : -INFINITY;
  for (int r = tid; r < a.k; r += kFinBT) {
    const int64_t o = j * a.k + r;
    if (r < mv) {
      a.ids[o] = a.row_offset + S.sid2[r];
      const double v = S.sc2[r];
      a.dists[o] = (float)(a.metric == VRS_L2 ? -v : v);
    } else {
      a.ids[o] = -1;
      a.dists[o] = pad;
    }
  }
}

// Per query (one CTA): the kth largest probe slot maximum (each the key of a
// distinct row) -> gtau, a lower bound of the kth best key over all rows.  The
// values are staged once in shared memory (ordered u32, 0 = no row) and a
// block-wide radix select (8 bits per pass) finds the kth largest.
// (block size: 256 threads for large batches, 1024 for small ones -- few queries,
// long value lists, so more threads per query)
template <int kThrThreads>
__global__ void __launch_bounds__(kThrThreads) threshold_kernel(ThresholdArgs a) {
  TL_SCOPE(0);
  extern __shared__ uint32_t s_val[];
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_bin, s_above, s_total;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t j = blockIdx.x;
  const float *v = a.vals + j * a.nvals;
  pdl_wait();
  TL_WAITED(0);
  pdl_trigger();
  const int nvals = (int)min((int64_t)a.nvals, kListsPerSplit * splits_used(a.split) * 32);   // lists of used splits only
  __shared__ uint32_t s_lo[32], s_hi[32], s_cnt[32], s_cv[64];
  __shared__ int s_bstar, s_upto, s_got;
  // fast path: min / max, one histogram over value buckets, the <= 64 values
  // from the K-th largest's bucket up sorted by warp 0 (else the radix passes)
  uint32_t lo = 0xffffffffu, hi = 0u, cnt = 0;
  for (int i = tid; i < nvals; i += kThrThreads) {
    const float f = __ldg(v + i);
    const uint32_t u = f > -INFINITY ? ordered_u32(f) : 0u;
    s_val[i] = u;
    if (u) { lo = min(lo, u); hi = max(hi, u); ++cnt; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if (lane == 0) { s_lo[warp] = lo; s_hi[warp] = hi; s_cnt[warp] = cnt; }
  for (int b = tid; b < 256; b += kThrThreads) hist[b] = 0;
  if (tid == 0) s_got = 0;
  __syncthreads();
  lo = 0xffffffffu; hi = 0u; cnt = 0;
  for (int w = 0; w < kThrThreads / 32; ++w) { lo = min(lo, s_lo[w]); hi = max(hi, s_hi[w]); cnt += s_cnt[w]; }
  if (cnt < (uint32_t)a.kth) {   // fewer than kth rows probed: no bound
    if (tid == 0) a.gtau[j] = 0u;
    return;
  }
  if (hi == lo || a.kth > 64) goto radix;
  {
    const float scale = 255.5f / (float)(hi - lo);
    auto bucket = [&](uint32_t u) { return (uint32_t)min(255, (int)((float)(u - lo) * scale)); };
    for (int i0 = 0; i0 < nvals; i0 += kThrThreads) {
      const int i = i0 + tid;
      const uint32_t u = i < nvals ? s_val[i] : 0u;
      hist_add_warp(hist, u ? bucket(u) : 256u);
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t c[8], sum = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) { c[t] = hist[255 - 8 * lane - t]; sum += c[t]; }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t before = incl - sum;
      if (before < (uint32_t)a.kth && (uint32_t)a.kth <= incl) {
        uint32_t run = before;
        for (int t = 0; t < 8; ++t) {
          if ((uint32_t)a.kth <= run + c[t]) { s_bstar = 255 - 8 * lane - t; s_upto = (int)(run + c[t]); break; }
          run += c[t];
        }
      }
    }
    __syncthreads();
    const int bstar = s_bstar, upto = s_upto;
    if (upto <= 64) {
      for (int i = tid; i < nvals; i += kThrThreads) {
        const uint32_t u = s_val[i];
        if (u && (int)bucket(u) >= bstar) s_cv[atomicAdd(&s_got, 1)] = u;
      }
      __syncthreads();
      if (warp == 0) {
        const int got = s_got;
        auto to_f = [](uint32_t o) { return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o); };
        float ka = lane < got ? to_f(s_cv[lane]) : -INFINITY, kb = lane + 32 < got ? to_f(s_cv[lane + 32]) : -INFINITY;
        int32_t ia = lane, ib = lane + 32;
        warp_reg_sort64(ka, ia, kb, ib);
        const float kth = __shfl_sync(0xffffffffu, a.kth - 1 < 32 ? ka : kb, (a.kth - 1) & 31);
        if (lane == 0) a.gtau[j] = ordered_u32(kth);
      }
      return;
    }
  }
radix:
  uint32_t prefix = 0, mask = 0;
  int rem = a.kth;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = tid; b < 256; b += kThrThreads) hist[b] = 0;
    __syncthreads();
    for (int i0 = 0; i0 < nvals; i0 += kThrThreads) {
      const int i = i0 + tid;
      const uint32_t u = i < nvals ? s_val[i] : 0u;
      hist_add_warp(hist, (u != 0u && (u & mask) == prefix) ? (u >> shift) & 255u : 256u);
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t c[8], sum = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) { c[t] = hist[255 - 8 * lane - t]; sum += c[t]; }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_total = incl;
      const uint32_t before = incl - sum;
      if (before < (uint32_t)rem && (uint32_t)rem <= incl) {
        uint32_t run = before;
        for (int t = 0; t < 8; ++t) {
          if ((uint32_t)rem <= run + c[t]) { s_bin = 255 - 8 * lane - t; s_above = run; break; }
          run += c[t];
        }
      }
    }
    __syncthreads();
    if (s_total < (uint32_t)rem) {   // first pass only: fewer than kth rows probed
      if (tid == 0) a.gtau[j] = 0u;
      return;
    }
    prefix |= s_bin << shift;
    mask |= 255u << shift;
    rem -= (int)s_above;
    __syncthreads();
  }
  if (tid == 0) a.gtau[j] = prefix;
}

// Per lane the E largest of v[first + S * t] (the warp's lanes at consecutive
// first), warp-sorted: returns element K-1 of the union (-inf if fewer).
template <int E, int S>
__device__ __forceinline__ void lane_top_sorted(const float *v, int nvals, int first, float (&t)[E]) {
#pragma unroll
  for (int h = 0; h < E; ++h) t[h] = -INFINITY;
  int i = first;
  for (; i + 3 * S < nvals; i += 4 * S) {
    float f[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) f[u] = __ldg(v + i + S * u);
#pragma unroll
    for (int u = 0; u < 4; ++u) top_insert_e<E>(t, f[u]);
  }
  for (; i < nvals; i += S) top_insert_e<E>(t, __ldg(v + i));
  int32_t id[E];
#pragma unroll
  for (int h = 0; h < E; ++h) id[h] = h * 32 + (int)(threadIdx.x & 31);
  warp_sort_e<E>(t, id);
}
template <int E, int S>
__device__ __forceinline__ float lane_top_kth(const float *v, int nvals, int first, int K) {
  float t[E];
  lane_top_sorted<E, S>(v, nvals, first, t);
  return elem_e<E>(t, K - 1);
}

// Large batches: one warp per query, registers only.  Each lane keeps the two
// largest of its values (slot `lane` of every list); the K-th largest of that
// union of 64 values is <= the K-th largest of all values (a subset's K-th
// largest never exceeds the whole set's), so it is still a valid lower bound of
// the K-th best key -- a slightly looser one when a lane holds more than two of
// the top K.  Exact when every lane holds <= 2 values.
// K > 64 stages the values in shared memory for the radix select.
__global__ void __launch_bounds__(kFinGroup * 32) threshold_warp_kernel(ThresholdArgs a) {
  TL_SCOPE(0);
  extern __shared__ uint32_t s_vals[];
  __shared__ uint32_t s_hist[kFinGroup][256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * kFinGroup + w;
  pdl_wait();
  TL_WAITED(0);
  pdl_trigger();
  if (j >= a.q) return;
  const float *v = a.vals + j * a.nvals;
  const int nvals = (int)a.nvals;   // (every probe slot is written, unused splits as -inf: no wait on the count)
  if (a.kth > 128) {
    uint32_t *mine = s_vals + (size_t)w * a.nvals;
    for (int i = lane; i < nvals; i += 32) {
      const float f = __ldg(v + i);
      mine[i] = f > -INFINITY ? ordered_u32(f) : 0u;
    }
    __syncwarp();
    uint32_t x = 0;
    const bool ok = warp_kth_value_fast(mine, nvals, a.kth, s_hist[w], &x);
    if (lane == 0) a.gtau[j] = ok ? x : 0u;
    return;
  }
  // (the union keeps 32E values, at least 2K: with 32E == K its K-th largest would be its
  // minimum, a far looser bound -- C4 k' = 128 at E = 4 cost the main pass 40 %)
  const float kth = a.kth <= 32   ? lane_top_kth<2, 32>(v, nvals, lane, a.kth)
                    : a.kth <= 64 ? lane_top_kth<4, 32>(v, nvals, lane, a.kth)
                                  : lane_top_kth<8, 32>(v, nvals, lane, a.kth);
  if (lane == 0) a.gtau[j] = kth > -INFINITY ? ordered_u32(kth) : 0u;
}

// Per-lane E largest of a strided share, all loads of a round issued together
// (U per lane), then sorted warp-wide (element h * 32 + lane).
template <int E, int S, int U>
__device__ __forceinline__ void lane_top_sorted_1r(const float *v, int nvals, int first, float (&t)[E]) {
#pragma unroll
  for (int h = 0; h < E; ++h) t[h] = -INFINITY;
#pragma unroll 1
  for (int i0 = first; i0 < nvals; i0 += U * S) {
    float f[U];
#pragma unroll
    for (int u = 0; u < U; ++u) f[u] = i0 + u * S < nvals ? __ldg(v + i0 + u * S) : -INFINITY;
#pragma unroll
    for (int u = 0; u < U; ++u) top_insert_e<E>(t, f[u]);
  }
  int32_t id[E];
#pragma unroll
  for (int h = 0; h < E; ++h) id[h] = h * 32 + (int)(threadIdx.x & 31);
  warp_sort_e<E>(t, id);
}

// Small batches (K <= 128): one CTA of NW warps per query, registers first.  Each
// lane keeps the E largest of its strided share (E = 2 for K <= 64, else 4),
// each warp sorts its 32E and keeps its best 32M (M = 1 for K <= 32), and a tree
// of bitonic merges (best 32M of two sorted lists) leaves the 32M largest of the
// warps' union in warp 0.  Every stage keeps a subset of the values that holds
// that subset's K best, so its K-th largest is <= the K-th largest of all values:
// a valid lower bound of the K-th best key (see threshold_warp_kernel).  Every
// probe slot is written (CTAs of unused splits publish -inf), so all a.nvals
// values are read -- no wait on the selection count -- in one round of loads.
template <int NW, int E, int M>
__global__ void __launch_bounds__(NW * 32) threshold_union_kernel(ThresholdArgs a) {
  static_assert(M <= E, "merged width within the per-lane lists");
  TL_SCOPE(0);
  __shared__ float s_f[NW][32 * M];
  __shared__ int32_t s_i[NW][32 * M];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = blockIdx.x;
  pdl_wait();
  TL_WAITED(0);
  pdl_trigger();
  const float *v = a.vals + j * a.nvals;
  TL_STAMP(0, 2);
  float t[E];
  lane_top_sorted_1r<E, NW * 32, 12>(v, (int)a.nvals, w * 32 + lane, t);
  TL_STAMP(0, 3);
  float tm[M];
  int32_t id[M];
#pragma unroll
  for (int h = 0; h < M; ++h) { tm[h] = t[h]; id[h] = (w * M + h) * 32 + lane; }   // (distinct tie-breakers)
#pragma unroll 1
  for (int stride = NW / 2; stride >= 1; stride >>= 1) {
    if (w < 2 * stride) {
#pragma unroll
      for (int h = 0; h < M; ++h) { s_f[w][h * 32 + lane] = tm[h]; s_i[w][h * 32 + lane] = id[h]; }
    }
    __syncthreads();
    if (w < stride) warp_merge_with_e<M>(tm, id, s_f[w + stride], s_i[w + stride]);
    __syncthreads();
  }
  TL_STAMP(0, 4);
  if (w == 0) {
    const float kth = elem_e<M>(tm, a.kth - 1);
    if (lane == 0) a.gtau[j] = kth > -INFINITY ? ordered_u32(kth) : 0u;
  }
}

// Small batches (q < 148, <= 32768 values per query): one CTA of 1024 threads per query,
// few block-wide steps -- every value loaded in one round (<= 32 per thread, registers),
// min / max, one 2048-bucket histogram over a monotone linear map of the values, the
// bucket holding the K-th largest found from the top; gtau = the smallest value in that
// bucket.  At least K values are >= it, so it is <= the K-th largest: a valid lower bound
// of the K-th best key (within one bucket of the K-th value).  Replaces the per-lane top-E
// union and its register sorts / merge tree (C3 / C4, Q = 1: 16-28 us on one SM).
constexpr int kThrHT = 1024;
constexpr int kThrHV = 32;      // values per thread
constexpr int kThrHNB = 2048;   // buckets
__global__ void __launch_bounds__(kThrHT, 1) threshold_hist_kernel(ThresholdArgs a) {
  TL_SCOPE(0);
  __shared__ uint32_t hist[kThrHNB];
  __shared__ uint32_t s_lo[32], s_hi[32], s_cnt[32], s_w[32];
  __shared__ uint32_t s_min;
  __shared__ int s_bstar;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t j = blockIdx.x;
  pdl_wait();
  TL_WAITED(0);
  pdl_trigger();
  const float *v = a.vals + j * a.nvals;
  TL_STAMP(0, 2);
  uint32_t u[kThrHV];
  uint32_t lo = 0xffffffffu, hi = 0u, cnt = 0;
#pragma unroll
  for (int i = 0; i < kThrHV; ++i) {
    const int idx = tid + i * kThrHT;
    const float f = idx < a.nvals ? __ldg(v + idx) : -INFINITY;
    u[i] = f > -INFINITY ? ordered_u32(f) : 0u;
  }
#pragma unroll
  for (int i = 0; i < kThrHV; ++i)
    if (u[i]) { lo = min(lo, u[i]); hi = max(hi, u[i]); ++cnt; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if (lane == 0) { s_lo[w] = lo; s_hi[w] = hi; s_cnt[w] = cnt; }
  for (int b = tid; b < kThrHNB; b += kThrHT) hist[b] = 0;
  if (tid == 0) s_min = 0xffffffffu;
  __syncthreads();
  lo = 0xffffffffu; hi = 0u; cnt = 0;
#pragma unroll
  for (int x = 0; x < 32; ++x) { lo = min(lo, s_lo[x]); hi = max(hi, s_hi[x]); cnt += s_cnt[x]; }
  if (cnt < (uint32_t)a.kth) {   // fewer than K probed rows: no bound
    if (tid == 0) a.gtau[j] = 0u;
    return;
  }
  if (hi == lo) {   // (block-uniform) one value: it is the K-th largest
    if (tid == 0) a.gtau[j] = lo;
    return;
  }
  const float scale = ((float)kThrHNB - 0.5f) / (float)(hi - lo);
  auto bucket = [&](uint32_t x) { return min(kThrHNB - 1, (int)((float)(x - lo) * scale)); };   // monotone
#pragma unroll
  for (int i = 0; i < kThrHV; ++i)
    if (u[i]) atomicAdd(&hist[bucket(u[i])], 1u);
  __syncthreads();
  // the bucket of the K-th largest: thread t sums buckets [NB-1-2t-1, NB-1-2t] (descending)
  constexpr int PB = kThrHNB / kThrHT;
  uint32_t hv[PB], sum = 0;
#pragma unroll
  for (int t = 0; t < PB; ++t) { hv[t] = hist[kThrHNB - 1 - PB * tid - t]; sum += hv[t]; }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[w] = incl;
  __syncthreads();
  uint32_t before = incl - sum;
  for (int x = 0; x < w; ++x) before += s_w[x];
  if (before < (uint32_t)a.kth && (uint32_t)a.kth <= before + sum) {
    uint32_t run = before;
#pragma unroll
    for (int t = 0; t < PB; ++t) {
      if ((uint32_t)a.kth <= run + hv[t]) { s_bstar = kThrHNB - 1 - PB * tid - t; break; }
      run += hv[t];
    }
  }
  __syncthreads();
  const int bstar = s_bstar;
  uint32_t mn = 0xffffffffu;
#pragma unroll
  for (int i = 0; i < kThrHV; ++i)
    if (u[i] && bucket(u[i]) == bstar) mn = min(mn, u[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if (lane == 0 && mn != 0xffffffffu) atomicMin(&s_min, mn);
  __syncthreads();
  TL_STAMP(0, 3);
  if (tid == 0) a.gtau[j] = s_min;
}

cudaError_t launch_threshold(const ThresholdArgs &a, cudaStream_t s) {
  // large batches with short value lists: a warp per query (A/B: VRS_BLOCK_THRESHOLD forces the block kernel)
  static const bool block_thr = getenv("VRS_BLOCK_THRESHOLD") != nullptr;
  const size_t wsmem = a.kth > 128 ? (size_t)kFinGroup * a.nvals * 4 : 0;
  if (!block_thr && a.q >= 4 * kSmCountB200 && wsmem <= 96 * 1024) {
    static size_t wattr = 0;
    const cudaError_t e = ensure_smem_attr(threshold_warp_kernel, wsmem, wattr);
    if (e != cudaSuccess) return e;
    return launch_k(threshold_warp_kernel, dim3((unsigned)((a.q + kFinGroup - 1) / kFinGroup)), dim3(kFinGroup * 32),
                    wsmem, s, a);
  }
  // (small batches with k' >= 64: the block histogram kernel -- C3 s = 10 %, Q = 1 threshold
  // 16 -> 9 us, C4 s = 5 %, Q = 1 28 -> 12 us (cells -4-5 %); with C2's k' = 26 the union
  // kernel is 4 us faster; VRS_THR_UNION=1 keeps the union kernels for A/B, r02_threshold_hist_ab.txt)
  static const bool thr_union = getenv("VRS_THR_UNION") != nullptr;
  if (!block_thr && !thr_union && a.q < kSmCountB200 && a.kth >= 64 && a.nvals <= kThrHT * kThrHV)
    return launch_k(threshold_hist_kernel, dim3((unsigned)a.q), dim3(kThrHT), 0, s, a);
  if (!block_thr && a.kth <= 128) {
    // per lane E values, merged width 32M >= 2K (M = E): the K-th of the kept union stays
    // close to the K-th of all values (see threshold_warp_kernel)
    const bool big = a.q < kSmCountB200;   // few queries: more warps per query
    if (a.kth <= 32)
      return big ? launch_k(threshold_union_kernel<32, 2, 2>, dim3((unsigned)a.q), dim3(1024), 0, s, a)
                 : launch_k(threshold_union_kernel<8, 2, 2>, dim3((unsigned)a.q), dim3(256), 0, s, a);
    if (a.kth <= 64)
      return big ? launch_k(threshold_union_kernel<16, 4, 4>, dim3((unsigned)a.q), dim3(512), 0, s, a)
                 : launch_k(threshold_union_kernel<8, 4, 4>, dim3((unsigned)a.q), dim3(256), 0, s, a);
    // (E = 8: a warp's register sort is costly -- 8 warps, each lane with more values, beat 16 / 32)
    return launch_k(threshold_union_kernel<8, 8, 8>, dim3((unsigned)a.q), dim3(256), 0, s, a);
  }
  const size_t smem = (size_t)a.nvals * 4;
  static size_t attr1024 = 0, attr256 = 0;
  cudaError_t e = ensure_smem_attr(threshold_kernel<1024>, smem, attr1024);
  if (e == cudaSuccess) e = ensure_smem_attr(threshold_kernel<256>, smem, attr256);
  if (e != cudaSuccess) return e;
  if (a.q < kSmCountB200) return launch_k(threshold_kernel<1024>, dim3((unsigned)a.q), dim3(1024), smem, s, a);
  return launch_k(threshold_kernel<256>, dim3((unsigned)a.q), dim3(256), smem, s, a);
}

cudaError_t launch_finalize(const FinalizeArgs &a, cudaStream_t s, int *launches) {
  if (launches) *launches += 1;
  // small batches: a CTA of 8 warps per query; large: a warp per query
  // (the refine's finalize: the CTA kernel -- its queries read F x the lists, refine_fold)
  // (the block kernel for q <= 256 when k' >= 64: C3 s = 10 %, Q = 1 finalize 91 -> 49 us, C4 s = 5 %,
  // Q = 256 -3 %; with C2's k' = 26 the CTA kernel is as fast at q = 1-16 and 10 us faster at
  // q = 256 -- VRS_FIN_BLOCK_Q overrides)
  static const int block_q_env = getenv("VRS_FIN_BLOCK_Q") ? atoi(getenv("VRS_FIN_BLOCK_Q")) : -1;
  const int block_q = block_q_env >= 0 ? block_q_env : (a.kprime >= 64 ? 256 : 0);
  if (a.q <= block_q && a.fold_qtiles == 0 && !a.sorted && a.lists <= kFinBlockMaxLists && a.kprime <= kFinMaxSel) {
    static size_t attrb = 0;
    const cudaError_t e = ensure_smem_attr(finalize_block_kernel, finalize_block_smem(kFinBlockMaxLists), attrb);
    if (e != cudaSuccess) return e;
    static const int stage_env = getenv("VRS_FIN_STAGE") ? atoi(getenv("VRS_FIN_STAGE")) : 0;
    FinalizeArgs b = a;
    b.stage_cap = stage_env;
    return launch_k(finalize_block_kernel, dim3((unsigned)a.q), dim3(kFinBT), finalize_block_smem(a.lists), s, b);
  }
  if (a.q < 4 * kSmCountB200 || a.fold_qtiles > 0) {
    // (16 warps per query for <= 64 queries with k' >= 64: C4 s = 5 %, Q = 1 finalize 93 -> 48 us;
    // k' = 32 (C2) gains nothing; 32 warps measured slower -- they spill at 64 registers,
    // r02_finalize_width_ab.txt)
    static const int wide_q_env = getenv("VRS_FIN_WIDE_Q") ? atoi(getenv("VRS_FIN_WIDE_Q")) : -1;
    const int wide_q = wide_q_env >= 0 ? wide_q_env : (a.kprime >= 64 ? 64 : 0);
    if (a.q <= wide_q && a.fold_qtiles == 0) {
      const size_t smem = sizeof(FinBufs) * 16;
      static size_t attr16 = 0;
      const cudaError_t e = ensure_smem_attr(finalize_cta_kernel<16>, smem, attr16);
      if (e != cudaSuccess) return e;
      return launch_k(finalize_cta_kernel<16>, dim3((unsigned)a.q), dim3(16 * 32), smem, s, a);
    }
    const size_t smem = sizeof(FinBufs) * kFinW;
    static size_t attr = 0;
    const cudaError_t e = ensure_smem_attr(finalize_cta_kernel<kFinW>, smem, attr);
    if (e != cudaSuccess) return e;
    return launch_k(finalize_cta_kernel<kFinW>, dim3((unsigned)a.q), dim3(kFinW * 32), smem, s, a);
  }
  const dim3 grid((unsigned)((a.q + kFinGroup - 1) / kFinGroup));
  if (a.kprime <= 64) return launch_k(finalize_warp_kernel<256, 64>, grid, dim3(kFinGroup * 32), 0, s, a);
  if (a.kprime <= 128) return launch_k(finalize_warp_kernel<256, 128>, grid, dim3(kFinGroup * 32), 0, s, a);
  return launch_k(finalize_warp_kernel<kBufCap, kFinMaxSel>, grid, dim3(kFinGroup * 32), 0, s, a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K10' merge

// One query of the K10' merge (one CTA): the k best of C candidates by (dist, global id) --
// block_select_top by key, then a warp sort -- written best-first with padding.
template <typename Get>
__device__ void merge_query(Get get, int64_t C, int k, int metric, int64_t j, int64_t *ids, float *dists) {
  __shared__ int64_t s_id[kFinMaxSel];
  __shared__ float s_key[kFinMaxSel];
  __shared__ double s_k2[kFinMaxSel];
  __shared__ int64_t s_i2[kFinMaxSel];
  const int tid = threadIdx.x, warp = tid >> 5;
  const int m = block_select_top<int64_t>(get, C, k, s_id, s_key);
  int np = 1;
  while (np < m) np <<= 1;
  for (int c = tid; c < np; c += kFinThreads) {
    s_k2[c] = c < m ? (double)s_key[c] : -INFINITY;
    s_i2[c] = c < m ? s_id[c] : INT64_MAX;
  }
  __syncthreads();
  if (warp == 0 && m > 1) warp_sort_desc_d(s_k2, s_i2, np);
  __syncthreads();
  const float pad = metric == VRS_L2 ? INFINITY : -INFINITY;
  for (int r = tid; r < k; r += kFinThreads) {
    const int64_t o = j * k + r;
    if (r < m) {
      ids[o] = s_i2[r];
      const float kv = (float)s_k2[r];
      dists[o] = metric == VRS_L2 ? -kv : kv;
    } else {
      ids[o] = -1;
      dists[o] = pad;
    }
  }
  __syncthreads();   // (shared buffers reused by the CTA's next query)
}

__global__ void __launch_bounds__(kFinThreads) merge_kernel(MergeArgs a) {
  TL_SCOPE(2);
  const int64_t j = blockIdx.x;
  pdl_wait();
  TL_WAITED(2);
  pdl_trigger();
  auto get = [&](int64_t c, float &key, int64_t &id) -> bool {
    const int64_t p = c / a.k, r = c - p * a.k;
    const int64_t o = (p * a.q + j) * a.k + r;
    id = a.cand_ids[o];
    const float dv = a.cand_dists[o];
    key = a.metric == VRS_L2 ? -dv : dv;
    return id >= 0;
  };
  merge_query(get, (int64_t)a.parts * a.k, a.k, a.metric, j, a.ids, a.dists);
}

// ------------------------------------------------------------------ K10'' push-merge
// The multi-GPU exchange + merge in one kernel over peer memory (NVLink P2P through
// symmetric-memory buffers; SURVEY 8(e) mitigation 2): every rank pushes its exact local
// [q x k] results into its slot of every rank's receive buffer (one-shot P2P stores), counts
// the push on each peer with a system-scope atomic, waits until every source's pushes of
// this call arrived, and merges its queries from its own buffer -- no all-gather launch, no
// host involvement.  Receive buffer of rank p (peer_bufs[p]): uint32 counts[64] (pushes
// received from each source, cumulative), then slots [2 parities][parts][q][k] of (int64 id)
// followed by (fp32 dist).  The call's epoch e (device state, so CUDA-graph replays advance
// it) picks the parity: a rank can run at most one call ahead of a peer (its merge waits for
// the peer's push), so the slot a faster rank overwrites was read by the slower one a call
// ago.  The grid (<= 2 CTAs per SM) is resident: every CTA's wait on all sources' pushes
// cannot block a CTA it waits for.  The wait is bounded (wait_ns, VRS_PUSH_TIMEOUT_MS).
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__global__ void __launch_bounds__(kFinThreads) push_merge_kernel(PushMergeArgs a) {
  pdl_wait();
  const int tid = threadIdx.x;
  const uint32_t e = a.state[0] + 1u, par = e & 1u, base = a.state[2];
  const uint32_t nblk = gridDim.x;
  const int64_t qk = a.q * a.k;
  auto slot = [&](const void *buf, uint32_t src) {
    return reinterpret_cast<int64_t *>(static_cast<char *>(const_cast<void *>(buf)) + kPushHeader +
                                       ((int64_t)(par * (uint32_t)a.parts + src) * qk) * 12);
  };
  // (1) push this CTA's queries to every rank (itself included)
  for (int p = 0; p < a.parts; ++p) {
    int64_t *di = slot(a.peer_bufs[p], (uint32_t)a.my_part);
    float *dd = reinterpret_cast<float *>(di + qk);
    for (int64_t j = blockIdx.x; j < a.q; j += nblk)
      for (int r = tid; r < a.k; r += kFinThreads) {
        const int64_t o = j * a.k + r;
        di[o] = a.local_ids[o];
        dd[o] = a.local_dists[o];
      }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    for (int p = 0; p < a.parts; ++p) atomicAdd_system(static_cast<uint32_t *>(a.peer_bufs[p]) + a.my_part, 1u);
  }
  // (2) every source's pushes of this call (all its CTAs) have landed in this rank's buffer
  const uint32_t *cnt = static_cast<const uint32_t *>(a.peer_bufs[a.my_part]);
  // (bounded: a peer that never calls -- a dead rank, a transport that does not deliver --
  // must not hang the GPU; the flag in state[3] tells the host the results are invalid)
  if (tid < a.parts) {
    uint64_t t0 = 0;
    while ((int32_t)(ld_acquire_sys(cnt + tid) - (base + nblk)) < 0) {
      uint64_t now;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
      if (t0 == 0) t0 = now;
      else if (now - t0 > a.wait_ns) {
        atomicOr(a.state + 3, 1u);
        break;
      }
    }
  }
  __syncthreads();
  // (3) merge this CTA's queries from the parts' slots
  const void *mine = a.peer_bufs[a.my_part];
  for (int64_t j = blockIdx.x; j < a.q; j += nblk) {
    auto get = [&](int64_t c, float &key, int64_t &id) -> bool {
      const uint32_t src = (uint32_t)(c / a.k);
      const int64_t r = c - (int64_t)src * a.k;
      const int64_t *si = slot(mine, src);
      const float *sd = reinterpret_cast<const float *>(si + qk);
      id = si[j * a.k + r];
      const float dv = sd[j * a.k + r];
      key = a.metric == VRS_L2 ? -dv : dv;
      return id >= 0;
    };
    merge_query(get, (int64_t)a.parts * a.k, a.k, a.metric, j, a.ids, a.dists);
  }
  // (4) the call's bookkeeping, by the last CTA to finish (every CTA read the state at its start)
  if (tid == 0) {
    __threadfence();
    const uint32_t t = atomicAdd(a.state + 1, 1u);
    if (t == nblk - 1) {
      a.state[1] = 0;
      a.state[2] = base + nblk;
      a.state[0] = e;
      __threadfence();
    }
  }
}

cudaError_t launch_push_merge(const PushMergeArgs &a, cudaStream_t s, int *launches) {
  if (launches) *launches += 1;
  const unsigned blocks = (unsigned)std::min<int64_t>(a.q, 2 * kSmCountB200);
  return launch_k(push_merge_kernel, dim3(blocks), dim3(kFinThreads), 0, s, a);
}

cudaError_t launch_merge(const MergeArgs &a, cudaStream_t s, int *launches) {
  if (launches) *launches += 1;
  return launch_k(merge_kernel, dim3((unsigned)a.q), dim3(kFinThreads), 0, s, a);
  return cudaGetLastError();
}

}  // namespace vrs

#ifdef VRS_TC_TIMING
namespace vrs {
int tl_read_fin(unsigned long long *host) { return tl_read(host); }
}
#endif
