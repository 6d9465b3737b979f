// gemm_range.cu -- range (threshold) selection on the tensor-core pass.
//
// The paper's own scan metric is a threshold, not a top-k: "We use cosine
// similarity > 0.9" (Sec. 5), and the exhaustive scan is the
// fall-back for "range instead of top-k search" (L1436, Sec. 6).  Result
// contract: per query every qualifying row whose score
// satisfies the threshold (>= tau for IP / COS, <= tau for squared L2 --
// reading R14), ascending row id, scores exact.
//
// Pipeline (vrs_range_search in vrs_api.cu drives it):
//   range_threshold_kernel  per query, the ranking-key threshold T_j that every
//                           row passing tau provably reaches under the tensor-core
//                           (16-bit / TF32) key error bound, i.e. tau minus a margin
//   tc pass MODE_RCOUNT     per (list, query): how many keys >= T_j
//   range_prefix_kernel     (query, list) segment offsets, total C
//   -- host: read C, size the candidate buffer --
//   tc pass MODE_RFILL      each list writes its candidates' row ids, ascending
//   range_verify_kernel     exact fp64 score of every candidate, keep iff it
//                           satisfies tau (the definition's own comparison)
//   range_prefix_kernel     per-query result offsets (the caller's), total R
//   -- host: read R, check the caller's capacity --
//   range_write_kernel      per query, the kListsPerSplit lists of each split merged by row
//                           id, splits in order -> ascending ids, exact dists
#include "tc_kernel.cuh"

namespace vrs {

// ---------------------------------------------------------------- thresholds
// Key domain (rank_key): L2 -> 2<q,x> - |x|^2, IP -> <q,x>, COS -> <q,x>/|x|, the
// IP / COS keys of 16-bit operands scaled by D = 2^(e_q + e_x) (tc_kernel.cuh).
// With |computed key - exact key| <= E (vrs_internal.cuh key_error_bound, the same
// bound as the top-k certificate):
//   IP : <q,x> >= tau        => key >= (tau - E) D
//   COS: cos >= tau          => key >= (tau |q| - E) D    (exact key = cos |q|)
//   L2 : |q-x|^2 <= tau      => key >= |q|^2 - tau - E
// plus a relative slack for the fp64 arithmetic here; rounded toward -inf to fp32.
// Rows below T_j can therefore never pass tau.
__global__ void __launch_bounds__(128) range_threshold_kernel(const float *__restrict__ Q, int64_t q, int32_t d,
                                                              int32_t metric, double tau, KeyBound kb,
                                                              const int32_t *__restrict__ qexp,
                                                              const float *__restrict__ rq, int32_t xexp,
                                                              uint32_t *__restrict__ gtau) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (j >= q) return;
  const float *qv = Q + j * d;
  double qq = 0.0;
  for (int t = lane; t < d; t += 32) qq += (double)qv[t] * (double)qv[t];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) qq += __shfl_xor_sync(0xffffffffu, qq, o);
  if (lane) return;
  const double nq = sqrt(qq), rel = 0x1p-30, N = kb.xmax;
  const double E = key_error_bound(kb, metric, nq, rq ? (double)rq[j] : 0.0);
  const double D = (qexp && metric != VRS_L2) ? ldexp(1.0, qexp[j] + xexp) : 1.0;
  double T;
  if (metric == VRS_IP) {
    T = (tau - E - rel * (fabs(tau) + nq * N)) * D;
  } else if (metric == VRS_COSINE) {
    T = qq > 0.0 ? (tau * nq - E - rel * nq * (1.0 + fabs(tau))) * D : INFINITY;   // zero query: nothing
  } else {
    T = qq - tau - E - rel * (fabs(qq - tau) + N * N + 2.0 * nq * N);
  }
  gtau[j] = ordered_u32(__double2float_rd(T));
}

// ---------------------------------------------------------------- prefix sums
// out[e] = sum of v(e') for e' < e, out[m] = total, over m values
// v(e) = cnt[(e % L) * q + e / L] (L > 1: counts laid out [list][q], offsets
// query-major) or cnt[e] (L == 1).  One CTA of 1024 threads.
__global__ void __launch_bounds__(1024) range_prefix_kernel(const int32_t *__restrict__ cnt, int64_t q, int32_t L,
                                                            int64_t *__restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ int64_t s_warp[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m = q * L;
  const int64_t per = (m + 1023) / 1024;
  const int64_t e0 = tid * per, e1 = min(m, e0 + per);
  auto val = [&](int64_t e) -> int64_t { return L > 1 ? cnt[(e % L) * q + e / L] : cnt[e]; };
  int64_t sum = 0;
  for (int64_t e = e0; e < e1; ++e) sum += val(e);
  int64_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t w = s_warp[lane], wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    s_warp[lane] = wi - w;   // exclusive over warps
  }
  __syncthreads();
  int64_t run = s_warp[warp] + incl - sum;
  for (int64_t e = e0; e < e1; ++e) {
    out[e] = run;
    run += val(e);
  }
  if (tid == 1023) out[m] = run;
}

// ---------------------------------------------------------------- verify
// One CTA (8 warps) per query: the exact fp64 score of every candidate (the
// definition: sequential-in-lane, butterfly-reduced sums of the fp32 inputs
// widened to fp64), keep iff it satisfies tau, count the kept rows.
constexpr int kRvWarps = 8;
__global__ void __launch_bounds__(kRvWarps * 32) range_verify_kernel(const float *__restrict__ X, int32_t d,
                                                                     const float *__restrict__ Q, int32_t metric,
                                                                     double tau, const int32_t *__restrict__ cand,
                                                                     const int64_t *__restrict__ coff, int32_t L,
                                                                     double *__restrict__ score,
                                                                     uint8_t *__restrict__ keep,
                                                                     int32_t *__restrict__ kept) {
  pdl_wait();
  pdl_trigger();
  __shared__ int s_cnt[kRvWarps];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = blockIdx.x;
  const int64_t c_begin = coff[j * L], c_end = coff[(j + 1) * L];
  const float *qv = Q + j * d;
  double qq = 0.0;
  if (metric == VRS_COSINE) {
    for (int t = lane; t < d; t += 32) qq += (double)qv[t] * (double)qv[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) qq += __shfl_xor_sync(0xffffffffu, qq, o);
  }
  int mine = 0;
  constexpr int U = 4;
  for (int64_t c0 = c_begin + (int64_t)w * U; c0 < c_end; c0 += kRvWarps * U) {
    const float *xr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xr[u] = X + (int64_t)cand[min(c0 + u, c_end - 1)] * d;
    double s[U], xx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { s[u] = 0.0; xx[u] = 0.0; }
    for (int t = lane; t < d; t += 32) {
      const double qt = qv[t];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double xt = __ldg(xr[u] + t);
        if (metric == VRS_L2) { const double df = qt - xt; s[u] += df * df; }
        else { s[u] += qt * xt; xx[u] += xt * xt; }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s[u] += __shfl_xor_sync(0xffffffffu, s[u], o);
        if (metric == VRS_COSINE) xx[u] += __shfl_xor_sync(0xffffffffu, xx[u], o);
      }
      const int64_t c = c0 + u;
      if (lane == u && c < c_end) {
        double v = s[u];
        if (metric == VRS_COSINE) v = qq > 0.0 ? v / (sqrt(qq) * sqrt(xx[u])) : -INFINITY;
        const bool k = metric == VRS_L2 ? (v <= tau) : (v >= tau);
        score[c] = v;
        keep[c] = k ? 1 : 0;
        mine += k ? 1 : 0;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if (lane == 0) s_cnt[w] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < kRvWarps; ++i) t += s_cnt[i];
    kept[j] = t;
  }
}

// ---------------------------------------------------------------- write
// One CTA per query: thread t owns a contiguous run of splits; per split the
// two (ascending) lists of its column halves are merged by row id, kept rows
// only; runs are written in split order after a block scan of their sizes.
constexpr int kRwThreads = 256;
__global__ void __launch_bounds__(kRwThreads) range_write_kernel(const int32_t *__restrict__ cand,
                                                                 const int64_t *__restrict__ coff, int32_t P,
                                                                 const double *__restrict__ score,
                                                                 const uint8_t *__restrict__ keep,
                                                                 const int64_t *__restrict__ offsets,
                                                                 int64_t row_offset, int64_t *__restrict__ ids,
                                                                 float *__restrict__ dists) {
  pdl_wait();
  pdl_trigger();
  __shared__ int64_t s_warp[kRwThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t j = blockIdx.x;
  constexpr int LPS = kListsPerSplit;
  const int L = LPS * P;
  const int per = (P + kRwThreads - 1) / kRwThreads;
  const int s0 = min(P, tid * per), s1 = min(P, s0 + per);
  const int64_t *seg = coff + j * L;
  int64_t mine = 0;
  for (int64_t c = seg[LPS * s0]; c < seg[LPS * s1]; ++c) mine += keep[c];
  int64_t incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  int64_t before = 0;
  for (int i = 0; i < warp; ++i) before += s_warp[i];
  int64_t o = offsets[j] + before + incl - mine;
  for (int s = s0; s < s1; ++s) {
    // the split's LPS lists (each ascending, interleaved column ranges) merged by row id
    int64_t h[LPS], he[LPS];
#pragma unroll
    for (int l = 0; l < LPS; ++l) { h[l] = seg[LPS * s + l]; he[l] = seg[LPS * s + l + 1]; }
    for (;;) {
      int best = -1;
      int32_t bid = 0;
#pragma unroll
      for (int l = 0; l < LPS; ++l)
        if (h[l] < he[l] && (best < 0 || cand[h[l]] < bid)) { best = l; bid = cand[h[l]]; }
      if (best < 0) break;
      int64_t c = 0;
#pragma unroll
      for (int l = 0; l < LPS; ++l)
        if (l == best) c = h[l]++;
      if (!keep[c]) continue;
      ids[o] = row_offset + cand[c];
      dists[o] = (float)score[c];
      ++o;
    }
  }
}

// ---------------------------------------------------------------- host
TcLaunch *range_tc_alloc() { return new TcLaunch(); }
void range_tc_free(TcLaunch *t) { delete t; }

cudaError_t launch_range_count(const GemmArgs &a, const GemmPlan &plan, RangeState &r, cudaStream_t s,
                               int *launches) {
  TcLaunch &L = *r.tc;
  cudaError_t e = tc_prepare(a, plan, s, launches, &L);
  if (e != cudaSuccess) return e;
  e = launch_k(range_threshold_kernel, dim3((unsigned)((a.q + 3) / 4)), dim3(128), 0, s, a.Q, a.q, a.d, a.metric,
               r.tau, r.kb, (const int32_t *)(a.bf16 ? a.qexp : nullptr), (const float *)(a.bf16 ? a.rq : nullptr),
               a.bf16 ? a.xexp : 0, r.gtau);
  if (e != cudaSuccess) return e;
  TcParams p = L.p;
  p.gtau = r.gtau;
  p.cand_cnt = r.cand_cnt;
  {
    ProfScope ps("range.count", s);
    e = tc_launch_mode<MODE_RCOUNT>(L, p, s);
    if (e != cudaSuccess) return e;
  }
  e = launch_k(range_prefix_kernel, dim3(1), dim3(1024), 0, s, (const int32_t *)r.cand_cnt, a.q, kListsPerSplit * plan.P, r.coff);
  if (launches) *launches += 3;
  return e;
}

cudaError_t launch_range_fill(const GemmArgs &a, const GemmPlan &plan, RangeState &r, cudaStream_t s,
                              int *launches) {
  TcLaunch &L = *r.tc;
  TcParams p = L.p;
  p.gtau = r.gtau;
  p.cand_id = r.cand;
  p.coff = r.coff;
  cudaError_t e;
  {
    ProfScope ps("range.fill", s);
    e = tc_launch_mode<MODE_RFILL>(L, p, s);
    if (e != cudaSuccess) return e;
  }
  {
    ProfScope ps("range.verify", s);
    e = launch_k(range_verify_kernel, dim3((unsigned)a.q), dim3(kRvWarps * 32), 0, s, a.X, a.d, a.Q, a.metric, r.tau,
                 (const int32_t *)r.cand, (const int64_t *)r.coff, kListsPerSplit * plan.P, r.score, r.keep, r.kept);
    if (e != cudaSuccess) return e;
  }
  e = launch_k(range_prefix_kernel, dim3(1), dim3(1024), 0, s, (const int32_t *)r.kept, a.q, 1, r.offsets);
  if (launches) *launches += 3;
  return e;
}

cudaError_t launch_range_write(const GemmArgs &a, const GemmPlan &plan, RangeState &r, cudaStream_t s,
                               int *launches) {
  if (launches) *launches += 1;
  return launch_k(range_write_kernel, dim3((unsigned)a.q), dim3(kRwThreads), 0, s, (const int32_t *)r.cand,
                  (const int64_t *)r.coff, plan.P, (const double *)r.score, (const uint8_t *)r.keep,
                  (const int64_t *)r.offsets, r.row_offset, r.ids, r.dists);
}

}  // namespace vrs
