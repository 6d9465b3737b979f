// exact.cu -- the certificate's fallback ("Certified exactness").
//
// finalize.cu certifies each query's result: the k-th exact score of the
// re-scored candidates must beat every unselected row's selection key plus the
// key error bound.  A query that fails (selection-precision ties, clustered
// data, adversarial inputs) is recomputed here from the definition itself
// (sigma_eps(v x sigma_theta(R)); Table 1 "Accuracy:
// Exact"): the exact fp64 score of EVERY qualifying row, the k best by (score,
// lower id).  One launch, no host synchronisation: the kernel reads the
// certificate flags itself and returns at once when every query is certified.
//
// Work: the uncertified queries in groups of up to 8 (the rows are read once per
// group), each group's row space split over the grid.  Each CTA keeps, per query,
// the rows scoring at least finalize's k-th sort key (no row below it can enter:
// k rows already reach it) in a shared-memory buffer, compacted to the k best
// when it fills; its best k go to a slot; the CTA finishing a group's last split
// merges the group's slots and overwrites the queries' results.
//
// Roofline: HBM (4d bytes per qualifying row per group) -- rarely launched work.
#include <float.h>

#include <algorithm>

#include "vrs_kernels.cuh"

namespace vrs {

constexpr int kExWarps = 8;
constexpr int kExThreads = kExWarps * 32;
constexpr int kExQG = 8;       // queries per group (max)
constexpr int kExCap = 512;    // buffered rows per query (>= k + 16 per batch; k <= VRS_K_MAX)
constexpr int kExGrid = 148;   // one CTA per SM
constexpr int kExQSmem = 96 * 1024;

// descending (key, id asc) bitonic sort of n = 2^p (double, int64) pairs in shared memory, one warp
__device__ void ex_sort_desc(double *key, int64_t *id, int n) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= n; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncwarp();
      for (int t = lane; t < (n >> 1); t += 32) {
        const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
        const bool desc = (lo & size) == 0;
        const double ka = key[lo], kb = key[hi];
        const int64_t ia = id[lo], ib = id[hi];
        const bool b_first = (kb > ka) || (kb == ka && ib < ia);
        const bool a_first = (ka > kb) || (ka == kb && ia < ib);
        if (desc ? b_first : a_first) { key[lo] = kb; key[hi] = ka; id[lo] = ib; id[hi] = ia; }
      }
    }
  __syncwarp();
}

// one warp: sort the query's buffer and keep its k best (count -> min(count, k))
__device__ void ex_compact(double *key, int64_t *id, int &cnt, int k) {
  const int lane = threadIdx.x & 31;
  for (int i = cnt + lane; i < kExCap; i += 32) { key[i] = -INFINITY; id[i] = INT64_MAX; }
  ex_sort_desc(key, id, kExCap);
  cnt = min(cnt, k);
}

int exact_group_size(int32_t d, int *q_smem) {
  const int64_t per = (int64_t)d * 4;
  int qg = (int)std::min<int64_t>(kExQG, std::max<int64_t>(1, kExQSmem / per));
  *q_smem = (int64_t)qg * per <= kExQSmem ? 1 : 0;
  return qg;
}
int64_t exact_items_max(int64_t q, int qg) { return std::max<int64_t>(kExGrid, (q + qg - 1) / qg); }

template <bool VEC>
__global__ void __launch_bounds__(kExThreads, 1) exact_fallback_kernel(ExactArgs a) {
  extern __shared__ __align__(16) uint8_t ex_smem[];
  double *s_key = reinterpret_cast<double *>(ex_smem);                  // [qg][kExCap]
  int64_t *s_id = reinterpret_cast<int64_t *>(s_key + kExQG * kExCap);   // [qg][kExCap]
  float *s_q = reinterpret_cast<float *>(s_id + kExQG * kExCap);         // [qg][d] (q_smem)
  __shared__ int s_cnt[kExQG];
  __shared__ double s_thr[kExQG], s_qq[kExQG];
  __shared__ int64_t s_qid[kExQG];
  __shared__ int s_wsum[kExWarps], s_last, s_full;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  pdl_wait();
  pdl_trigger();
  // ---- how many queries failed their certificate
  int u = 0;
  for (int64_t j = tid; j < a.q; j += kExThreads) u += a.cert[j] == 0 ? 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
  if (lane == 0) s_wsum[warp] = u;
  __syncthreads();
  int U = 0;
#pragma unroll
  for (int w = 0; w < kExWarps; ++w) U += s_wsum[w];
  if (U == 0) return;
  const int QG = a.qg;
  const int64_t ngroups = (U + QG - 1) / QG;
  const int64_t R = std::max<int64_t>(1, (int64_t)gridDim.x / ngroups);
  const int64_t n_space = a.ids ? *a.count : a.n;
  for (int64_t item = blockIdx.x; item < ngroups * R; item += gridDim.x) {
    const int64_t g = item / R, r = item - g * R;
    const int nq = (int)std::min<int64_t>(QG, U - g * QG);
    __syncthreads();   // (the previous item's shared state is no longer read)
    // ---- the group's queries: the uncertified ones of rank g*QG .. g*QG + nq - 1
    {
      int64_t base = 0;
      for (int64_t c0 = 0; c0 < a.q && base < g * QG + nq; c0 += kExThreads) {
        const int64_t j = c0 + tid;
        const bool f = j < a.q && a.cert[j] == 0;
        const uint32_t bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) s_wsum[warp] = __popc(bal);
        __syncthreads();
        int64_t before = base;
        for (int w = 0; w < warp; ++w) before += s_wsum[w];
        const int64_t rank = before + __popc(bal & lanemask_lt());
        if (f && rank >= g * QG && rank < g * QG + nq) s_qid[rank - g * QG] = j;
        int tot = 0;
        for (int w = 0; w < kExWarps; ++w) tot += s_wsum[w];
        __syncthreads();
        base += tot;
      }
    }
    __syncthreads();
    if (tid < nq) {
      const int64_t j = s_qid[tid];
      s_cnt[tid] = 0;
      const double skv = a.sk[j];
      // (fp64 sums in another order than finalize's: a slack of 2^-40 of the scale)
      s_thr[tid] = skv - 0x1p-40 * (fabs(skv) + a.xmax * a.xmax + 1e-300);
    }
    if (a.q_smem)
      for (int i = tid; i < nq * a.d; i += kExThreads) {
        const int qi = i / a.d;
        s_q[i] = __ldg(a.Q + s_qid[qi] * a.d + (i - qi * a.d));
      }
    __syncthreads();
    if (warp < nq) {   // |q|^2 (COS)
      const float *qv = a.Q + s_qid[warp] * a.d;
      double qq = 0.0;
      for (int t = lane; t < a.d; t += 32) qq += (double)__ldg(qv + t) * (double)__ldg(qv + t);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) qq += __shfl_xor_sync(0xffffffffu, qq, o);
      if (lane == 0) s_qq[warp] = qq;
    }
    __syncthreads();
    const float *qbase[kExQG];
#pragma unroll
    for (int i = 0; i < kExQG; ++i)
      qbase[i] = i < nq ? (a.q_smem ? s_q + i * a.d : a.Q + s_qid[i] * a.d) : (a.q_smem ? s_q : a.Q + s_qid[0] * a.d);
    // ---- this split's rows, 2 per warp per step
    const int64_t r0 = n_space * r / R, r1 = n_space * (r + 1) / R;
    for (int64_t b0 = r0; b0 < r1; b0 += 2 * kExWarps) {
      double acc[2][kExQG], xx[2];
      int32_t rid[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t pos = b0 + 2 * warp + h;
        rid[h] = pos < r1 ? (a.ids ? __ldg(a.ids + pos) : (int32_t)pos) : -1;
        xx[h] = 0.0;
#pragma unroll
        for (int i = 0; i < kExQG; ++i) acc[h][i] = 0.0;
      }
      if (VEC) {
        for (int t = 4 * lane; t < a.d; t += 128) {
          float4 xv[2];
#pragma unroll
          for (int h = 0; h < 2; ++h)
            xv[h] = rid[h] >= 0 ? __ldg(reinterpret_cast<const float4 *>(a.X + (int64_t)rid[h] * a.d + t))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int i = 0; i < kExQG; ++i) {
            if (i >= nq) break;
            const float4 qv = *reinterpret_cast<const float4 *>(qbase[i] + t);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (a.metric == VRS_L2) {
                const double d0 = (double)qv.x - xv[h].x, d1 = (double)qv.y - xv[h].y, d2 = (double)qv.z - xv[h].z,
                             d3 = (double)qv.w - xv[h].w;
                acc[h][i] += d0 * d0; acc[h][i] += d1 * d1; acc[h][i] += d2 * d2; acc[h][i] += d3 * d3;
              } else {
                acc[h][i] += (double)qv.x * xv[h].x; acc[h][i] += (double)qv.y * xv[h].y;
                acc[h][i] += (double)qv.z * xv[h].z; acc[h][i] += (double)qv.w * xv[h].w;
              }
            }
          }
          if (a.metric == VRS_COSINE)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              xx[h] += (double)xv[h].x * xv[h].x + (double)xv[h].y * xv[h].y + (double)xv[h].z * xv[h].z +
                       (double)xv[h].w * xv[h].w;
        }
      } else {
        for (int t = lane; t < a.d; t += 32) {
          double xv[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) xv[h] = rid[h] >= 0 ? (double)__ldg(a.X + (int64_t)rid[h] * a.d + t) : 0.0;
#pragma unroll
          for (int i = 0; i < kExQG; ++i) {
            if (i >= nq) break;
            const double qv = qbase[i][t];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (a.metric == VRS_L2) { const double df = qv - xv[h]; acc[h][i] += df * df; }
              else acc[h][i] += qv * xv[h];
            }
          }
          if (a.metric == VRS_COSINE)
#pragma unroll
            for (int h = 0; h < 2; ++h) xx[h] += xv[h] * xv[h];
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double tot = warp_sum_transpose<kExQG>(acc[h]);   // lane: query (lane >> 2) & 7
        double xt = xx[h];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) xt += __shfl_xor_sync(0xffffffffu, xt, o);
        const int i = (lane >> 2) & 7;
        if ((lane & 3) == 0 && i < nq && rid[h] >= 0) {
          double v = tot;
          if (a.metric == VRS_L2) v = -v;
          else if (a.metric == VRS_COSINE) v = s_qq[i] > 0.0 ? v / (sqrt(s_qq[i]) * sqrt(xt)) : -INFINITY;
          if (v >= s_thr[i]) {
            const int p = atomicAdd(&s_cnt[i], 1);
            s_key[i * kExCap + p] = v;
            s_id[i * kExCap + p] = rid[h];
          }
        }
      }
      __syncthreads();
      // make room for the next step's <= 2 * kExWarps appends per query
      if (tid == 0) {
        int full = 0;
        for (int i = 0; i < nq; ++i) full |= s_cnt[i] > kExCap - 2 * kExWarps;
        s_full = full;
      }
      __syncthreads();
      if (s_full) {
        if (warp < nq && s_cnt[warp] > kExCap - 2 * kExWarps) {
          int c = s_cnt[warp];
          ex_compact(s_key + warp * kExCap, s_id + warp * kExCap, c, a.k);
          if (lane == 0) {
            s_cnt[warp] = c;
            if (c >= a.k) s_thr[warp] = fmax(s_thr[warp], s_key[warp * kExCap + a.k - 1]);
          }
        }
        __syncthreads();
      }
    }
    // ---- this split's k best per query -> its slot
    if (warp < nq) {
      int c = s_cnt[warp];
      ex_compact(s_key + warp * kExCap, s_id + warp * kExCap, c, a.k);
      const int64_t so = (item * a.qg + warp);
      for (int e = lane; e < c; e += 32) {
        a.slot_key[so * a.k + e] = s_key[warp * kExCap + e];
        a.slot_id[so * a.k + e] = s_id[warp * kExCap + e];
      }
      if (lane == 0) a.slot_cnt[so] = c;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(a.gcnt + s_qid[0], 1) == (int)(R - 1);
    __syncthreads();
    if (!s_last) continue;
    __threadfence();
    // ---- the group's last split: merge every split's slot, write the k best
    if (warp < nq) {
      double *bk = s_key + warp * kExCap;
      int64_t *bi = s_id + warp * kExCap;
      int c = 0;
      for (int64_t rr = 0; rr < R; ++rr) {
        const int64_t so = ((g * R + rr) * a.qg + warp);
        const int sc = __ldcg(a.slot_cnt + so);
        if (c + sc > kExCap) ex_compact(bk, bi, c, a.k);
        for (int e = lane; e < sc; e += 32) {
          bk[c + e] = __ldcg(a.slot_key + so * a.k + e);
          bi[c + e] = __ldcg(a.slot_id + so * a.k + e);
        }
        c += sc;
        __syncwarp();
      }
      ex_compact(bk, bi, c, a.k);
      const int64_t j = s_qid[warp];
      const float pad = a.metric == VRS_L2 ? INFINITY : -INFINITY;
      for (int e = lane; e < a.k; e += 32) {
        const int64_t o = j * a.k + e;
        if (e < c) {
          a.out_ids[o] = a.row_offset + bi[e];
          a.out_dists[o] = (float)(a.metric == VRS_L2 ? -bk[e] : bk[e]);
        } else {
          a.out_ids[o] = -1;
          a.out_dists[o] = pad;
        }
      }
    }
  }
}

cudaError_t launch_exact(const ExactArgs &a, cudaStream_t s, int *launches) {
  const bool vec = (a.d % 4 == 0) && (((uintptr_t)a.X | (uintptr_t)a.Q) % 16 == 0);
  const size_t smem = (size_t)kExQG * kExCap * 16 + (a.q_smem ? (size_t)a.qg * a.d * 4 : 0);
  static size_t attr[2] = {0, 0};
  auto kern = vec ? exact_fallback_kernel<true> : exact_fallback_kernel<false>;
  const cudaError_t e = ensure_smem_attr(kern, smem, attr[vec ? 1 : 0]);
  if (e != cudaSuccess) return e;
  if (launches) *launches += 1;
  return launch_k(kern, dim3(kExGrid), dim3(kExThreads), smem, s, a);
}

}  // namespace vrs
