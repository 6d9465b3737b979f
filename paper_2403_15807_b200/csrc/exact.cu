// exact.cu -- the certificate's fallback ("Certified exactness").
//
// finalize.cu certifies each query's result: the k-th exact score of the
// re-scored candidates must beat every unselected row's selection key plus the
// key error bound.  A query that fails (selection-precision ties, clustered
// data, adversarial inputs) is recomputed here from the definition (PAPER.md
// L285-L288: sigma_eps(v x sigma_theta(R)); Table 1 "Accuracy: Exact"):
// every qualifying row is examined, and the k best by (exact score, lower id)
// are returned.  One launch, no host synchronisation: the kernel reads the
// certificate flags itself and returns at once when every query is certified.
//
// Per work item (a group of up to QG uncertified queries x a split of the row
// space), two stages:
//   filter  lane-per-row fp32 FFMA dot products of each qualifying row with the
//           group's queries (rows staged HBM -> shared memory by 16-byte
//           cp.async in a per-warp ring; queries in shared memory), keys as in
//           rank_key; a row survives for a query when its fp32 key reaches
//           s_k - E32, where s_k is finalize's k-th EXACT key -- k rows reach s_k,
//           and E32 bounds the fp32 key's error (vrs_internal.cuh, KEY_FP32), so no
//           row of the true top k is dropped;
//   exact   each survivor's fp64 score (coalesced warp re-read of the row); rows
//           at or above the k-th sort key go to a per-query shared buffer,
//           compacted to the k best by (score, lower id) when it fills.
// Each item's k best go to a slot; the CTA finishing a group's last split merges
// the group's slots and overwrites those queries' results.
//
// Roofline: HBM (4d bytes per qualifying row per query group) -- launched on
// every search, it works only when a certificate failed.
#include <float.h>

#include <algorithm>

#include "vrs_kernels.cuh"

namespace vrs {

constexpr int kExWarps = 8;
constexpr int kExThreads = kExWarps * 32;
constexpr int kExBatch = 64;    // survivors exact-scored between buffer checks (buffer: pow2 >= k + kExBatch)
constexpr int kExGrid = 148;    // one CTA per SM
constexpr int kExKC = 16;       // fp32 columns per staged chunk
constexpr int kExPad = kExKC + 4;
constexpr int kExStages = 2;
constexpr int kExSurv = 8192;   // survivor list; flushed before a step could overflow it
constexpr int kExQMax = 16;

__host__ __device__ constexpr int exact_cap(int k) {
  int c = 128;
  while (c < k + kExBatch) c <<= 1;
  return c;
}
__host__ __device__ constexpr size_t exact_smem_bytes(int qg, int dpad, int cap) {
  return (size_t)qg * cap * 16                                 // exact buffers (key, id)
         + (size_t)kExWarps * kExStages * 32 * kExPad * 4      // row stages
         + (size_t)kExSurv * 8                                 // survivors (row, query slot)
         + (size_t)qg * dpad * 4;                              // queries
}

int exact_group_size(int32_t d, int32_t k) {
  const int dpad = (d + kExKC - 1) / kExKC * kExKC;
  int qg = kExQMax;
  while (qg > 1 && exact_smem_bytes(qg, dpad, exact_cap(k)) > 200 * 1024) qg >>= 1;
  return qg;
}
int64_t exact_items_max(int64_t q, int qg) { return std::max<int64_t>(4 * kExGrid, (q + qg - 1) / qg); }

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

// one warp: sort the query's buffer (cap entries, a power of two) and keep its k best
__device__ void ex_compact(double *key, int64_t *id, int &cnt, int k, int cap) {
  const int lane = threadIdx.x & 31;
  for (int i = cnt + lane; i < cap; i += 32) { key[i] = -INFINITY; id[i] = INT64_MAX; }
  ex_sort_desc(key, id, cap);
  cnt = min(cnt, k);
}

// exact fp64 sort key of row `rid` for query row qv (one warp, coalesced): L2 -|q-x|^2, IP <q,x>, COS cos
template <bool VEC4>
__device__ double ex_exact(const ExactArgs &a, const float *qv, double qq, int32_t rid) {
  const int lane = threadIdx.x & 31;
  const float *x = a.X + (int64_t)rid * a.d;
  double s = 0.0, xx = 0.0;
  if (VEC4) {
    for (int t = 4 * lane; t < a.d; t += 128) {
      const float4 xv = __ldg(reinterpret_cast<const float4 *>(x + t));
      const float4 q4 = *reinterpret_cast<const float4 *>(qv + t);
      if (a.metric == VRS_L2) {
        const double d0 = (double)q4.x - xv.x, d1 = (double)q4.y - xv.y, d2 = (double)q4.z - xv.z, d3 = (double)q4.w - xv.w;
        s += d0 * d0; s += d1 * d1; s += d2 * d2; s += d3 * d3;
      } else {
        s += (double)q4.x * xv.x; s += (double)q4.y * xv.y; s += (double)q4.z * xv.z; s += (double)q4.w * xv.w;
        xx += (double)xv.x * xv.x + (double)xv.y * xv.y + (double)xv.z * xv.z + (double)xv.w * xv.w;
      }
    }
  } else {
    for (int t = lane; t < a.d; t += 32) {
      const double xv = __ldg(x + t), q1 = qv[t];
      if (a.metric == VRS_L2) { const double df = q1 - xv; s += df * df; }
      else { s += q1 * xv; xx += xv * xv; }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    xx += __shfl_xor_sync(0xffffffffu, xx, o);
  }
  if (a.metric == VRS_L2) return -s;
  if (a.metric == VRS_COSINE) return qq > 0.0 && xx > 0.0 ? s / (sqrt(qq) * sqrt(xx)) : -INFINITY;
  return s;
}

template <int QG, bool VEC4>
__global__ void __launch_bounds__(kExThreads, 1) exact_fallback_kernel(ExactArgs a) {
  extern __shared__ __align__(16) uint8_t ex_smem[];
  const int dpad = (a.d + kExKC - 1) / kExKC * kExKC;
  const int nk = dpad / kExKC;
  const int cap = exact_cap(a.k);
  double *s_key = reinterpret_cast<double *>(ex_smem);                       // [QG][cap]
  int64_t *s_id = reinterpret_cast<int64_t *>(s_key + QG * cap);              // [QG][cap]
  float *s_stage = reinterpret_cast<float *>(s_id + QG * cap);                // [warps][stages][32][kExPad]
  uint2 *s_surv = reinterpret_cast<uint2 *>(s_stage + kExWarps * kExStages * 32 * kExPad);   // (row, slot)
  float *s_q = reinterpret_cast<float *>(s_surv + kExSurv);                   // [QG][dpad]
  __shared__ int s_cnt[QG], s_nsurv;
  __shared__ double s_thr[QG], s_qq[QG];
  __shared__ float s_thr32[QG];
  __shared__ int64_t s_qid[QG];
  __shared__ int s_wsum[kExWarps], s_last;
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
  if (a.stats && blockIdx.x == 0 && tid == 0) atomicAdd(a.stats + 3, (unsigned long long)U);
  const int64_t ngroups = (U + QG - 1) / QG;
  const int64_t R = std::max<int64_t>(1, (2 * (int64_t)gridDim.x + ngroups - 1) / ngroups);
  const int64_t n_space = a.ids ? *a.count : a.n;
  KeyBound kb32{};
  kb32.kind = KEY_FP32;
  kb32.d = a.d;
  kb32.xmax = a.xmax;
  float *wst = s_stage + warp * kExStages * 32 * kExPad;

  // survivors -> exact fp64 scores -> per-query buffers (all threads; clears the list)
  auto flush = [&]() {
    const int ns = s_nsurv;
    for (int b0 = 0; b0 < ns; b0 += kExBatch) {
      for (int e = b0 + warp; e < min(ns, b0 + kExBatch); e += kExWarps) {
        const uint2 sv = s_surv[e];
        const int i = (int)sv.y;
        const double v = ex_exact<VEC4>(a, s_q + i * dpad, s_qq[i], (int32_t)sv.x);
        if (lane == 0 && v >= s_thr[i]) {
          const int p = atomicAdd(&s_cnt[i], 1);
          s_key[i * cap + p] = v;
          s_id[i * cap + p] = (int32_t)sv.x;
        }
      }
      __syncthreads();
      for (int w = warp; w < QG; w += kExWarps)   // room for the next batch
        if (s_cnt[w] > cap - kExBatch) {
          int c = s_cnt[w];
          ex_compact(s_key + w * cap, s_id + w * cap, c, a.k, cap);
          if (lane == 0) {
            s_cnt[w] = c;
            if (c >= a.k) s_thr[w] = fmax(s_thr[w], s_key[w * cap + a.k - 1]);
          }
        }
      __syncthreads();
    }
    if (tid == 0) s_nsurv = 0;
    __syncthreads();
  };

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
    for (int i = tid; i < QG * dpad; i += kExThreads) {
      const int qi = i / dpad, t = i - qi * dpad;
      s_q[i] = (qi < nq && t < a.d) ? __ldg(a.Q + s_qid[qi] * a.d + t) : 0.f;
    }
    if (tid == 0) s_nsurv = 0;
    __syncthreads();
    for (int w = warp; w < QG; w += kExWarps) {   // |q|^2, thresholds
      double qq = 0.0;
      for (int t = lane; t < a.d; t += 32) qq += (double)s_q[w * dpad + t] * (double)s_q[w * dpad + t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) qq += __shfl_xor_sync(0xffffffffu, qq, o);
      if (lane == 0) {
        s_qq[w] = qq;
        s_cnt[w] = 0;
        if (w < nq) {
          const double skv = a.sk[s_qid[w]], qn = sqrt(qq);
          // exact stage: finalize's k-th sort key, less a slack for fp64 sums in another order
          s_thr[w] = skv - 0x1p-40 * (fabs(skv) + (qn + a.xmax) * (qn + a.xmax));
          // filter: the fp32 key of a row scoring >= s_k is >= s_k (natural units) - E32
          const double nat = a.metric == VRS_L2 ? qq + skv : (a.metric == VRS_COSINE ? skv * qn : skv);
          s_thr32[w] = __double2float_rd(nat - key_error_bound(kb32, a.metric, qn, 0.0));
        } else {
          s_thr[w] = INFINITY;
          s_thr32[w] = INFINITY;
        }
      }
    }
    __syncthreads();
    // ---- filter: this split's rows, 256 per block step, one per lane
    const int64_t r0 = n_space * r / R, r1 = n_space * (r + 1) / R;
    for (int64_t b0 = r0; b0 < r1; b0 += kExThreads) {
      const int64_t pos = b0 + warp * 32 + lane;
      const int32_t myid = pos < r1 ? (a.ids ? __ldg(a.ids + pos) : (int32_t)pos) : -1;
      auto issue = [&](int kc) {
        float *buf = wst + (kc % kExStages) * 32 * kExPad;
        if (VEC4) {
#pragma unroll
          for (int h = 0; h < 4; ++h) {   // 32 rows x 4 x 16 B: lane -> (row lane/4 + 8h, part lane % 4)
            const int rr = (lane >> 2) + 8 * h, part = lane & 3;
            const int32_t idr = __shfl_sync(0xffffffffu, myid, rr);
            const int col = kc * kExKC + part * 4;
            const bool ok = idr >= 0 && col < a.d;
            cp_async16(buf + rr * kExPad + part * 4, ok ? (const void *)(a.X + (int64_t)idr * a.d + col) : a.X, ok);
          }
        } else {
#pragma unroll 4
          for (int rr = 0; rr < 32; ++rr) {
            const int32_t idr = __shfl_sync(0xffffffffu, myid, rr);
            for (int c = lane; c < kExKC; c += 32) {
              const int col = kc * kExKC + c;
              const bool ok = idr >= 0 && col < a.d;
              cp_async4(buf + rr * kExPad + c, ok ? (const void *)(a.X + (int64_t)idr * a.d + col) : a.X, ok);
            }
          }
        }
        cp_async_commit();
      };
      float acc[QG];
#pragma unroll
      for (int i = 0; i < QG; ++i) acc[i] = 0.f;
      issue(0);
      for (int kc = 0; kc < nk; ++kc) {
        if (kc + 1 < nk) issue(kc + 1);
        else cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        const float *xb = wst + (kc % kExStages) * 32 * kExPad + lane * kExPad;
        const float *qk = s_q + kc * kExKC;
#pragma unroll
        for (int c4 = 0; c4 < kExKC / 4; ++c4) {
          const float4 xv = *reinterpret_cast<const float4 *>(xb + c4 * 4);
#pragma unroll
          for (int i = 0; i < QG; ++i) {   // sequential in t: the KEY_FP32 bound's accumulation model
            const float4 qv = *reinterpret_cast<const float4 *>(qk + i * dpad + c4 * 4);
            acc[i] = fmaf(xv.x, qv.x, acc[i]);
            acc[i] = fmaf(xv.y, qv.y, acc[i]);
            acc[i] = fmaf(xv.z, qv.z, acc[i]);
            acc[i] = fmaf(xv.w, qv.w, acc[i]);
          }
        }
        __syncwarp();
      }
      cp_async_wait<0>();
      if (myid >= 0) {
        const float nx2 = a.metric == VRS_L2 ? __ldg(a.nx2 + myid) : 0.f;
        const float inx = a.metric == VRS_COSINE ? __ldg(a.inv_nx + myid) : 0.f;
#pragma unroll
        for (int i = 0; i < QG; ++i) {
          const float key = rank_key(a.metric, acc[i], nx2, inx);
          if (key >= s_thr32[i]) {
            const int p = atomicAdd(&s_nsurv, 1);
            s_surv[p] = make_uint2((uint32_t)myid, (uint32_t)i);
          }
        }
      }
      __syncthreads();
      if (s_nsurv > kExSurv - kExThreads * QG) flush();   // (a step adds <= 256 * QG)
    }
    flush();
    // ---- this split's k best per query -> its slot
    for (int w = warp; w < nq; w += kExWarps) {
      int c = s_cnt[w];
      ex_compact(s_key + w * cap, s_id + w * cap, c, a.k, cap);
      const int64_t so = item * a.qg + w;
      for (int e = lane; e < c; e += 32) {
        a.slot_key[so * a.k + e] = s_key[w * cap + e];
        a.slot_id[so * a.k + e] = s_id[w * cap + e];
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
    for (int w = warp; w < nq; w += kExWarps) {
      double *bk = s_key + w * cap;
      int64_t *bi = s_id + w * cap;
      int c = 0;
      for (int64_t rr = 0; rr < R; ++rr) {
        const int64_t so = (g * R + rr) * a.qg + w;
        const int sc = __ldcg(a.slot_cnt + so);
        if (c + sc > cap) ex_compact(bk, bi, c, a.k, cap);
        for (int e = lane; e < sc; e += 32) {
          bk[c + e] = __ldcg(a.slot_key + so * a.k + e);
          bi[c + e] = __ldcg(a.slot_id + so * a.k + e);
        }
        c += sc;
        __syncwarp();
      }
      ex_compact(bk, bi, c, a.k, cap);
      const int64_t j = s_qid[w];
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

template <int QG>
static cudaError_t launch_exact_qg(const ExactArgs &a, bool vec, size_t smem, cudaStream_t s) {
  static size_t attr[2] = {0, 0};
  auto kern = vec ? exact_fallback_kernel<QG, true> : exact_fallback_kernel<QG, false>;
  const cudaError_t e = ensure_smem_attr(kern, smem, attr[vec ? 1 : 0]);
  if (e != cudaSuccess) return e;
  return launch_k(kern, dim3(kExGrid), dim3(kExThreads), smem, s, a);
}

cudaError_t launch_exact(const ExactArgs &a, cudaStream_t s, int *launches) {
  const bool vec = (a.d % 4 == 0) && (((uintptr_t)a.X | (uintptr_t)a.Q) % 16 == 0);
  const int dpad = (a.d + kExKC - 1) / kExKC * kExKC;
  const size_t smem = exact_smem_bytes(a.qg, dpad, exact_cap(a.k));
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;   // (d beyond ~40k)
  if (launches) *launches += 1;
  switch (a.qg) {
    case 1: return launch_exact_qg<1>(a, vec, smem, s);
    case 2: return launch_exact_qg<2>(a, vec, smem, s);
    case 4: return launch_exact_qg<4>(a, vec, smem, s);
    case 8: return launch_exact_qg<8>(a, vec, smem, s);
    default: return launch_exact_qg<16>(a, vec, smem, s);
  }
}

}  // namespace vrs
