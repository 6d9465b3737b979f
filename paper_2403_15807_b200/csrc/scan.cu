// scan.cu -- K6' norms at load and K2' the per-tuple scan path with fused top-k.
//
// K2' realises the paper's per-tuple strategies for small query batches
// (1:1 / 1:N / N:1, "Explicit SIMD" L535) over the
// late-materialized selection (L319): the qualifying rows, addressed through
// the compacted id list (or the identity when theta_R is empty), are streamed
// HBM -> shared memory with 16-byte cp.async (LDGSTS) in a 3-stage per-warp
// ring; each lane owns one row and accumulates exact fp32 FFMA dot products
// against up to QG queries held in shared memory (read as broadcasts).  The
// score matrix never leaves the SM: each 256-row block's ranking keys go to a
// small shared buffer, warp j keeps query j's running top-k' (threshold in a
// register, warp-ballot append of rows that beat it, warp-cooperative bitonic
// merge when the append buffer fills).  One sorted list per (CTA, query) is
// written out; finalize.cu merges the lists and re-scores exactly.
//
// Roofline: HBM.  Algorithmic bytes per selected row: 4*d (vector) + 4 (id)
// + 8 (norm terms); per call + 4*d*q (queries) + 12*q*k (results).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <float.h>

#include <algorithm>

#include "vrs_kernels.cuh"

namespace vrs {

// ------------------------------------------------------------------ K6' norms
// |x|^2 and 1/|x| per row, computed once at vrs_load ("then
// normalized"): fp64 sums of the fp32 inputs, each rounded once to fp32 (2^-24
// relative -- the certificate's key bound counts on it).
// flags[0]: a zero-norm row exists (COSINE degenerate); flags[1]: the largest
// |x|^2 and flags[2]: the largest |x_t|, as float bits (non-negative floats order
// as integers) -- the error bounds use max |x|, the fp16 shadow's scale max |x_t|.
__global__ void norms_kernel(const float *__restrict__ X, int64_t n, int32_t d, float *__restrict__ nx2,
                             float *__restrict__ inv_nx, int32_t *__restrict__ flags) {
  __shared__ float s_max[8], s_amax[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
  double s = 0.0;
  float am = 0.f;
  if (row < n) {
    const float *x = X + row * d;
    for (int t = lane; t < d; t += 32) {
      const float v = x[t];
      s = fma((double)v, (double)v, s);
      am = fmaxf(am, fabsf(v));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
  }
  if (lane == 0) {
    const float s32 = __double2float_rn(s);
    if (row < n) {
      nx2[row] = s32;
      inv_nx[row] = s > 0.0 ? __double2float_rn(1.0 / sqrt(s)) : 0.f;
      if (!(s > 0.0)) atomicOr(flags, 1);
    }
    s_max[w] = __double2float_ru(s);
    s_amax[w] = am;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = s_max[0], a = s_amax[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
      m = fmaxf(m, s_max[i]);
      a = fmaxf(a, s_amax[i]);
    }
    atomicMax(flags + 1, __float_as_int(m));
    atomicMax(flags + 2, __float_as_int(a));
  }
}

cudaError_t launch_norms(const float *X, int64_t n, int32_t d, float *nx2, float *inv_nx, int32_t *flags,
                         cudaStream_t stream) {
  const int warps = 8;
  norms_kernel<<<(unsigned)((n + warps - 1) / warps), warps * 32, 0, stream>>>(X, n, d, nx2, inv_nx, flags);
  return cudaGetLastError();
}

// ------------------------------------------------------------------- K2' scan
constexpr int kScWarps = 8;
constexpr int kScThreads = kScWarps * 32;
constexpr int kScRows = kScThreads;  // rows per block iteration (one per lane)
constexpr int kScKC = 32;            // fp32 columns per stage
constexpr int kScStages = 3;
constexpr int kScPad = kScKC + 4;    // padded row stride in the stage (conflict-free LDS.128)


__host__ __device__ constexpr size_t scan_smem_bytes(int QG, int KPE, int dpad) {
  return (size_t)QG * dpad * 4                        // queries
         + (size_t)kScWarps * kScStages * 32 * kScPad * 4  // row stages
         + (size_t)2 * QG * kScRows * 4                  // key double buffer
         + (size_t)2 * kScRows * 4                       // row-id double buffer
         + (size_t)QG * 2 * KPE * 8;                     // per-query list + append buffer
}

// ESZ: row element size -- 4 (the fp32 corpus) or 2 (the index's 16-bit shadow: half
// the bytes; the value read is x~ = 16-bit(x 2^e_x), its dot products are scaled back by
// 2^-e_x exactly, the queries stay fp32).  A stage holds 128 bytes of each row either way.
template <int QG, int KPE, bool VEC4, int ESZ>
__global__ void __launch_bounds__(kScThreads, 1) scan_topk_kernel(ScanArgs a) {
  extern __shared__ __align__(16) float smem[];
  constexpr int KCE = kScKC * 4 / ESZ;   // elements per 128-byte stage chunk
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = a.d;
  const int dpad = (d + KCE - 1) / KCE * KCE;
  const int nk = dpad / KCE;
  const char *xbase = ESZ == 4 ? reinterpret_cast<const char *>(a.X) : static_cast<const char *>(a.Xh);

  float *q_s = smem;
  float *stage = q_s + QG * dpad;
  float *sc = stage + kScWarps * kScStages * 32 * kScPad;
  int32_t *sid = reinterpret_cast<int32_t *>(sc + 2 * QG * kScRows);
  float *lk = reinterpret_cast<float *>(sid + 2 * kScRows);
  int32_t *li = reinterpret_cast<int32_t *>(lk + QG * 2 * KPE);

  const int64_t q0 = a.q_base + (int64_t)blockIdx.y * QG;
  const int nq = (int)(a.q - q0 < QG ? a.q - q0 : QG);
  pdl_wait();
  pdl_trigger();

  for (int i = threadIdx.x; i < QG * dpad; i += kScThreads) {
    const int j = i / dpad, t = i - j * dpad;
    q_s[i] = (j < nq && t < d) ? a.Q[(q0 + j) * d + t] : 0.f;
  }
  for (int i = threadIdx.x; i < QG * 2 * KPE; i += kScThreads) {
    lk[i] = -INFINITY;
    li[i] = -1;
  }

  const int64_t n_sel = a.ids ? *a.count : a.n;
  int64_t chunk = (n_sel + a.P - 1) / a.P;
  chunk = (chunk + kScRows - 1) / kScRows * kScRows;
  const int64_t start = (int64_t)blockIdx.x * chunk;
  const int64_t end = min(n_sel, start + chunk);
  const int niter = end > start ? (int)((end - start + kScRows - 1) / kScRows) : 0;
  __syncthreads();

  float *wst = stage + warp * kScStages * 32 * kScPad;
  const int total = niter * nk;

  auto row_id = [&](int it, int r) -> int32_t {
    const int64_t pos = start + (int64_t)it * kScRows + warp * 32 + r;
    if (pos >= end) return -1;
    return a.ids ? __ldg(a.ids + pos) : (int32_t)pos;
  };
  auto issue = [&](int t) {
    const int it = t / nk, kc = t - it * nk;
    float *buf = wst + (t % kScStages) * 32 * kScPad;
    const int32_t myid = row_id(it, lane);
    if constexpr (VEC4) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = (lane >> 3) + 4 * i;
        const int32_t idr = __shfl_sync(0xffffffffu, myid, r);
        const int col = kc * KCE + (lane & 7) * (16 / ESZ);
        const bool ok = idr >= 0 && col < d;
        cp_async16(buf + r * kScPad + (lane & 7) * 4, ok ? (const void *)(xbase + ((int64_t)idr * d + col) * ESZ) : xbase,
                   ok);
      }
    } else {
#pragma unroll 4
      for (int r = 0; r < 32; ++r) {
        const int32_t idr = __shfl_sync(0xffffffffu, myid, r);
        const int col = kc * kScKC + lane;
        const bool ok = idr >= 0 && col < d;
        cp_async4(buf + r * kScPad + lane, ok ? (const void *)(a.X + (int64_t)idr * d + col) : a.X, ok);
      }
    }
    cp_async_commit();
  };

#pragma unroll
  for (int t = 0; t < kScStages - 1; ++t) {
    if (t < total) issue(t);
    else cp_async_commit();
  }

  float acc[QG];
#pragma unroll
  for (int j = 0; j < QG; ++j) acc[j] = 0.f;
  float tau = -INFINITY;  // warp j's running k'-th best key of query j
  int cnt = 0;            // entries in warp j's append buffer
  float *L = lk + warp * 2 * KPE;
  int32_t *I = li + warp * 2 * KPE;

  auto merge = [&]() {
    for (int i = cnt + lane; i < KPE; i += 32) {
      L[KPE + i] = -INFINITY;
      I[KPE + i] = -1;
    }
    warp_bitonic_sort_desc(L, I, 2 * KPE);
    tau = L[a.kprime - 1];
    cnt = 0;
  };

  for (int t = 0; t < total; ++t) {
    if (t + kScStages - 1 < total) issue(t + kScStages - 1);
    else cp_async_commit();
    cp_async_wait<kScStages - 1>();
    __syncwarp();
    const int kc = t % nk;
    const float *buf = wst + (t % kScStages) * 32 * kScPad + lane * kScPad;
    const float *qk = q_s + kc * KCE;
    if constexpr (ESZ == 4) {
#pragma unroll
      for (int c4 = 0; c4 < kScKC / 4; ++c4) {
        const float4 rv = *reinterpret_cast<const float4 *>(buf + c4 * 4);
#pragma unroll
        for (int j = 0; j < QG; ++j) {
          const float4 qv = *reinterpret_cast<const float4 *>(qk + j * dpad + c4 * 4);
          acc[j] = fmaf(rv.x, qv.x, acc[j]);
          acc[j] = fmaf(rv.y, qv.y, acc[j]);
          acc[j] = fmaf(rv.z, qv.z, acc[j]);
          acc[j] = fmaf(rv.w, qv.w, acc[j]);
        }
      }
    } else {   // 16-bit rows: 8 elements per 16 bytes, converted exactly to fp32
#pragma unroll
      for (int c8 = 0; c8 < kScKC / 4; ++c8) {
        const uint4 raw = *reinterpret_cast<const uint4 *>(buf + c8 * 4);
        float xv[8];
        const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          float2 f;
          if (a.fmt16 == 0) f = __half22float2(*reinterpret_cast<const __half2 *>(&w[h]));
          else f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&w[h]));
          xv[2 * h] = f.x;
          xv[2 * h + 1] = f.y;
        }
#pragma unroll
        for (int j = 0; j < QG; ++j) {
          const float4 q0 = *reinterpret_cast<const float4 *>(qk + j * dpad + c8 * 8);
          const float4 q1 = *reinterpret_cast<const float4 *>(qk + j * dpad + c8 * 8 + 4);
          acc[j] = fmaf(xv[0], q0.x, acc[j]);
          acc[j] = fmaf(xv[1], q0.y, acc[j]);
          acc[j] = fmaf(xv[2], q0.z, acc[j]);
          acc[j] = fmaf(xv[3], q0.w, acc[j]);
          acc[j] = fmaf(xv[4], q1.x, acc[j]);
          acc[j] = fmaf(xv[5], q1.y, acc[j]);
          acc[j] = fmaf(xv[6], q1.z, acc[j]);
          acc[j] = fmaf(xv[7], q1.w, acc[j]);
        }
      }
    }
    __syncwarp();
    if (kc == nk - 1) {
      // ---- one 256-row block done: ranking keys -> shared, then per-query selection
      const int it = t / nk, b = it & 1;
      const int32_t myid = row_id(it, lane);
      float nx2 = 0.f, inx = 0.f;
      if (myid >= 0) {
        nx2 = __ldg(a.nx2 + myid);
        inx = __ldg(a.inv_nx + myid);
      }
#pragma unroll
      for (int j = 0; j < QG; ++j) {
        sc[(b * QG + j) * kScRows + warp * 32 + lane] =
            (myid >= 0 && j < nq) ? rank_key(a.metric, ESZ == 4 ? acc[j] : ldexpf(acc[j], -a.xexp), nx2, inx) : -INFINITY;
        acc[j] = 0.f;
      }
      sid[b * kScRows + warp * 32 + lane] = myid;
      __syncthreads();
      if (warp < nq) {
        const float *keys = sc + (b * QG + warp) * kScRows;
        const int32_t *rid = sid + b * kScRows;
#pragma unroll 1
        for (int s = 0; s < kScRows / 32; ++s) {
          const float key = keys[s * 32 + lane];
          bool c = key > tau;
          uint32_t mask = __ballot_sync(0xffffffffu, c);
          if (mask) {
            if (cnt + 32 > KPE) {
              merge();
              c = key > tau;
              mask = __ballot_sync(0xffffffffu, c);
            }
            if (c) {
              const int pos = cnt + __popc(mask & lanemask_lt());
              L[KPE + pos] = key;
              I[KPE + pos] = rid[s * 32 + lane];
            }
            cnt += __popc(mask);
          }
        }
      }
    }
  }
  cp_async_wait<0>();

  if (warp < nq) {
    if (cnt > 0) merge();
    const int64_t o = ((int64_t)blockIdx.x * a.q + q0 + warp) * a.kprime;
    for (int r = lane; r < a.kprime; r += 32) {
      a.part_key[o + r] = L[r];
      a.part_id[o + r] = I[r];
    }
  }
}

template <int QG, int KPE, bool VEC4, int ESZ>
static cudaError_t launch_scan_t(const ScanArgs &a, int gy, cudaStream_t stream) {
  constexpr int KCE = kScKC * 4 / ESZ;
  const int dpad = (a.d + KCE - 1) / KCE * KCE;
  const size_t smem = scan_smem_bytes(QG, KPE, dpad);
  auto fn = scan_topk_kernel<QG, KPE, VEC4, ESZ>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_k(fn, dim3(a.P, gy), dim3(kScThreads), smem, stream, a);
}

template <int QG, int KPE>
static cudaError_t launch_scan_v(const ScanArgs &a, int gy, bool vec4, cudaStream_t s) {
  if (a.Xh) return launch_scan_t<QG, KPE, true, 2>(a, gy, s);   // (the shadow: d % 8 == 0, aligned)
  return vec4 ? launch_scan_t<QG, KPE, true, 4>(a, gy, s) : launch_scan_t<QG, KPE, false, 4>(a, gy, s);
}

template <int QG>
static cudaError_t launch_scan_k(const ScanArgs &a, int kpe, int gy, bool vec4, cudaStream_t s) {
  if (kpe <= 64) return launch_scan_v<QG, 64>(a, gy, vec4, s);
  if (kpe <= 128) return launch_scan_v<QG, 128>(a, gy, vec4, s);
  return launch_scan_v<QG, 256>(a, gy, vec4, s);
}

static constexpr size_t kSmemLimit = 227 * 1024;

// Pick the query group size: the smallest of {1,2,4,8} covering q (8 for q > 8),
// shrunk until the shared-memory plan fits.
int scan_query_group(int64_t q, int d, int kpe) {
  const int dpad = (d + 2 * kScKC - 1) / (2 * kScKC) * (2 * kScKC);   // (the 16-bit variant's padding)
  int qg = q <= 1 ? 1 : q <= 2 ? 2 : q <= 4 ? 4 : 8;
  const int kp = kpe <= 64 ? 64 : kpe <= 128 ? 128 : 256;
  while (qg > 1 && scan_smem_bytes(qg, kp, dpad) > kSmemLimit) qg >>= 1;
  if (scan_smem_bytes(qg, kp, dpad) > kSmemLimit) return 0;
  return qg;
}

cudaError_t launch_scan(const ScanArgs &a, int qg, int kpe, cudaStream_t s, int *launches) {
  const bool vec4 = (a.d % 4 == 0) && ((uintptr_t)a.X % 16 == 0);
  // query groups on grid.y, at most 65535 per launch (larger batches: several launches)
  const int64_t groups = (a.q + qg - 1) / qg;
  for (int64_t g0 = 0; g0 < groups; g0 += 65535) {
    ScanArgs b = a;
    b.q_base = g0 * qg;
    const int gy = (int)std::min<int64_t>(65535, groups - g0);
    if (launches) *launches += 1;
    cudaError_t e;
    switch (qg) {
      case 1: e = launch_scan_k<1>(b, kpe, gy, vec4, s); break;
      case 2: e = launch_scan_k<2>(b, kpe, gy, vec4, s); break;
      case 4: e = launch_scan_k<4>(b, kpe, gy, vec4, s); break;
      default: e = launch_scan_k<8>(b, kpe, gy, vec4, s); break;
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace vrs
