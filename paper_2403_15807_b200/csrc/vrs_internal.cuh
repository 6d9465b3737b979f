// vrs_internal.cuh -- device-side building blocks shared by the libvrs kernels.
// Product code only: nothing here is shared with oracle/ (DESIGN.md "Boundary").
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "vrs.h"

#include <stdlib.h>

#include <mutex>
#include <utility>

namespace vrs {

constexpr int kSmCountB200 = 148;

// ---- programmatic dependent launch ---------------------------------------------
// Every libvrs kernel is launched with programmatic stream serialization: it may
// be scheduled while its stream predecessor drains, runs its prologue (barrier
// init, TMEM allocation, tensor-map prefetch) and calls pdl_wait() -- which
// returns once every predecessor grid has completed and its writes are visible
// -- before it touches global memory.  pdl_trigger() lets the successor launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args &&...args) {
  static const bool pdl = getenv("VRS_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// launch_k with a thread-block cluster of `cluster_x` CTAs along x (1: none)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                    int cluster_x, Args &&...args) {
  if (cluster_x <= 1) return launch_k(kern, grid, block, smem, s, std::forward<Args>(args)...);
  static const bool pdl = getenv("VRS_NO_PDL") == nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cluster_x;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---- debug timeline (compile-time only: -DVRS_TC_TIMING; tools/tc_timeline.py) --
// Per translation unit: globaltimer stamps [region][cta][8] -- slot 0 kernel entry,
// 1 after griddepcontrol.wait, 5 thread 0 leaving the kernel (the tensor-core
// kernels add 2-4 and the SM id / tile count in 6 / 7).  Product builds compile
// every TL_* to nothing.
#ifdef VRS_TC_TIMING
static __device__ unsigned long long g_tl[8][4096][8];
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TL_STAMP(region, slot) \
  ((blockIdx.x < 4096 && threadIdx.x == 0) ? (void)(g_tl[(region)][blockIdx.x][(slot)] = tl_now()) : (void)0)
#define TL_STAMP_ANY(region, slot) \
  (blockIdx.x < 4096 ? (void)(g_tl[(region)][blockIdx.x][(slot)] = tl_now()) : (void)0)
struct TlEnd {
  int r;
  __device__ ~TlEnd() { TL_STAMP(r, 5); }
};
#define TL_SCOPE(region) TL_STAMP(region, 0); TlEnd tl_end_{region}
#define TL_WAITED(region) TL_STAMP(region, 1)
static inline int tl_read(unsigned long long *host) {
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  void *d = nullptr;
  if (cudaGetSymbolAddress(&d, g_tl) != cudaSuccess) return -1;
  if (cudaMemcpy(host, d, sizeof(g_tl), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return cudaMemset(d, 0, sizeof(g_tl)) == cudaSuccess ? 0 : -1;
}
#else
#define TL_STAMP(region, slot) ((void)0)
#define TL_STAMP_ANY(region, slot) ((void)0)
#define TL_SCOPE(region) ((void)0)
#define TL_WAITED(region) ((void)0)
#endif

// ---- host-side one-time setup ---------------------------------------------------
// Function attributes and pool tuning are set lazily on first use, possibly from
// several host threads at once: serialised here.
inline std::mutex &setup_mutex() {
  static std::mutex m;
  return m;
}
// Raise a kernel's dynamic shared-memory limit to >= bytes (done: the limit this
// call site already set; idempotent, thread-safe).
template <typename Kern>
inline cudaError_t ensure_smem_attr(Kern kern, size_t bytes, size_t &done) {
  if (bytes <= 32 * 1024) return cudaSuccess;   // (static shared memory adds to the 48 KB default limit)
  std::lock_guard<std::mutex> g(setup_mutex());
  if (bytes <= done) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done = bytes;
  return e;
}

// One clause of theta_R in device form: the [lo, hi] interval clamped to the
// column type's range (empty => the whole predicate selects nothing).
struct ClauseDev {
  const void *col;
  int32_t type;  // VRS_ATTR_I32 / VRS_ATTR_U8
  int32_t lo;
  int32_t hi;
};

struct PredDev {
  int32_t n;      // number of clauses (0 => all rows)
  int32_t empty;  // some clause is empty after clamping => no row qualifies
  ClauseDev c[VRS_MAX_CLAUSES];
};

// theta_R for one row (reading R4): AND of closed intervals.
__device__ __forceinline__ bool eval_pred(const PredDev &p, int64_t row) {
  if (p.empty) return false;
  bool ok = true;
#pragma unroll 1
  for (int c = 0; c < p.n; ++c) {
    int32_t v = (p.c[c].type == VRS_ATTR_I32) ? __ldg(static_cast<const int32_t *>(p.c[c].col) + row)
                                              : (int32_t)__ldg(static_cast<const uint8_t *>(p.c[c].col) + row);
    ok = ok && (p.c[c].lo <= v) && (v <= p.c[c].hi);
  }
  return ok;
}

// float -> uint32 whose unsigned order equals the float order (-inf < ... < +inf).
__device__ __forceinline__ uint32_t ordered_u32(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Warp-aggregated histogram increment for radix selection: the lanes holding
// the same bin add once (keys in one radix pass share their leading bits, so
// plain shared atomics would serialise on one or two bins).  All 32 lanes of
// the warp must call it; bin >= 256 means "no value".
__device__ __forceinline__ void hist_add_warp(uint32_t *hist, uint32_t bin) {
  const uint32_t peers = __match_any_sync(0xffffffffu, bin);
  if (bin < 256u && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- cp.async (LDGSTS) helpers -------------------------------------------------
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem, bool valid) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  int n = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// How many of the tensor-core pass's P row splits carry work: the row space
// (gathered selection or all rows) is decided on the device from the selection
// count, and each used split spans >= 4 row tiles.  The probe / main kernels,
// the threshold and the finalize kernels all derive it the same way, so the
// latter two skip the lists of unused splits.  bn == 0: all P splits.
struct SplitInfo {
  const int32_t *ids;      // compacted selection (nullptr: no predicate)
  const int64_t *count;
  int32_t allow_gather;
  int32_t P;
  int64_t n_rows;
  int64_t xsel_cap;
  int32_t bn;              // rows per tile
  int32_t min_span;        // >= this many row tiles per used split ...
  int32_t min_p;           // ... unless fewer than min_p splits would leave SMs idle (>= 1 tile each)
};
__device__ __forceinline__ bool gather_mode(const int32_t *ids, int allow, int64_t n_sel, int64_t cap) {
  return ids != nullptr && allow != 0 && n_sel <= cap;
}
// Gathered rows fetched by id (cp.async) rather than through the X_sel copy (vrs_api row_plan's
// rule, applied on the device to N_sel): selections of >= cp_min bytes, or of >= cp_min_rows
// rows -- enough row tiles that the per-SM fetch spreads over every SM.  Every kernel that
// takes the decision (the gather copy, select_finish, the tensor-core pass) calls this.
__host__ __device__ __forceinline__ bool cp_fetch(int64_t n_sel, int64_t row_bytes, int64_t cp_min_bytes,
                                                  int64_t cp_min_rows) {
  return n_sel * row_bytes >= cp_min_bytes || n_sel >= cp_min_rows;
}
// The one rule (probe / main kernels, threshold, finalize): >= min_span row tiles
// per split, but at least min_p splits (about one CTA per SM over the query
// tiles) while every split keeps >= 1 tile, and never more than P.
__host__ __device__ __forceinline__ int64_t used_splits(int64_t row_tiles, int64_t P, int64_t min_span, int64_t min_p) {
  int64_t p = row_tiles / min_span;
  if (p < min_p) p = min_p < row_tiles ? min_p : row_tiles;
  if (p > P) p = P;
  return p > 1 ? p : 1;
}
// The refine pass (qcount set on the device) folds its P x qtiles CTAs onto the
// `tiles` query tiles its compacted queries fill: F row-split groups per tile (P F
// splits), group f's lists stored at rows f Qa + j of the level-0 lists ([2P][q]),
// F Qa <= q.  The refine's main pass and its finalize both map through this.
struct RefineFold {
  int32_t tiles;   // active query tiles, ceil(qcount / 128) (>= 1)
  int32_t F;       // split groups per tile
  int64_t Qa;      // tiles * 128: list-row stride between groups
};
__host__ __device__ __forceinline__ RefineFold refine_fold(int64_t qcount, int64_t qtiles, int64_t q) {
  RefineFold r;
  r.tiles = (int32_t)(qcount > 0 ? (qcount + 127) / 128 : 1);
  r.Qa = (int64_t)r.tiles * 128;
  int64_t F = qtiles / r.tiles;
  if (F > q / r.Qa) F = q / r.Qa;
  r.F = (int32_t)(F > 1 ? F : 1);
  return r;
}
__device__ __forceinline__ int64_t splits_used(const SplitInfo &si) {
  if (si.bn == 0) return si.P;
  const int64_t n_sel = si.ids ? *si.count : si.n_rows;
  const int64_t n_space = gather_mode(si.ids, si.allow_gather, n_sel, si.xsel_cap) ? n_sel : si.n_rows;
  return used_splits((n_space + si.bn - 1) / si.bn, si.P, si.min_span, si.min_p);
}

// Ranking key used by the selection passes, larger = better for every metric
// (DESIGN.md "Selection key"):  L2: 2<q,x> - |x|^2  (= |q|^2 - L2, same order),
// IP: <q,x>,  COS: <q,x>/|x|  (1/|q| > 0 does not change the order).
__device__ __forceinline__ float rank_key(int metric, float dot, float nx2, float inv_nx) {
  if (metric == VRS_L2) return fmaf(2.0f, dot, -nx2);
  if (metric == VRS_IP) return dot;
  return dot * inv_nx;
}

// ---- selection-key error bound ("Certified exactness") -------
// The selection passes rank rows by a computed key (rank_key units, "natural"
// units below: L2 2<q,x> - |x|^2, IP <q,x>, COS <q,x>/|x|).  For one query q
// and ANY row x, |computed key - exact key| <= E(q) with E from:
//   operands   x~ = x + eps_x, q~ = q + eta (the 16-bit shadow / query, natural
//              units):  |<q~,x~> - <q,x>| <= |q| |eps_x| + |eta| |x| + |eta| |eps_x|
//              (Cauchy-Schwarz), with |eps_x| <= rmax and |eps_x| / |x| <= rho
//              MEASURED at load (fp64, exact) and |eta| = rq measured per query;
//              TF32 (hardware rounding of the fp32 operands, truncation or RN):
//              |eps| <= 2^-10 |x| per element, likewise for q;
//   accumulation  fp32 sums of exact products (16-bit x 16-bit fits fp32's 24-bit
//              significand; TF32 11 x 11 bits too): <= c (|q~| |x~|) with
//              c = (#MMA instructions along K + K per instruction) 2^-22 -- every
//              accumulate and every in-instruction add within 2 ulp of the largest
//              partial magnitude; fp32 FFMA scan: c = (d + 4) 2^-24;
//   key arithmetic  |x|^2 and 1/|x| are fp32 roundings of fp64 values (2^-24
//              relative), the key's own fma / product rounding (2^-24 relative);
// each term rounded up generously (x2 on the fp32 rounding terms), then
// x (1 + 2^-6) and an absolute 2^-40 slack for the fp64 arithmetic of the caller.
enum KeyKind : int32_t { KEY_H16 = 0, KEY_TF32 = 1, KEY_FP32 = 2, KEY_H16_FFMA = 3, KEY_H16X3 = 4 };
struct KeyBound {
  int32_t kind;   // KeyKind
  int32_t d;
  double rmax;    // KEY_H16: max over rows of |x~ - x| (natural units, rounded up)
  double rho;     // KEY_H16: max over rows of |x~ - x| / |x|
  double xmax;    // max row norm (rounded up)
  double rmax2 = 0, rho2 = 0;   // KEY_H16X3: the same after x~ + x_lo
};
// The refine pass (KEY_H16X3): keys from q_hi.x_hi + q_hi.x_lo + q_lo.x_hi with
// q = q_hi + q_lo + eta2, x = x_hi + x_lo + eps2 (natural units; |q_lo| <= rqa, |eta2| = rq2,
// |x_lo| <= R + R2, |eps2| <= R2): the exact dot differs from the computed three products by
// q_lo.x_lo + (q_hi + q_lo).eps2 + eta2.(x_hi + x_lo) + eta2.eps2, and the fp32 accumulation
// of 3 x ceil(d/16) MMA instructions over partial magnitudes <= (|q| + 2 rqa + rq2)(N + 2R + R2).
__host__ __device__ inline double key_error_bound_x3(const KeyBound &b, int metric, double qn, double rqa, double rq2) {
  const double R = b.rmax, R2 = b.rmax2, rho = b.rho, rho2 = b.rho2, N = b.xmax;
  const double c = (double)(3 * ((b.d + 15) / 16) + 16) * 0x1p-22;
  double E;
  if (metric == VRS_COSINE) {   // divided by |x|: |x_lo| <= (rho + rho2)|x|, |eps2| <= rho2 |x|
    E = rqa * (rho + rho2) + (qn + rq2) * rho2 + rq2 * (1.0 + rho2) +
        c * (qn + 2.0 * rqa + rq2) * (1.0 + 2.0 * rho + rho2) + 0x1p-21 * qn;
  } else {
    const double ed = rqa * (R + R2) + (qn + rq2) * R2 + rq2 * (N + R2) + c * (qn + 2.0 * rqa + rq2) * (N + 2.0 * R + R2);
    E = metric == VRS_IP ? ed + 0x1p-23 * qn * N : 2.0 * ed + 0x1p-22 * N * N + 0x1p-22 * qn * N;
  }
  return E * (1.0 + 0x1p-6) + 0x1p-40 * (qn * N + N * N + qn * qn);
}
__host__ __device__ inline double key_error_bound(const KeyBound &b, int metric, double qn, double rq) {
  double R = b.rmax, rho = b.rho, N = b.xmax, c;
  if (b.kind == KEY_TF32) {
    rq = 0x1p-10 * qn;
    R = 0x1p-10 * N;
    rho = 0x1p-10;
    c = (double)((b.d + 7) / 8 + 8) * 0x1p-22;
  } else if (b.kind == KEY_FP32) {
    rq = 0.0;
    R = 0.0;
    rho = 0.0;
    c = (double)(b.d + 4) * 0x1p-24;
  } else if (b.kind == KEY_H16_FFMA) {   // 16-bit shadow rows, exact fp32 queries, FFMA (scan path)
    rq = 0.0;
    c = (double)(b.d + 4) * 0x1p-24;
  } else {
    c = (double)((b.d + 15) / 16 + 16) * 0x1p-22;
  }
  double E;
  if (metric == VRS_COSINE) {
    E = qn * rho + rq + rq * rho + c * (qn + rq) * (1.0 + rho) + 0x1p-21 * qn;
  } else {
    const double ed = qn * R + rq * N + rq * R + c * (qn + rq) * (N + R);
    E = metric == VRS_IP ? ed + 0x1p-23 * qn * N : 2.0 * ed + 0x1p-22 * N * N + 0x1p-22 * qn * N;
  }
  return E * (1.0 + 0x1p-6) + 0x1p-40 * (qn * N + N * N + qn * qn);
}

// Candidate (key, id) total order: key descending, then id ascending.
__device__ __forceinline__ bool cand_better(float ka, int32_t ia, float kb, int32_t ib) {
  return (ka > kb) || (ka == kb && ia < ib);
}

// Warp-cooperative bitonic sort, descending in (key, -id), of n = 2^p entries
// held in shared memory.  All 32 lanes must call it.
__device__ __forceinline__ void warp_bitonic_sort_desc(float *key, int32_t *id, int n) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncwarp();
      for (int t = lane; t < (n >> 1); t += 32) {
        int lo = 2 * t - (t & (stride - 1));
        int hi = lo + stride;
        bool desc = ((lo & size) == 0);  // direction of this bitonic half
        float ka = key[lo], kb = key[hi];
        int32_t ia = id[lo], ib = id[hi];
        bool swap = desc ? cand_better(kb, ib, ka, ia) : cand_better(ka, ia, kb, ib);
        if (swap) {
          key[lo] = kb; key[hi] = ka;
          id[lo] = ib;  id[hi] = ia;
        }
      }
    }
  }
  __syncwarp();
}

// Sums of U (4 or 8) per-lane values over the warp: on return every lane holds
// the total of value (lane >> (5 - log2 U)) & (U - 1).  Each step swaps half of
// the remaining values with the partner lane (xor 16, 8, ...), then a plain
// butterfly over the remaining lane bits.
template <int U>
constexpr int log2u() { return U == 8 ? 3 : (U == 4 ? 2 : (U == 2 ? 1 : 0)); }
template <int U>
__device__ __forceinline__ double warp_sum_transpose(const double (&v)[U]) {
  static_assert(U == 4 || U == 8, "U = 4 or 8");
  const int lane = threadIdx.x & 31;
  double w[U];
#pragma unroll
  for (int i = 0; i < U; ++i) w[i] = v[i];
#pragma unroll
  for (int h = U / 2, o = 16; h >= 1; h >>= 1, o >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int i = 0; i < h; ++i) w[i] = (up ? w[i + h] : w[i]) + __shfl_xor_sync(0xffffffffu, up ? w[i] : w[i + h], o);
  }
  double y = w[0];
#pragma unroll
  for (int o = 16 / U; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
  return y;
}

}  // namespace vrs
