// gemm_tc.cu -- K3': the batched tensor formulation on 5th-generation tensor cores.
//
// PAPER.md L302-L304 (Sec. 3.1): batch the query vectors AND the data vectors
// and compute their similarity as one matrix product ("Tensor formulation,
// based on BLAS"); L305 cosine as a dot product with normalised operands;
// L319 late materialization (filter first, then batch).  Here the product
// S = Q . X_sel^T is never materialised: it lives in TMEM one 128 x 256 tile
// at a time and is consumed by a fused top-k epilogue.
//
// Per CTA: one work item = (query tile of 128, contiguous split of the row
// tiles).  Warp roles (384 threads, 1 CTA / SM):
//   warp 0    TMA producer: query block [128 x 32 fp32] (resident for d <= 128)
//             + row block [256 x 32] per stage, 128-byte swizzle, mbarrier ring
//   warp 1    TMEM allocator + tcgen05.mma issuer (kind::tf32, M=128, N=256,
//             K=8 per instruction), fp32 accumulators double-buffered in TMEM
//             (2 x 256 columns)
//   warp 2    per-row epilogue terms: ranking-key scale/bias of each of the 256
//             rows of a tile (norm terms, bitmap mask -> -inf) and row ids
//   warps 4-11 epilogue, 2 per TMEM lane quadrant (one query per lane, 128 of
//             the tile's 256 columns per warp): tcgen05.ld 32 columns at a time,
//             key = fma(dot, a, b), then
//     PROBE pass (every 16th row tile): per-lane running maxima of 32 disjoint
//             row slots -> [q][list][32]; branch-free.  threshold_kernel takes
//             the k'-th largest of a query's slot maxima: k' distinct rows reach
//             it, so it is a lower bound of the k'-th best key over all rows
//     MAIN pass: compare with the query's threshold (own list / shared bound
//             from the probe), rare append of (key, row) to a per-(list, query)
//             candidate buffer, warp-cooperative radix compaction on overflow.
// Precision: TF32 products, fp32 accumulation -> selection only; the k' = k+16
// best per query are re-scored exactly in finalize.cu.
//
// Roofline: tensor (2*q*N_rows*d TF32 flops) for large q, HBM (4*d bytes per
// row) for small q.
#include <cuda_fp16.h>
#include <string.h>

#include "tc_kernel.cuh"
#include "convert16.cuh"

namespace vrs {

// (gather_mode: gathered rows iff a selection exists and fits the materialisation
// buffer, whose capacity the host sized by the selectivity break-even, vrs_api.cu)

// Late materialization ("(re-)materialized into dense
// vectors"): X_sel[r] = X[ids[r]] (rows of row_bytes, a multiple of 16: the fp32
// corpus or its 16-bit shadow), one warp per row, 16-byte vector copies.
// HBM-bound: 2 * row_bytes per selected row.
__global__ void __launch_bounds__(256) gather_copy_kernel(const void *__restrict__ X, int32_t row_bytes,
                                                          const int32_t *__restrict__ ids,
                                                          const int64_t *__restrict__ count, int64_t n, int allow,
                                                          int64_t cap, void *__restrict__ xsel,
                                                          const float *__restrict__ norm_src,
                                                          float *__restrict__ norm_dst, int64_t cp_min_bytes,
                                                          int64_t cp_min_rows) {
  TL_SCOPE(4);
  pdl_wait();
  TL_WAITED(4);
  pdl_trigger();
  const int64_t n_sel = *count;
  if (!gather_mode(ids, allow, n_sel, cap)) return;
  if (cp_fetch(n_sel, row_bytes, cp_min_bytes, cp_min_rows)) return;   // the tensor-core pass fetches them by cp.async
  // a warp per row (4 rows in flight), lanes along the row's 16-byte vectors (coalesced);
  // the row id is one broadcast load (round 1 divided a 64-bit element index per vector:
  // C5 s = 10 %, 128 MB of 512-byte rows took 336 us)
  const int v16 = row_bytes >> 4;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const char *Xc = static_cast<const char *>(X);
  char *Yc = static_cast<char *>(xsel);
  for (int64_t r0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 4; r0 < n_sel; r0 += warps * 4) {
    int32_t id[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) id[u] = r0 + u < n_sel ? __ldg(ids + r0 + u) : -1;
    for (int v = lane; v < v16; v += 32) {
      int4 w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (id[u] >= 0) w[u] = __ldg(reinterpret_cast<const int4 *>(Xc + (int64_t)id[u] * row_bytes) + v);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (id[u] >= 0) reinterpret_cast<int4 *>(Yc + (r0 + u) * row_bytes)[v] = w[u];
    }
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (norm_dst)   // the rows' norm terms, contiguous, for the bias producer
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_sel; r += stride)
      norm_dst[r] = __ldg(norm_src + __ldg(ids + r));
}

// select_finish (after launch_select_local): every CTA turns the per-chunk counts
// into an exclusive prefix table in shared memory; CTA 0 writes the count; in
// gathered mode (decided here from the count, like gather_copy_kernel) each warp
// takes 32 consecutive dense positions, each lane resolves its position's chunk
// by binary search and writes the dense id (and the norm term), then the warp
// copies the 32 rows with 16-byte vectors.  One launch replaces select_scatter +
// gather_copy.
__global__ void __launch_bounds__(256) select_finish_kernel(const uint32_t *__restrict__ chunk_count, int nchunks,
                                                            const int32_t *__restrict__ ids_local,
                                                            int64_t *__restrict__ count, int32_t *__restrict__ ids,
                                                            int allow, int64_t cap, const void *__restrict__ X,
                                                            int32_t row_bytes, void *__restrict__ xsel,
                                                            const float *__restrict__ norm_src,
                                                            float *__restrict__ norm_dst, int64_t cp_min_bytes,
                                                            int64_t cp_min_rows) {
  TL_SCOPE(6);
  extern __shared__ uint32_t s_pre[];   // [nchunks + 1]
  __shared__ uint32_t s_wsum[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  pdl_wait();
  TL_WAITED(6);
  pdl_trigger();
  // exclusive prefix of the chunk counts: thread t sums a contiguous segment
  const int seg = (nchunks + 255) / 256;
  const int c0 = min(nchunks, tid * seg), c1 = min(nchunks, c0 + seg);
  uint32_t sum = 0;
  for (int c = c0; c < c1; ++c) sum += __ldg(chunk_count + c);
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  uint32_t run = incl - sum;
  for (int i = 0; i < warp; ++i) run += s_wsum[i];
  for (int c = c0; c < c1; ++c) {
    s_pre[c] = run;
    run += __ldg(chunk_count + c);
  }
  if (tid == 255) s_pre[nchunks] = run;
  __syncthreads();
  const int64_t total = s_pre[nchunks];
  if (blockIdx.x == 0 && tid == 0) *count = total;
  if (!gather_mode(ids, allow, total, cap)) return;
  if (cp_fetch(total, row_bytes, cp_min_bytes, cp_min_rows)) {   // rows by id in the pass: ids only
    xsel = nullptr;
    norm_dst = nullptr;
  }
  const int v16 = row_bytes >> 4;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t base = ((int64_t)blockIdx.x * 8 + warp) * 32; base < total; base += nwarps * 32) {
    const int64_t r = base + lane;
    int32_t src = 0;
    if (r < total) {
      int lo = 0, hi = nchunks;   // s_pre[lo] <= r < s_pre[hi]: lo = the last chunk starting at or before r
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if ((int64_t)s_pre[mid] <= r) lo = mid; else hi = mid;
      }
      src = __ldg(ids_local + (int64_t)lo * kSelChunkRows + (r - s_pre[lo]));
      ids[r] = src;
      if (norm_dst) norm_dst[r] = __ldg(norm_src + src);
    }
    if (xsel) {
      const int nr = (int)min((int64_t)32, total - base);
      // the warp's 32 rows, 32 x v16 vectors, 8 loads in flight per lane
      for (int it0 = 0; it0 < v16; it0 += 8) {
        int4 v[8];
        int64_t dst[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = (it0 + u) * 32 + lane;
          const int rr = i / v16, vv = i - rr * v16;
          const int32_t sr = __shfl_sync(0xffffffffu, src, rr & 31);
          dst[u] = -1;
          if (it0 + u < v16 && rr < nr) {
            v[u] = __ldg(reinterpret_cast<const int4 *>(static_cast<const char *>(X) + (int64_t)sr * row_bytes) + vv);
            dst[u] = (base + rr) * (int64_t)v16 + vv;
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (dst[u] >= 0) reinterpret_cast<int4 *>(xsel)[dst[u]] = v[u];
      }
    }
  }
}

cudaError_t launch_select_finish(const GemmArgs &a, int64_t xcap, int allow, const void *xsrc, int32_t row_bytes,
                                 bool copy, cudaStream_t s) {
  const int nchunks = (int)select_chunks(a.n);
  const size_t smem = (size_t)(nchunks + 1) * 4;
  static size_t attr = 0;
  const cudaError_t e = ensure_smem_attr(select_finish_kernel, smem, attr);
  if (e != cudaSuccess) return e;
  static const int blocks = getenv("VRS_FINISH_BLOCKS") ? atoi(getenv("VRS_FINISH_BLOCKS")) : 2 * 148;
  return launch_k(select_finish_kernel, dim3(blocks), dim3(256), smem, s, a.chunk_count, nchunks, a.ids_local,
                  const_cast<int64_t *>(a.count), const_cast<int32_t *>(a.ids), allow, xcap, xsrc, row_bytes,
                  copy ? a.xsel : (void *)nullptr, a.metric == VRS_L2 ? a.nx2 : a.inv_nx,
                  copy && a.metric != VRS_IP ? a.xsel_norm : (float *)nullptr, copy ? a.cp_min_bytes : INT64_MAX,
                  copy ? a.cp_min_rows : INT64_MAX);
}

// ---------------------------------------------------------------- 16-bit operands
// The tensor-core selection runs kind::f16 on 16-bit copies of the corpus (the
// shadow, built at load) and of the queries (per search).  fp16 (default): every
// value is scaled by a power of two before rounding -- the corpus by one 2^e_x
// for the whole index, each query row by its own 2^e_q -- so the largest |value|
// lands in [2^14, 2^15): the 11-bit significand is used in full and nothing
// overflows.  bf16: e = 0.  Powers of two are exact, so the MMA's dot product is
// 2^(e_q + e_x) <q~, x~> (the key domain).  Each row's rounding
// residual |x~ 2^-e - x| is measured exactly (fp64) -- the certificate's bound.
// The shadow (load): warp per row.  res[0] = max |x~ - x|, res[1] = max |x~ - x| / |x|;
// with out_lo (fp16): the refine pass's second half x_lo = fp16(x 2^e - x~), and
// res[2] / res[3] the same maxima for |(x~ + x_lo) 2^-e - x| (rounded up; u64 bits of
// non-negative doubles order as integers).
__global__ void __launch_bounds__(256) shadow_kernel(const float *__restrict__ X, int64_t n, int32_t d, int32_t e,
                                                     int32_t fmt, uint16_t *__restrict__ out,
                                                     uint16_t *__restrict__ out_lo, const float *__restrict__ nx2,
                                                     unsigned long long *res) {
  const int lane = threadIdx.x & 31;
  double rmax = 0.0, rho = 0.0, rmax2 = 0.0, rho2 = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); row < n; row += (int64_t)gridDim.x * 8) {
    double r, r2 = 0.0;
    if (out_lo) {
      const double2 rr = row_to16x2(X + row * d, out + row * d, out_lo + row * d, d, e);
      r = sqrt(rr.x) * (1.0 + 0x1p-50);
      r2 = sqrt(rr.y) * (1.0 + 0x1p-50);
    } else {
      r = sqrt(row_to16(X + row * d, out + row * d, d, e, fmt)) * (1.0 + 0x1p-50);
    }
    rmax = fmax(rmax, r);
    rmax2 = fmax(rmax2, r2);
    const double xn = sqrt((double)__ldg(nx2 + row));
    if (xn > 0.0) {   // (|x| from the fp32 |x|^2: 2^-24 relative)
      rho = fmax(rho, r / xn * (1.0 + 0x1p-20));
      rho2 = fmax(rho2, r2 / xn * (1.0 + 0x1p-20));
    }
  }
  if (lane == 0) {
    atomicMax(res, (unsigned long long)__double_as_longlong(rmax));
    atomicMax(res + 1, (unsigned long long)__double_as_longlong(rho));
    atomicMax(res + 2, (unsigned long long)__double_as_longlong(rmax2));
    atomicMax(res + 3, (unsigned long long)__double_as_longlong(rho2));
  }
}

cudaError_t launch_shadow(const float *X, int64_t n, int32_t d, int32_t e, int32_t fmt, void *out, void *out_lo,
                          const float *nx2, unsigned long long *res, cudaStream_t s) {
  const int64_t blocks = std::min<int64_t>((n + 7) / 8, 148 * 16);
  shadow_kernel<<<(unsigned)blocks, 256, 0, s>>>(X, n, d, e, fmt, static_cast<uint16_t *>(out),
                                                 static_cast<uint16_t *>(out_lo), nx2, res);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) query16_kernel(QueryFuse f) {
  TL_SCOPE(5);
  pdl_wait();
  TL_WAITED(5);
  pdl_trigger();
  for (int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); row < f.rows; row += (int64_t)gridDim.x * 8)
    query_row_to16(f, row);
}

cudaError_t launch_query16(const QueryFuse &f, cudaStream_t s) {
  if (f.rows <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((f.rows + 7) / 8, 148 * 8);
  return launch_k(query16_kernel, dim3((unsigned)blocks), dim3(256), 0, s, f);
}


// ---------------------------------------------------------------- host side
static int kp_of(int32_t kprime) {
  int kp = 32;
  while (kp < kprime) kp <<= 1;
  return kp;
}

// Splits that keep the SMs busy on small row spaces (VRS_NO_MIN_P=1: off, for A/B).
static int32_t tc_min_p(const GemmPlan &plan) {
  static const bool off = getenv("VRS_NO_MIN_P") != nullptr;
  return off ? 1 : plan.min_p;
}

// The main pass runs as CTA pairs (tc_kernel.cuh PAIR) for an even number of query tiles
// on 16-bit operands with a streamed query tile (d > 256: nk > 4).  VRS_PAIR=0 disables.
// (C4 bench 285.8 -> 297.8 k q/s: s = 50 %, Q = 256 3.24 -> 2.71 ms, Q = 8192 70.1 -> 68.1 ms;
// r02_pair_ab.txt)
bool pair_main(int64_t qtiles, int32_t d, bool h16) {
  static const bool on = !getenv("VRS_PAIR") || atoi(getenv("VRS_PAIR")) > 0;
  return on && h16 && qtiles % 2 == 0 && (d + 2 * tc::BK - 1) / (2 * tc::BK) > 4;
}

GemmPlan gemm_plan(int64_t q, int32_t d, int64_t n_upper, int32_t kprime, int num_sms, bool h16) {
  GemmPlan g{0, 0, 0, 1};
  if (d % 4 != 0 || d < 4 || q < 1 || n_upper < 1 || kprime > 256) return g;
  if (!encode_fn()) return g;
  const int64_t qtiles = (q + tc::BM - 1) / tc::BM;
  const int64_t row_tiles = (n_upper + tc::BN - 1) / tc::BN;
  // one CTA per SM; aim for up to 4 waves of (query tile, row split) items while keeping
  // items >= ~128 row tiles
  int64_t waves = std::max<int64_t>(1, std::min<int64_t>(4, row_tiles * qtiles / ((int64_t)num_sms * 128)));
  // (two query tiles as one CTA pair per split: one wave -- C4 s = 5 %, Q = 256 0.433 -> 0.411 ms)
  if (qtiles == 2 && pair_main(qtiles, d, h16)) waves = 1;
  int64_t P = std::max<int64_t>(1, (int64_t)num_sms * waves / qtiles);
  static const int p_env = getenv("VRS_P") ? atoi(getenv("VRS_P")) : 0;   // (experiments)
  if (p_env > 0) P = p_env;
  P = std::min<int64_t>(std::min<int64_t>(P, row_tiles), 2 * num_sms);
  g.P = (int32_t)P;
  g.qtiles = (int32_t)qtiles;
  g.ok = 1;
  // (small row spaces: splits of a single tile rather than idle SMs -- C2 Q = 4096, s = 0.1 %:
  // 975 rows = 4 tiles would otherwise run on 32 CTAs)
  g.min_p = (int32_t)std::max<int64_t>(1, ((int64_t)num_sms + qtiles - 1) / qtiles);
  return g;
}

// scratch: cand_key, cand_id [2P][q][cap] | cand_cnt [2P][q] | gtau [q] | probe_max [q][2P][32]
namespace {
struct GemmScratch {
  float *cand_key;
  int32_t *cand_id;
  int32_t *cand_cnt;
  uint32_t *gtau;
  float *probe_max;
  size_t bytes;
};
GemmScratch carve_gemm(void *base, const GemmPlan &plan, int64_t q, int32_t kprime) {
  const size_t lists = (size_t)plan.P * kListsPerSplit;
  const size_t cap = (size_t)kp_of(kprime) * tc::CAP_FACTOR;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  char *p = static_cast<char *>(base);
  GemmScratch s;
  size_t off = 0;
  s.cand_key = reinterpret_cast<float *>(p + off); off += al(lists * q * cap * 4);
  s.cand_id = reinterpret_cast<int32_t *>(p + off); off += al(lists * q * cap * 4);
  s.cand_cnt = reinterpret_cast<int32_t *>(p + off); off += al(lists * q * 4);
  s.gtau = reinterpret_cast<uint32_t *>(p + off); off += al((size_t)q * 4);
  s.probe_max = reinterpret_cast<float *>(p + off); off += al(lists * q * tc::SLOTS * 4);
  s.bytes = off;
  return s;
}
}  // namespace

size_t gemm_scratch_bytes(const GemmPlan &plan, int64_t q, int32_t kprime) {
  return carve_gemm(nullptr, plan, q, kprime).bytes;
}

cudaError_t tc_prepare(const GemmArgs &a, const GemmPlan &plan, cudaStream_t s, int *launches, TcLaunch *L) {
  const int64_t xcap = a.ids ? a.xsel_cap : 0;
  // gathered rows without a buffer: fetched from X by id (cp.async, or TMA gather4)
  const bool g4 = xcap > 0 && a.xsel == nullptr;
  const bool bf = a.bf16 != 0;
  cudaError_t e = cudaSuccess;
  if (bf && !a.prepped) {   // queries -> 16-bit (the corpus shadow was converted at load)
    const QueryFuse f{a.Q, a.Qb, a.q, (int64_t)plan.qtiles * tc::BM, a.d, a.fmt16, a.qexp, a.rq};
    e = launch_query16(f, s);
    if (e != cudaSuccess) return e;
    if (launches) *launches += 1;
  }
  const void *qsrc = bf ? a.Qb : (const void *)a.Q;
  const void *xsrc = bf ? a.Xb : (const void *)a.X;
  if (!make_map(&L->mq, qsrc, bf ? (int64_t)plan.qtiles * tc::BM : a.q, a.d, tc::BM, bf, a.fmt16) ||
      !make_map(&L->mx, xsrc, a.n, a.d, tc::BN, bf, a.fmt16) ||
      !(g4 ? make_map(&L->mg, xsrc, a.n, a.d, 1, bf, a.fmt16)
           : make_map(&L->mg, xcap > 0 ? a.xsel : xsrc, xcap > 0 ? xcap : a.n, a.d, tc::BN, bf, a.fmt16)))
    return cudaErrorInvalidValue;
  L->ml = L->mx;   // (the refine pass's x_lo maps; launch_refine sets them)
  L->mlg = L->mx;
  TcParams &p = L->p;
  memset(&p, 0, sizeof p);
  p.nseg = 1;   // (one K segment; the refine pass sets 3)
  p.n_rows = a.n;
  p.d = a.d;
  p.nk = (a.d + (bf ? 2 * tc::BK : tc::BK) - 1) / (bf ? 2 * tc::BK : tc::BK);
  p.q = a.q;
  p.qtiles = plan.qtiles;
  p.P = plan.P;
  p.ids = a.ids;
  p.count = a.count;
  p.allow_gather = a.masked == 1 ? 0 : (a.masked == 2 ? 2 : 1);
  p.xsel_cap = xcap;
  p.xsel_norm = a.xsel_norm;
  // Gathered row delivery (decided per launch on the device from the selection size):
  //  * no X_sel buffer (VRS_GATHER4 / VRS_CPGATHER): rows by id from X -- TMA gather4 or cp.async;
  //  * <= 2 query tiles: cp.async when the selection holds >= 64 MB or >= 2 x 148 row tiles
  //    (cp_fetch), else the X_sel
  //    copy (r01_s3_cp_gather_ab.txt: C3 s = 10 % Q = 1 0.95 -> 0.74 ms, small selections
  //    are faster copied);  * several query tiles: the copy (rows are re-read per tile).
  static const bool tma_gather4 = getenv("VRS_GATHER4") != nullptr;
  if (g4) {
    p.g4 = tma_gather4 ? 1 : 2;
    p.cp_min_bytes = 0;
    p.cp_min_rows = 0;
  } else {
    p.g4 = a.cp_min_bytes < INT64_MAX ? 2 : 0;
    p.cp_min_bytes = a.cp_min_bytes;
    p.cp_min_rows = a.cp_min_rows;
  }
  p.xrows = xsrc;
  p.row_bytes = a.d * (bf ? 2 : 4);
  p.bitmap = a.bitmap;
  p.nx2 = a.nx2;
  p.inv_nx = a.inv_nx;
  p.metric = a.metric;
  p.kp = kp_of(a.kprime);
  p.cap = p.kp * tc::CAP_FACTOR;
  p.idesc = mma_idesc(tc::BM, tc::BN, bf ? (uint32_t)a.fmt16 : 2u);
  p.qexp = bf ? a.qexp : nullptr;
  p.xexp = bf ? a.xexp : 0;
  p.tile_step = 1;
  p.probe_div = 0;
  p.probe_rows = 0;
  static const bool no_helpers = getenv("VRS_NO_HELPERS") != nullptr;   // (A/B only)
  p.no_helpers = no_helpers ? 1 : 0;
  p.min_span = tc_min_span();
  p.min_p = tc_min_p(plan);
  static const bool no_ar = getenv("VRS_NO_AR") != nullptr;
  L->bf = bf;
  L->ar = p.nk <= 4 && !no_ar;
  L->rowscale = a.metric == VRS_COSINE;
  if (a.ids_local) {   // count + dense ids (+ gathered rows) from launch_select_local's output
    ProfScope ps("gemm.gather", s);
    e = launch_select_finish(a, xcap, xcap > 0 ? (int)p.allow_gather : 0, xsrc, a.d * (bf ? 2 : 4), !g4, s);
    if (e != cudaSuccess) return e;
    if (launches) *launches += 1;
  } else if (xcap > 0 && p.allow_gather && !g4 && !a.xsel_ready) {
    ProfScope ps("gemm.gather", s);
    e = launch_k(gather_copy_kernel, dim3(8 * 148), dim3(256), 0, s, xsrc, a.d * (bf ? 2 : 4), a.ids, a.count, a.n,
                 (int)p.allow_gather, xcap, a.xsel, a.metric == VRS_L2 ? a.nx2 : a.inv_nx,
                 a.metric == VRS_IP ? (float *)nullptr : a.xsel_norm, p.cp_min_bytes, p.cp_min_rows);
    if (e != cudaSuccess) return e;
    if (launches) *launches += 1;
  }
  return cudaSuccess;
}

cudaError_t launch_gemm(const GemmArgs &a, const GemmPlan &plan, void *scratch, cudaStream_t s, int *launches) {
  TcLaunch L;
  cudaError_t e = tc_prepare(a, plan, s, launches, &L);
  if (e != cudaSuccess) return e;
  const GemmScratch gs = carve_gemm(scratch, plan, a.q, a.kprime);
  TcParams &p = L.p;
  p.cand_key = gs.cand_key;
  p.cand_id = gs.cand_id;
  p.cand_cnt = gs.cand_cnt;
  p.gtau = gs.gtau;
  p.probe_max = gs.probe_max;
  // AR8 (tc_kernel.cuh): <= 8 queries held resident as 8 rows per K block -- the stages carry
  // rows only (5 in flight instead of 4 stages of rows + query tile); probe and main pass
  static const bool ar8_on = !getenv("VRS_AR8") || atoi(getenv("VRS_AR8")) > 0;
  if (ar8_on && L.bf && !L.ar && plan.qtiles == 1 && a.q <= 8 && p.nk <= 32 && p.nseg == 1) {
    if (!make_map(&L.mq, a.Qb, (int64_t)plan.qtiles * tc::BM, a.d, 8, true, a.fmt16)) return cudaErrorInvalidValue;
    L.ar8 = true;
  }
  static const bool no_probe = getenv("VRS_NO_PROBE") != nullptr;
  if (no_probe) {   // (otherwise threshold_kernel writes every query's gtau)
    e = cudaMemsetAsync(p.gtau, 0, (size_t)a.q * 4, s);
    if (e != cudaSuccess) return e;
  }
  // Threshold before the main pass: probe pass over every PROBE_STEP-th row tile
  // (slot maxima) -> per query the k'-th largest slot maximum -> gtau.
  if (!no_probe) {
    ProfScope pf("gemm.probe", s);
    TcParams pp = p;
    // probe density: a denser probe gives a tighter threshold (fewer slow-path
    // chunks in the main pass, which matters once the main pass is TMEM / MMA
    // bound); small batches are HBM-bound and want the cheapest probe
    // (C2 measurements: 1/8 best at Q = 4096, 1/16 at Q = 256, 1/32 at Q = 16)
    static const int probe_env = getenv("VRS_PROBE_STEP") ? atoi(getenv("VRS_PROBE_STEP")) : 0;
    // (large d: the main pass is MMA-bound and its epilogue has slack, so a sparser probe
    // costs the main pass nothing -- C3 Q = 1024: 13.4 -> 12.5 ms, C4 Q = 8192 s = 50 %:
    // 72 -> 68 ms at step 16; step 32 overflows C4's lists, r01_s3_probe_step_large_d.txt)
    // (d >= 512 below 1024 queries: the main pass is HBM-bound, its epilogue has slack -- the
    // sparsest probe; C3 s = 10 %, Q = 64: the dense probe took 193 us of a 608 us search)
    const bool hbm_bound = a.d >= 512 && a.q < 1024;
    // (d >= 1024, q >= 1024: every 32nd tile -- C4: probe 5.6 -> 3.2 ms per step, main pass and
    // finalize within noise, +1 % overall, r02_probe_step_c4_ab.txt)
    pp.tile_step = probe_env > 0 ? probe_env
                                 : (a.q >= 1024 ? (a.d >= 1024 ? 32 : (a.d >= 512 ? 16 : 8))
                                                : (a.q >= 64 && !hbm_bound ? tc::PROBE_STEP : 32));
    // (C2 sweep, r01_cells_probe_step.txt: Q = 4096, s = 10 %: step 2 beats 8 by 18 %; Q = 256, s = 100 %: 4 beats 16)
    static const int div_env = getenv("VRS_PROBE_DIV") ? atoi(getenv("VRS_PROBE_DIV")) : -1;
    pp.probe_div = div_env >= 0 ? div_env : (a.q >= 64 && probe_env <= 0 && !hbm_bound ? 8 : 0);
    // partial probe tiles (rows by cp.async only, decided on the device): VRS_PROBE_ROWS rows per probed tile
    static const int prow_env = getenv("VRS_PROBE_ROWS") ? atoi(getenv("VRS_PROBE_ROWS")) : 0;
    static const int prow_q = getenv("VRS_PROBE_ROWS_Q") ? atoi(getenv("VRS_PROBE_ROWS_Q")) : 8;
    pp.probe_rows = prow_env > 0 && a.q <= prow_q ? (std::min(prow_env, 256) + 7) / 8 * 8 : 0;
    // one wave: the probe's CTAs are few-tile items, so fixed per-CTA costs (prologue,
    // pipeline fill / drain) dominate over several waves -- use at most 148 / qtiles
    // splits (the same density: the step follows the main pass's span)
    static const bool full_p = getenv("VRS_PROBE_FULLP") != nullptr;
    // ... but enough splits that a query has >= 4 k' probe values (2 lists x 32 slots per split):
    // gtau is the k'-th largest of them, and with k' near their count it degenerates to their
    // minimum (C4 Q = 8192: 128 values for k' = 128 doubled the main pass's survivors)
    const int32_t p_probe = full_p ? plan.P
                                   : std::max(1, std::min(plan.P, std::max(kSmCountB200 / std::max(1, plan.qtiles),
                                                                           (4 * a.kprime + 63) / 64)));
    pp.P = p_probe;
    pp.P_main = plan.P;
    pp.min_p_main = p.min_p;
    e = tc_launch_mode<MODE_PROBE>(L, pp, s);
    if (e != cudaSuccess) return e;
    ThresholdArgs ta{gs.probe_max, pp.P * kListsPerSplit * tc::SLOTS, a.q, a.kprime, gs.gtau,
                     SplitInfo{a.ids, a.count, p.allow_gather, pp.P, a.n, p.xsel_cap, tc::BN, p.min_span, p.min_p}};
    ProfScope pt("gemm.threshold", s);
    e = launch_threshold(ta, s);
    if (e != cudaSuccess) return e;
    if (launches) *launches += 2;
  }
  // CTA pairs (tc_kernel.cuh PAIR): an even number of query tiles, 16-bit operands streamed
  // A, no gather4 -- every row tile is staged once per query-tile pair, half in each CTA
  if (pair_main(plan.qtiles, a.d, L.bf) && !L.ar && p.g4 != 1 && p.nseg == 1) {
    const int64_t xcap = a.ids ? a.xsel_cap : 0;
    const bool by_id = xcap > 0 && a.xsel == nullptr;   // (rows by id: no X_sel map to resize)
    if (!make_map(&L.mx, a.Xb, a.n, a.d, tc::BN / 2, true, a.fmt16) ||
        (!by_id && !make_map(&L.mg, xcap > 0 ? a.xsel : a.Xb, xcap > 0 ? xcap : a.n, a.d, tc::BN / 2, true, a.fmt16)))
      return cudaErrorInvalidValue;
    L.pair = true;
    p.idesc = mma_idesc(2 * tc::BM, tc::BN, (uint32_t)a.fmt16);
  }
  {
    ProfScope pf("gemm.main", s);
    e = tc_launch_mode<MODE_MAIN>(L, p, s);
    if (e != cudaSuccess) return e;
  }
  if (launches) *launches += 1;
  return cudaGetLastError();
}

// Where the finalize pass reads the GEMM candidate lists.
GemmLists gemm_lists(const GemmArgs &a, const GemmPlan &plan, void *scratch) {
  const GemmScratch gs = carve_gemm(scratch, plan, a.q, a.kprime);
  GemmLists l;
  l.key = gs.cand_key;
  l.id = gs.cand_id;
  l.cnt = gs.cand_cnt;
  l.lists = plan.P * kListsPerSplit;
  l.stride = kp_of(a.kprime) * tc::CAP_FACTOR;
  l.gtau = gs.gtau;
  l.split = SplitInfo{a.ids, a.count, a.masked == 1 ? 0 : (a.masked == 2 ? 2 : 1), plan.P, a.n,
                      a.ids ? a.xsel_cap : 0, tc::BN, tc_min_span(), tc_min_p(plan)};
  return l;
}

}  // namespace vrs

#ifdef VRS_TC_TIMING
namespace vrs {
int tl_read_gemm(unsigned long long *host) { return tl_read(host); }
}
#endif

// ---------------------------------------------------------------- the refine pass
// ("Refine".)  The queries whose fp16 selection was not certified
// (cert = 0 after finalize) are re-selected with keys that carry fp32-level accuracy:
// each 16-bit operand is split into hi + lo halves (x_lo built at load, q_lo here) and
// the pass multiplies q_hi.x_hi + q_hi.x_lo + q_lo.x_hi into one fp32 accumulator --
// three K segments of the same tcgen05 kernel over masked row tiles.  The threshold is
// provable from level 0: the true k-th score is >= s_k (k re-scored rows reach it), so a
// row of the true top k has a refine key >= s_k - E1; the pass needs no probe.

namespace vrs {

// One CTA of 1024 threads: compact the uncertified queries (ascending), then per compacted
// row (a warp each): the [q_hi | q_lo] fp16 row with its exponent and residuals, and the
// key threshold (s_k - E1) in the pass's key domain.  Rows past the count up to the tile
// boundary are zero with an unreachable threshold.
__global__ void __launch_bounds__(1024) refine_prep_kernel(RefineArgs r) {
  __shared__ int s_wsum[32];
  __shared__ int s_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  pdl_wait();
  pdl_trigger();
  if (tid == 0) s_base = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < r.q; c0 += 1024) {
    const int64_t j = c0 + tid;
    const bool f = j < r.q && r.cert[j] == 0;
    const uint32_t bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_wsum[warp] = __popc(bal);
    __syncthreads();
    int before = s_base;
    for (int w = 0; w < warp; ++w) before += s_wsum[w];
    if (f) r.qlist[before + __popc(bal & lanemask_lt())] = (int32_t)j;
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < 32; ++w) t += s_wsum[w];
      s_base += t;
    }
    __syncthreads();
  }
  const int U = s_base;
  if (tid == 0) *r.ucount = U;
  if (U == 0) return;
  const int64_t upad = std::min<int64_t>(r.rows, ((int64_t)U + tc::BM - 1) / tc::BM * tc::BM);
  for (int64_t row = warp; row < upad; row += 32) {
    uint16_t *hi = r.qr + row * 2 * r.dpad, *lo = hi + r.dpad;
    if (row >= U) {   // padding rows of the last tile
      for (int t = lane; t < 2 * r.dpad; t += 32) hi[t] = 0;
      if (lane == 0) {
        r.qexp[row] = 0;
        r.rqa[row] = 0.f;
        r.rq2[row] = 0.f;
        r.gtau[row] = 0xffffffffu;   // (+inf: nothing passes)
      }
      continue;
    }
    const int64_t j = r.qlist[row];
    const float *qv = r.Q + j * r.d;
    float am = 0.f;
    double qq = 0.0;
    for (int t = lane; t < r.d; t += 32) {
      am = fmaxf(am, fabsf(qv[t]));
      qq += (double)qv[t] * (double)qv[t];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
      qq += __shfl_xor_sync(0xffffffffu, qq, o);
    }
    const int e = scale_exp16(am, 0);
    const double2 rr = row_to16x2(qv, hi, lo, r.d, e);
    for (int t = r.d + lane; t < r.dpad; t += 32) { hi[t] = 0; lo[t] = 0; }
    if (lane == 0) {
      const double r1 = sqrt(rr.x), r2 = sqrt(rr.y) * (1.0 + 0x1p-50);
      const double rqa = (r1 + r2) * (1.0 + 0x1p-50);   // |q_lo| <= |q_hi - q| + |q_hi + q_lo - q|
      r.qexp[row] = e;
      r.rqa[row] = __double2float_ru(rqa);
      r.rq2[row] = __double2float_ru(r2);
      const double qn = sqrt(qq), skv = r.sk[j];
      const double E1 = key_error_bound_x3(r.kb, r.metric, qn, (double)__double2float_ru(rqa), (double)__double2float_ru(r2));
      const double nat = r.metric == VRS_L2 ? qq + skv : (r.metric == VRS_COSINE ? skv * qn : skv);
      double T = nat - E1 - 0x1p-30 * (fabs(nat) + qn * r.kb.xmax);
      if (r.metric != VRS_L2) T = ldexp(T, e + r.xexp);   // IP / COS keys are in the domain 2^(e_q + e_x)
      r.gtau[row] = ordered_u32(__double2float_rd(T));
    }
  }
}

cudaError_t launch_refine(const RefineArgs &r, const GemmArgs &a, const GemmPlan &plan, void *gemm_scratch,
                          const void *x_lo, cudaStream_t s, int *launches) {
  cudaError_t e = launch_k(refine_prep_kernel, dim3(1), dim3(1024), 0, s, r);
  if (e != cudaSuccess) return e;
  // row delivery: with xsel_lo, level 0's (the same device decision from the same count):
  // X_sel (its x_hi rows, still in place) + X_sel_lo (x_lo rows, copied here) by TMA, rows by
  // id (cp.async), or masked tiles.  Without (no memory for it): gathered by cp.async (hi and
  // lo halves by id) up to the masked break-even, else masked tiles.
  GemmArgs b = a;
  b.prepped = 1;
  b.xsel_ready = 1;
  const bool own = r.xsel_lo != nullptr && a.xsel != nullptr;
  if (!own) {
    b.masked = 0;
    b.xsel_cap = a.ids ? r.gather_cap : 0;
    b.xsel = nullptr;
    b.cp_min_bytes = 0;
  }
  TcLaunch L;
  e = tc_prepare(b, plan, s, launches, &L);
  if (e != cudaSuccess) return e;
  if (!make_map(&L.mq, r.qr, r.rows, 2 * r.dpad, tc::BM, true, 0) || !make_map(&L.ml, x_lo, a.n, a.d, tc::BN, true, 0))
    return cudaErrorInvalidValue;
  L.mlg = L.ml;
  if (own) {
    if (!make_map(&L.mlg, r.xsel_lo, L.p.xsel_cap, a.d, tc::BN, true, 0)) return cudaErrorInvalidValue;
    ProfScope pg("refine.gather", s);   // x_lo rows of the selection (exactly when level 0 copied x_hi)
    e = launch_k(gather_copy_kernel, dim3(8 * 148), dim3(256), 0, s, x_lo, a.d * 2, a.ids, a.count, a.n,
                 (int)L.p.allow_gather, L.p.xsel_cap, r.xsel_lo, (const float *)nullptr, (float *)nullptr,
                 L.p.cp_min_bytes, L.p.cp_min_rows);
    if (e != cudaSuccess) return e;
    if (launches) *launches += 1;
  }
  const GemmScratch gs = carve_gemm(gemm_scratch, plan, a.q, a.kprime);
  TcParams &p = L.p;
  p.cand_key = gs.cand_key;   // (level 0's lists: its finalize has read them)
  p.cand_id = gs.cand_id;
  p.cand_cnt = gs.cand_cnt;
  p.probe_max = gs.probe_max;
  p.gtau = r.gtau;
  p.qexp = r.qexp;
  p.nseg = 3;
  p.a_lo_off = r.dpad;
  p.qcount = r.ucount;
  p.xrows_lo = x_lo;
  if (!own) {
    p.g4 = 2;
    p.cp_min_bytes = 0;
  }
  L.ar = false;
  {
    ProfScope pf("refine.main", s);
    e = tc_launch_mode<MODE_MAIN>(L, p, s);
  }
  if (launches) *launches += 2;
  return e;
}

}  // namespace vrs
