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
// tiles).  Warp roles (256 threads, 1 CTA / SM):
//   warp 0  TMA producer: query block [128 x 32 fp32] + row block [256 x 32]
//           per stage, 128-byte swizzle, 4-stage mbarrier ring
//   warp 1  TMEM allocator + tcgen05.mma issuer (kind::tf32, M=128, N=256,
//           K=8 per instruction), fp32 accumulators double-buffered in TMEM
//           (2 x 256 columns)
//   warp 2  per-row epilogue terms: ranking-key scale/bias of each of the 256
//           rows of a tile (norm terms, bitmap mask) and row ids, 2-stage ring
//   warps 4-7 epilogue: tcgen05.ld 32 columns at a time, key = fma(dot, a, b),
//           compare with the query's running threshold, rare append to a
//           per-(work item, query) candidate buffer, warp-cooperative radix
//           compaction to the best KP when a buffer fills.
// Precision: TF32 products, fp32 accumulation -> selection only; the k' = k+16
// best per query are re-scored exactly in finalize.cu.
//
// Roofline: tensor (2*q*N_rows*d TF32 flops) for large q, HBM (4*d bytes per
// row) for small q.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "vrs_kernels.cuh"

namespace vrs {

namespace tc {
constexpr int BM = 128;         // queries per tile (TMEM lanes)
constexpr int BN = 256;         // rows per tile (TMEM columns, MMA N)
constexpr int BK = 32;          // fp32 per K block = 128 bytes = one swizzle span
constexpr int PIPE_BYTES = 192 * 1024;   // shared-memory pipeline region (A resident and/or stages)
constexpr int MAX_STAGES = 8;
constexpr int A_BYTES = BM * BK * 4;   // 16 KB
constexpr int B_BYTES = BN * BK * 4;   // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int ACC_STAGES = 2;   // accumulator tiles in TMEM (2 x 256 columns)
constexpr int TMEM_COLS = 512;
constexpr int EPI_WARP0 = 4;
constexpr int EPI_WARPS = 8;    // 2 per TMEM lane quadrant, each owning half of the tile's columns
constexpr int EPI_COLS = BN / 2;
constexpr int THREADS = (EPI_WARP0 + EPI_WARPS) * 32;
constexpr int CAP_FACTOR = 4;   // candidate buffer = CAP_FACTOR * KP entries per (item, query, half)
constexpr int BIAS_STAGES = 4;
constexpr int STAGE_COLS = 16;  // per-warp key staging: one private row of 16 fp32 per lane
// dynamic smem: [stages][A|B] (1024-aligned) + bias a/b/id [BIAS_STAGES][BN] + per-warp key staging
// (the staging area doubles as the compaction histogram)
constexpr size_t SMEM_BYTES =
    1024 + (size_t)PIPE_BYTES + BIAS_STAGES * BN * 12 + EPI_WARPS * 32 * STAGE_COLS * 4 + 256;
}  // namespace tc

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// ---- CTA-pair (cta_group::2) helpers: the even CTA of a 2-CTA cluster issues the
// MMA for both; barrier addresses with bit 24 cleared name the even CTA's copy.
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;" ::: "memory");
}
// TMA executed by both CTAs of the pair; the transaction bytes land on the even CTA's barrier.
__device__ __forceinline__ void tma_load_2d_pair(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_mma_tf32_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// MMA completion -> arrive on the barrier at this offset in both CTAs of the pair.
__device__ __forceinline__ void tc_commit_pair(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & kPeerMask)
               : "memory");
}

// D[tmem] (+)= A[smem] . B[smem]^T, kind::tf32, both operands K-major.
__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Shared-memory matrix descriptor, K-major operand in the canonical
// 128-byte-swizzle layout written by TMA (8-row groups of 1024 bytes).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);   // start address
  d |= (uint64_t)1 << 16;                   // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;         // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                   // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                   // SWIZZLE_128B
  return d;
}

// Instruction descriptor: D fp32, A/B tf32, both K-major, N = BN, M = BM.
__host__ __device__ constexpr uint32_t tf32_idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

#define TMEM_LD_32x32b_X32(taddr, r)                                                                              \
  asm volatile(                                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19," \
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                                  \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),  \
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),      \
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),     \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                  \
      : "r"(taddr))

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- kernel
struct TcParams {
  int64_t n_rows;          // rows of the index (identity / masked row space)
  const int32_t *ids;      // compacted ascending selection (nullptr: no predicate)
  const int64_t *count;    // device count of ids
  int32_t allow_gather;    // gathered-row mode allowed (selectivity switch decides on device)
  int32_t d;
  int32_t nk;              // K blocks = ceil(d / 32)
  int64_t q;
  int32_t qtiles;
  int32_t P;               // splits
  int32_t tile_step;       // 1: every tile; > 1: probe pass over every tile_step-th tile
  float *dense;            // sample pass: raw keys [q][ldd] of the first dense_tiles row tiles (no top-k)
  int32_t ldd;
  int32_t dense_tiles;
  int64_t row_tiles_max;   // ceil(n_rows / BN)
  const uint32_t *bitmap;  // nullptr => every row qualifies
  const float *nx2;
  const float *inv_nx;
  int32_t metric;
  int32_t kp;              // retained entries per (item, query) (pow2 >= k')
  int32_t cap;             // buffer capacity per (item, query)
  float *cand_key;         // [2P][q][cap]
  int32_t *cand_id;
  const float *X;          // corpus base
  int64_t xsel_cap;        // rows of the materialised-selection buffer
  uint32_t *gtau;          // [q] ordered-u32 threshold shared by all lists of a query (0 = none yet)
  float *list_tau;         // [2P][q] final KP-th best key per list (-inf: list never filled)
  unsigned long long *stats;  // optional counters: chunks, slow chunks, flagged queries, compactions
  float *dense_buf;        // host-provided scratch for the sample pass [q][SAMPLE_TILES * BN]
  int32_t epi_skip;        // debug: epilogue only drains TMEM (pipeline-bound measurement)
  int32_t part;            // 0: whole item; 1: first 1/PART_DIV of its tiles; 2: the rest (resumes part 1)
  int32_t *cnt_state;      // [2P][q] list fill carried from part 1 to part 2
  float *tau_state;        // [2P][q] list threshold carried from part 1 to part 2
};

// Warp-cooperative compaction of one lane's candidate buffer to its best KP
// entries (key desc, then buffer order = ascending row id).  Returns the new
// threshold key (the KP-th best).  All 32 lanes call it with the same `owner`.
__device__ float compact_lane(float *key, int32_t *id, int cnt, int kp, uint32_t *hist) {
  const int lane = threadIdx.x & 31;
  uint32_t prefix = 0, mask = 0;
  int rem = kp;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = lane; b < 256; b += 32) hist[b] = 0;
    __syncwarp();
    for (int i = lane; i < cnt; i += 32) {
      const uint32_t ok = ordered_u32(key[i]);
      if ((ok & mask) == prefix) atomicAdd(&hist[(ok >> shift) & 255u], 1u);
    }
    __syncwarp();
    uint32_t v[8], s = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) { v[t] = hist[255 - 8 * lane - t]; s += v[t]; }
    uint32_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
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
    const uint32_t who = __ballot_sync(0xffffffffu, bin >= 0);
    const int src = __ffs(who) - 1;
    bin = __shfl_sync(0xffffffffu, bin, src);
    above = __shfl_sync(0xffffffffu, above, src);
    prefix |= (uint32_t)bin << shift;
    mask |= 255u << shift;
    rem -= above;
    __syncwarp();
  }
  // stable in-place compaction: keys strictly above the threshold, plus the
  // first `rem` ties in buffer order
  int out = 0, ties = 0;
  for (int base = 0; base < cnt; base += 32) {
    const int i = base + lane;
    float kv = -INFINITY;
    int32_t iv = -1;
    uint32_t ok = 0;
    if (i < cnt) { kv = key[i]; iv = id[i]; ok = ordered_u32(kv); }
    const bool tie = (i < cnt) && ok == prefix;
    const uint32_t tmask = __ballot_sync(0xffffffffu, tie);
    const int my_tie_rank = ties + __popc(tmask & lanemask_lt());
    ties += __popc(tmask);
    const bool keep = (i < cnt) && (ok > prefix || (tie && my_tie_rank < rem));
    const uint32_t kmask = __ballot_sync(0xffffffffu, keep);
    const int pos = out + __popc(kmask & lanemask_lt());
    __syncwarp();
    if (keep) { key[pos] = kv; id[pos] = iv; }
    out += __popc(kmask);
    __syncwarp();
  }
  const uint32_t u = (prefix & 0x80000000u) ? (prefix & 0x7fffffffu) : ~prefix;
  return __uint_as_float(u);
}

// Gathered rows iff a selection exists, it is at most half the rows (or forced)
// and it fits the materialisation buffer.
__device__ __forceinline__ bool gather_mode(const int32_t *ids, int allow, int64_t n_sel, int64_t n, int64_t cap) {
  if (ids == nullptr || allow == 0 || n_sel > cap) return false;
  return allow == 2 || n_sel * 2 <= n;
}

// Late materialization ("(re-)materialized into dense
// vectors"): X_sel[r] = X[ids[r]], one warp per row, 16-byte vector copies.
// HBM-bound: 2 * 4d bytes per selected row.
__global__ void __launch_bounds__(256) gather_copy_kernel(const float *__restrict__ X, int32_t d,
                                                          const int32_t *__restrict__ ids,
                                                          const int64_t *__restrict__ count, int64_t n, int allow,
                                                          int64_t cap, float *__restrict__ xsel) {
  const int64_t n_sel = *count;
  if (!gather_mode(ids, allow, n_sel, n, cap)) return;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int d4 = d >> 2;
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n_sel; r += warps) {
    const float4 *src = reinterpret_cast<const float4 *>(X + (int64_t)__ldg(ids + r) * d);
    float4 *dst = reinterpret_cast<float4 *>(xsel + r * d);
    for (int i = lane; i < d4; i += 32) dst[i] = __ldg(src + i);
  }
}

// AR: the query tile stays resident in shared memory (d <= 128).
// CG: 1 = one CTA per 128-query tile; 2 = CTA pair (cluster of 2) sharing every row
//     tile: M = 256 queries per MMA, each CTA stages half of the rows (cta_group::2),
//     halving the L2 -> SM traffic per query.
template <bool AR, int CG>
__global__ void __launch_bounds__(tc::THREADS, 1)
    tc_topk_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_x,
                   const __grid_constant__ CUtensorMap tmap_g, TcParams p) {
  using namespace tc;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment (128B swizzle atoms) by pointer arithmetic on the shared
  // array itself, so the compiler keeps the shared address space (LDS, not LD)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // pipeline region (STAGES * STAGE_BYTES): AR ? [A: nk x 16 KB][B stages of 32 KB]
  //                                              : [stages of (A 16 KB | B 32 KB)]
  uint8_t *stage_base = smem;
  constexpr int B_LOCAL = B_BYTES / CG;                  // this CTA's share of a row tile
  constexpr int SSTRIDE = AR ? B_LOCAL : A_BYTES + B_LOCAL;   // bytes per pipeline stage
  // as many stages as the 192 KB pipeline region holds (TMA latency needs depth)
  constexpr int NST = ((PIPE_BYTES - (AR ? 4 * A_BYTES : 0)) / SSTRIDE) < MAX_STAGES
                          ? ((PIPE_BYTES - (AR ? 4 * A_BYTES : 0)) / SSTRIDE)
                          : MAX_STAGES;
  constexpr int BOFF = AR ? 0 : A_BYTES;                 // B offset within a stage
  uint8_t *a_res = smem;                                 // AR: resident query tile
  uint8_t *b_base = AR ? smem + 4 * A_BYTES : smem;
  float *bias_a = reinterpret_cast<float *>(smem + PIPE_BYTES);               // [BIAS_STAGES][BN]
  float *bias_b = bias_a + BIAS_STAGES * BN;                                    // [BIAS_STAGES][BN]
  int32_t *row_id = reinterpret_cast<int32_t *>(bias_b + BIAS_STAGES * BN);     // [BIAS_STAGES][BN]
  float *kstage = reinterpret_cast<float *>(row_id + BIAS_STAGES * BN);        // [EPI_WARPS][32][STAGE_COLS]

  __shared__ __align__(8) uint64_t full_bar[MAX_STAGES], empty_bar[MAX_STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[ACC_STAGES], tempty_bar[ACC_STAGES];
  __shared__ __align__(8) uint64_t bfull_bar[BIAS_STAGES], bempty_bar[BIAS_STAGES];
  __shared__ __align__(8) uint64_t afull_bar;
  __shared__ uint32_t tmem_base_s;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = CG == 2 ? (int)cluster_ctarank() : 0;
  const int qgroups = (p.qtiles + CG - 1) / CG;
  const int item = blockIdx.x / CG;
  const int qtile = (item % qgroups) * CG + rank;
  const int split = item / qgroups;
  // Selectivity-driven row delivery (decided on the device, no host sync):
  //  gather: the selection was materialised densely (gather_copy_kernel, late
  //          materialization) and streams by TMA from X_sel; ids map rows back
  //  masked: every row streams by TMA, unqualified rows are masked by the bitmap
  const int64_t n_sel = p.ids ? *p.count : p.n_rows;
  const bool gather = gather_mode(p.ids, p.allow_gather, n_sel, p.n_rows, p.xsel_cap);
  const int64_t n_space = gather ? n_sel : p.n_rows;
  const int64_t row_tiles = (n_space + BN - 1) / BN;
  // splits actually used: >= 16 row tiles per item when the (device-side) row
  // space allows -- the fused top-k warms up once per item; CTAs of unused
  // splits only publish empty candidate lists
  // (sample pass: the first dense_tiles row tiles, split over all P splits)
  const int64_t t_space = p.dense ? std::min<int64_t>(row_tiles, p.dense_tiles) : row_tiles;
  const int64_t p_eff = p.dense ? p.P : std::max<int64_t>(1, std::min<int64_t>(p.P, row_tiles / 4));
  const int64_t i_begin = split < p_eff ? (t_space * split) / p_eff : 0;
  const int64_t i_end = split < p_eff ? (t_space * (split + 1)) / p_eff : 0;
  // two-part main pass: part 1 covers the first 1/PART_DIV of the item's tiles,
  // a per-query selection over every list then raises the shared threshold, and
  // part 2 resumes the lists over the remaining tiles
  constexpr int PART_DIV = 8;
  const int64_t i_mid = i_begin + (i_end - i_begin + PART_DIV - 1) / PART_DIV;
  const int64_t t_begin = p.part == 2 ? i_mid : i_begin;
  const int64_t t_end = p.part == 1 ? i_mid : i_end;
  // probe pass (tile_step > 1): every tile_step-th tile of the item, and only when
  // the item is long enough for a threshold to pay off
  const int64_t span = t_end - t_begin;
  // probe: ~1/tile_step of the item's tiles (at least 4 of them, at most every 2nd)
  const int step = p.tile_step == 1 ? 1 : (int)std::max<int64_t>(2, std::min<int64_t>(p.tile_step, span / 4));
  // (the probe only pays off for masked full tiles: the gathered selection is short)
  const int ntiles = p.tile_step == 1 ? (int)span : (span >= 8 && !gather ? (int)((span + step - 1) / step) : 0);
  auto tile_of = [&](int t) -> int64_t { return t_begin + (int64_t)t * step; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    mbar_init(&afull_bar, 1);
    for (int s = 0; s < ACC_STAGES; ++s) { mbar_init(&tfull_bar[s], 1); mbar_init(&tempty_bar[s], EPI_WARPS * CG); }
    for (int s = 0; s < BIAS_STAGES; ++s) {
      mbar_init(&bfull_bar[s], 32);
      mbar_init(&bempty_bar[s], EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) { prefetch_tmap(&tmap_q); prefetch_tmap(&tmap_x); prefetch_tmap(&tmap_g); }
  if (warp == 1) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                   "n"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                   "n"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // (pair: both CTAs load their own A and their half of B; the even CTA
      //  accounts for the pair's bytes on its barriers)
      auto load = [&](void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
        if (CG == 2) tma_load_2d_pair(dst, map, bar, c0, c1);
        else tma_load_2d(dst, map, bar, c0, c1);
      };
      if (AR && ntiles > 0) {
        if (rank == 0) mbar_expect_tx(&afull_bar, CG * p.nk * A_BYTES);
        for (int kb = 0; kb < p.nk; ++kb) load(a_res + kb * A_BYTES, &tmap_q, &afull_bar, kb * BK, qtile * BM);
      }
      for (int t = 0; t < ntiles; ++t) {
        const int row0 = (int)(tile_of(t) * BN) + rank * (BN / CG);
        for (int kb = 0; kb < p.nk; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t *st = b_base + stage * SSTRIDE;
          if (rank == 0) mbar_expect_tx(&full_bar[stage], CG * (AR ? B_LOCAL : A_BYTES + B_LOCAL));
          if (!AR) load(st, &tmap_q, &full_bar[stage], kb * BK, qtile * BM);
          load(st + BOFF, gather ? &tmap_g : &tmap_x, &full_bar[stage], kb * BK, row0);
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (even CTA of a pair)
    constexpr uint32_t idesc = tf32_idesc(BM * CG, BN);
    if (CG == 1 || rank == 0) {
    int stage = 0;
    uint32_t phase = 0;
    if (AR && ntiles > 0) mbar_wait(&afull_bar, 0);
    for (int t = 0; t < ntiles; ++t) {
      const int acc = t % ACC_STAGES;
      const uint32_t acc_phase = (t / ACC_STAGES) & 1;
      mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < p.nk; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sb = smem_u32(b_base + stage * SSTRIDE + BOFF);
          const uint32_t sa = AR ? smem_u32(a_res + kb * A_BYTES) : sb - A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {  // K = 8 tf32 = 32 bytes per instruction
            if (CG == 2) tc_mma_tf32_pair(d_tmem, sw128_desc(sa + k * 32), sw128_desc(sb + k * 32), idesc, (kb | k) != 0);
            else tc_mma_tf32(d_tmem, sw128_desc(sa + k * 32), sw128_desc(sb + k * 32), idesc, (kb | k) != 0);
          }
          // frees the smem slot(s) when these MMAs finish; accumulator ready after the last K block
          if (CG == 2) {
            tc_commit_pair(&empty_bar[stage]);
            if (kb == p.nk - 1) tc_commit_pair(&tfull_bar[acc]);
          } else {
            tc_commit(&empty_bar[stage]);
            if (kb == p.nk - 1) tc_commit(&tfull_bar[acc]);
          }
        }
        __syncwarp();
        if (++stage == NST) { stage = 0; phase ^= 1; }
      }
    }
    }
  } else if (warp == 2) {
    // ------------------------------------------------ per-row epilogue terms
    // Loads for tile t + PF are issued before tile t is written out: the warp is
    // memory-latency bound otherwise (one ~us round trip per tile).
    constexpr int PF = 4;
    const float *src = p.metric == VRS_L2 ? p.nx2 : p.inv_nx;
    constexpr int RPL = BN / 32;   // rows per lane
    float nv[PF][RPL];
    int32_t iv[PF][RPL];
    uint32_t wv[PF];
    auto fetch = [&](int t, float (&n8)[RPL], int32_t (&i8)[RPL], uint32_t &w) {
      if (t >= ntiles) return;
      const int64_t pos0 = tile_of(t) * BN + lane * RPL;   // this lane: RPL consecutive row-space slots
      if (gather) {
        if (pos0 + RPL <= n_sel) {
#pragma unroll
          for (int v = 0; v < RPL / 4; ++v) {
            const int4 i0 = __ldg(reinterpret_cast<const int4 *>(p.ids + pos0) + v);
            i8[4 * v] = i0.x; i8[4 * v + 1] = i0.y; i8[4 * v + 2] = i0.z; i8[4 * v + 3] = i0.w;
          }
        } else {
#pragma unroll
          for (int u = 0; u < RPL; ++u) i8[u] = pos0 + u < n_sel ? __ldg(p.ids + pos0 + u) : -1;
        }
#pragma unroll
        for (int u = 0; u < RPL; ++u) n8[u] = i8[u] >= 0 ? __ldg(src + i8[u]) : 0.f;
        w = 0xffffffffu;
      } else {
        w = 0xffffffffu;
        if (p.bitmap && pos0 < p.n_rows) w = __ldg(p.bitmap + (pos0 >> 5));
        if (pos0 + RPL <= p.n_rows) {
#pragma unroll
          for (int v = 0; v < RPL / 4; ++v) {
            const float4 v0 = __ldg(reinterpret_cast<const float4 *>(src + pos0) + v);
            n8[4 * v] = v0.x; n8[4 * v + 1] = v0.y; n8[4 * v + 2] = v0.z; n8[4 * v + 3] = v0.w;
          }
        } else {
#pragma unroll
          for (int u = 0; u < RPL; ++u) n8[u] = pos0 + u < p.n_rows ? __ldg(src + pos0 + u) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < RPL; ++u) i8[u] = pos0 + u < p.n_rows ? (int32_t)(pos0 + u) : -1;
      }
    };
#pragma unroll
    for (int u = 0; u < PF; ++u) fetch(u, nv[u], iv[u], wv[u]);
    for (int t0 = 0; t0 < ntiles; t0 += PF) {
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int t = t0 + u;
        if (t >= ntiles) break;
        const int s = t % BIAS_STAGES;
        mbar_wait(&bempty_bar[s], ((t / BIAS_STAGES) & 1) ^ 1);
        const int64_t pos0 = tile_of(t) * BN + lane * RPL;
        float av[RPL], bv[RPL];
#pragma unroll
        for (int k = 0; k < RPL; ++k) {
          const bool valid = iv[u][k] >= 0 && (gather || ((wv[u] >> ((pos0 + k) & 31)) & 1u));
          float a = 1.f, b = valid ? 0.f : -INFINITY;
          if (p.metric == VRS_L2) {
            a = 2.f;
            if (valid) b = -nv[u][k];
          } else if (p.metric == VRS_COSINE) {
            a = valid ? nv[u][k] : 0.f;
          }
          av[k] = a; bv[k] = b;
        }
#pragma unroll
        for (int v = 0; v < RPL / 4; ++v) {
          reinterpret_cast<float4 *>(bias_a + s * BN + lane * RPL)[v] =
              make_float4(av[4 * v], av[4 * v + 1], av[4 * v + 2], av[4 * v + 3]);
          reinterpret_cast<float4 *>(bias_b + s * BN + lane * RPL)[v] =
              make_float4(bv[4 * v], bv[4 * v + 1], bv[4 * v + 2], bv[4 * v + 3]);
          reinterpret_cast<int4 *>(row_id + s * BN + lane * RPL)[v] =
              make_int4(iv[u][4 * v], iv[u][4 * v + 1], iv[u][4 * v + 2], iv[u][4 * v + 3]);
        }
        mbar_arrive(&bfull_bar[s]);
        fetch(t + PF, nv[u], iv[u], wv[u]);
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ------------------------------------------------ epilogue: fused top-k
    const int ew = warp - EPI_WARP0;
    const int quad = warp & 3;                     // TMEM lane quadrant this warp may access
    const int half = ew >> 2;                      // which 128 of the tile's 256 columns
    const int m = quad * 32 + lane;                // query row within the tile
    const int64_t qg = (int64_t)qtile * BM + m;    // global query index
    const bool active = qg < p.q;
    const int list = split * 2 + half;             // candidate list index
    const int64_t cbase = ((int64_t)list * p.q + (active ? qg : 0)) * p.cap;
    float *ckey = p.cand_key + cbase;
    int32_t *cid = p.cand_id + cbase;
    float *wst = kstage + ew * 32 * STAGE_COLS;
    uint32_t *whist = reinterpret_cast<uint32_t *>(wst);   // compaction histogram aliases the staging area
    float tau = active ? -INFINITY : INFINITY;     // inactive lanes never accept
    int cnt = 0;
    if (p.part == 2 && active) {   // resume the list built by part 1
      cnt = p.cnt_state[(int64_t)list * p.q + qg];
      tau = p.tau_state[(int64_t)list * p.q + qg];
    }

    // Thresholds: `tau` (own list, strict: later rows have larger ids) and the
    // query's shared threshold gtau (max over every list's KP-th best key --
    // any list's KP-th best bounds the global KP-th best from below).  A key is
    // a candidate iff key > tau and key >= gtau; both fold into `thr`.
    uint32_t *gtau_q = p.gtau + (active ? qg : 0);
    auto shared_bound = [](uint32_t o) -> float {   // largest float strictly below the shared key
      if (o == 0) return -INFINITY;
      const uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
      return nextafterf(__uint_as_float(u), -INFINITY);
    };
    float thr = tau;
    uint32_t st_chunks = 0, st_slow = 0, st_flag = 0, st_comp = 0;
    auto compact_needed = [&](int threshold) {
      uint32_t need = __ballot_sync(0xffffffffu, cnt > threshold);
      while (need) {
        const int owner = __ffs(need) - 1;
        need &= need - 1;
        const int oc = __shfl_sync(0xffffffffu, cnt, owner);
        const int64_t ob = ((int64_t)list * p.q + (int64_t)qtile * BM + quad * 32 + owner) * p.cap;
        const float nt = compact_lane(p.cand_key + ob, p.cand_id + ob, oc, p.kp, whist);
        ++st_comp;
        if (lane == owner) {
          tau = nt;
          cnt = p.kp;
          thr = fmaxf(thr, tau);
          atomicMax(gtau_q, ordered_u32(tau));
        }
      }
    };

    uint32_t g_next = active ? __ldcg(gtau_q) : 0u;
    for (int t = 0; t < ntiles; ++t) {
      const int acc = t % ACC_STAGES;
      const int bs = t % BIAS_STAGES;
      if (active) thr = fmaxf(thr, shared_bound(g_next));
      if (active) g_next = __ldcg(gtau_q);   // consumed at the next tile (latency hidden)
      mbar_wait(&bfull_bar[bs], (t / BIAS_STAGES) & 1);
      mbar_wait(&tfull_bar[acc], (t / ACC_STAGES) & 1);
      tc_fence_after();
      const float *ba = bias_a + bs * BN + half * EPI_COLS;
      const float *bb = bias_b + bs * BN + half * EPI_COLS;
      const int32_t *rid = row_id + bs * BN + half * EPI_COLS;
      const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * BN + half * EPI_COLS);
      if (p.epi_skip) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 2) mbar_arrive_leader(&tempty_bar[acc]);
          else mbar_arrive(&tempty_bar[acc]);
          mbar_arrive(&bempty_bar[bs]);
        }
        continue;
      }
      uint32_t r[2][32];
      TMEM_LD_32x32b_X32(tbase, r[0]);
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < EPI_COLS / 32; ++c) {
        uint32_t(&cur)[32] = r[c & 1];
        if (c + 1 < EPI_COLS / 32) TMEM_LD_32x32b_X32(tbase + (c + 1) * 32, r[(c + 1) & 1]);
        float key[32];
        float kmax = -INFINITY;
        if (p.metric == VRS_COSINE) {   // per-row scale 1/|x|
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 a4 = *reinterpret_cast<const float4 *>(ba + c * 32 + i);
            const float4 b4 = *reinterpret_cast<const float4 *>(bb + c * 32 + i);
            key[i] = fmaf(__uint_as_float(cur[i]), a4.x, b4.x);
            key[i + 1] = fmaf(__uint_as_float(cur[i + 1]), a4.y, b4.y);
            key[i + 2] = fmaf(__uint_as_float(cur[i + 2]), a4.z, b4.z);
            key[i + 3] = fmaf(__uint_as_float(cur[i + 3]), a4.w, b4.w);
          }
        } else {                        // constant scale (L2: 2, IP: 1), per-row bias
          const float sc = p.metric == VRS_L2 ? 2.f : 1.f;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b4 = *reinterpret_cast<const float4 *>(bb + c * 32 + i);
            key[i] = fmaf(__uint_as_float(cur[i]), sc, b4.x);
            key[i + 1] = fmaf(__uint_as_float(cur[i + 1]), sc, b4.y);
            key[i + 2] = fmaf(__uint_as_float(cur[i + 2]), sc, b4.z);
            key[i + 3] = fmaf(__uint_as_float(cur[i + 3]), sc, b4.w);
          }
        }
#pragma unroll
        for (int i = 0; i < 32; i += 2) kmax = fmaxf(kmax, fmaxf(key[i], key[i + 1]));
        ++st_chunks;
        if (p.dense) {   // sample pass: raw keys out, no selection
          if (active) {
            float *dst = p.dense + qg * p.ldd + tile_of(t) * BN + half * EPI_COLS + c * 32;
#pragma unroll
            for (int i = 0; i < 32; i += 4)
              *reinterpret_cast<float4 *>(dst + i) = make_float4(key[i], key[i + 1], key[i + 2], key[i + 3]);
          }
          tmem_ld_wait();
          continue;
        }
        if (__any_sync(0xffffffffu, kmax > thr)) {
          ++st_slow;
          uint32_t amask = 0;   // bit i: column i beats the query's threshold
#pragma unroll
          for (int i = 0; i < 32; ++i) amask |= (key[i] > thr ? 1u : 0u) << i;
          // rare once a threshold exists: make room (<= 32 appends follow; the
          // compaction histogram aliases the staging rows), re-test against the
          // possibly raised threshold, then each lane appends its own columns in
          // row order from its private staging row (16 columns at a time)
          if (__any_sync(0xffffffffu, cnt + __popc(amask) > p.cap)) {
            compact_needed(p.cap - 32);
            amask = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) amask |= (key[i] > thr ? 1u : 0u) << i;
          }
          float *myrow = wst + lane * STAGE_COLS;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t m = (amask >> (16 * h)) & 0xffffu;
            if (m) {
              st_flag += __popc(m);
#pragma unroll
              for (int i = 0; i < 16; i += 4)
                *reinterpret_cast<float4 *>(myrow + i) =
                    make_float4(key[h * 16 + i], key[h * 16 + i + 1], key[h * 16 + i + 2], key[h * 16 + i + 3]);
              const int32_t *rrow = rid + c * 32 + h * 16;
              while (m) {
                const int i = __ffs(m) - 1;
                m &= m - 1;
                ckey[cnt] = myrow[i];
                cid[cnt] = rrow[i];
                ++cnt;
              }
            }
          }
          __syncwarp();
        }
        tmem_ld_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_leader(&tempty_bar[acc]);
        else mbar_arrive(&tempty_bar[acc]);
        mbar_arrive(&bempty_bar[bs]);
      }
    }
    if (p.stats && lane == 0) {
      atomicAdd(p.stats + 0, (unsigned long long)st_chunks);
      atomicAdd(p.stats + 1, (unsigned long long)st_slow);
      atomicAdd(p.stats + 2, (unsigned long long)st_flag);
      atomicAdd(p.stats + 3, (unsigned long long)st_comp);
    }
    if (p.part == 1) {   // hand the list over to part 2
      if (active) {
        p.cnt_state[(int64_t)list * p.q + qg] = cnt;
        p.tau_state[(int64_t)list * p.q + qg] = tau;
      }
    } else {
    // final: keep the best KP, pad the rest of the KP window
    if (!p.dense) compact_needed(p.kp);
    if (active && !p.dense) {
      for (int i = cnt; i < p.kp; ++i) { ckey[i] = -INFINITY; cid[i] = -1; }
      p.list_tau[(int64_t)list * p.q + qg] = tau;
    }
    }
  }

  tc_fence_before();
  if (CG == 2) cluster_sync_all();   // the pair's MMAs and remote arrivals are done
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS) : "memory");
  }
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void *f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

static bool make_map(CUtensorMap *m, const float *base, int64_t rows, int32_t d, int box_rows, int box_cols = tc::BK) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int kp_of(int32_t kprime) {
  int kp = 32;
  while (kp < kprime) kp <<= 1;
  return kp;
}

GemmPlan gemm_plan(int64_t q, int32_t d, int64_t n_upper, int32_t kprime, int num_sms) {
  GemmPlan g{0, 0, 0};
  if (d % 4 != 0 || d < 4 || q < 1 || n_upper < 1 || kprime > 256) return g;
  if (!encode_fn()) return g;
  const int64_t qtiles = (q + tc::BM - 1) / tc::BM;
  const int64_t row_tiles = (n_upper + tc::BN - 1) / tc::BN;
  // one CTA per SM; aim for up to 4 waves of (query tile, row split) items while keeping
  // items >= ~128 row tiles (the fused top-k warms up once per item)
  int64_t waves = std::max<int64_t>(1, std::min<int64_t>(4, row_tiles * qtiles / ((int64_t)num_sms * 128)));
  int64_t P = std::max<int64_t>(1, (int64_t)num_sms * waves / qtiles);
  P = std::min<int64_t>(P, row_tiles);
  g.P = (int32_t)P;
  g.qtiles = (int32_t)qtiles;
  g.ok = 1;
  return g;
}

size_t gemm_scratch_bytes(const GemmPlan &plan, int64_t q, int32_t kprime) {
  const int kp = kp_of(kprime);
  return (size_t)plan.P * 2 * q * kp * tc::CAP_FACTOR * 8 + (size_t)q * 4 + (size_t)plan.P * 2 * q * 4 +
         (size_t)q * 4096 * 4 + (size_t)plan.P * 2 * q * 8 + 8192;
}

cudaError_t launch_gemm(const GemmArgs &a, const GemmPlan &plan, void *scratch, cudaStream_t s, int *launches) {
  const int64_t xcap = a.ids ? a.xsel_cap : 0;
  // CTA pairs (cta_group::2) halve the L2->SM row traffic per query but add pair
  // synchronisation; measured slower while the single-CTA pass is MMA-bound, so opt-in
  static const bool use_pair = getenv("VRS_PAIR") != nullptr;
  const int bn_rows = (plan.qtiles >= 2 && use_pair) ? tc::BN / 2 : tc::BN;   // a pair stages half a row tile per CTA
  CUtensorMap mq, mx, mg;
  if (!make_map(&mq, a.Q, a.q, a.d, tc::BM) || !make_map(&mx, a.X, a.n, a.d, bn_rows) ||
      !make_map(&mg, xcap > 0 ? a.xsel : a.X, xcap > 0 ? xcap : a.n, a.d, bn_rows))
    return cudaErrorInvalidValue;
  TcParams p;
  p.n_rows = a.n;
  p.d = a.d;
  p.nk = (a.d + tc::BK - 1) / tc::BK;
  p.q = a.q;
  p.qtiles = plan.qtiles;
  p.P = plan.P;
  p.row_tiles_max = (a.n + tc::BN - 1) / tc::BN;
  p.ids = a.ids;
  p.count = a.count;
  p.allow_gather = a.masked == 1 ? 0 : (a.masked == 2 ? 2 : 1);
  p.X = a.X;
  p.xsel_cap = xcap;
  p.bitmap = a.bitmap;
  p.nx2 = a.nx2;
  p.inv_nx = a.inv_nx;
  p.metric = a.metric;
  p.kp = kp_of(a.kprime);
  p.cap = p.kp * tc::CAP_FACTOR;
  p.cand_key = static_cast<float *>(scratch);
  p.cand_id = reinterpret_cast<int32_t *>(p.cand_key + (size_t)plan.P * 2 * a.q * p.cap);
  p.gtau = reinterpret_cast<uint32_t *>(p.cand_id + (size_t)plan.P * 2 * a.q * p.cap);
  p.list_tau = reinterpret_cast<float *>(p.gtau + ((a.q + 63) / 64) * 64);
  p.dense_buf = p.list_tau + (((size_t)plan.P * 2 * a.q + 63) / 64) * 64;
  p.cnt_state = reinterpret_cast<int32_t *>(p.dense_buf + (size_t)a.q * 4096);
  p.tau_state = reinterpret_cast<float *>(p.cnt_state + (((size_t)plan.P * 2 * a.q + 63) / 64) * 64);
  p.part = 0;
  {
    cudaError_t e = cudaMemsetAsync(p.gtau, 0, (size_t)a.q * 4, s);
    if (e != cudaSuccess) return e;
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaSuccess;
    for (auto fn : {tc_topk_kernel<true, 1>, tc_topk_kernel<false, 1>, tc_topk_kernel<true, 2>, tc_topk_kernel<false, 2>})
      if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (xcap > 0 && p.allow_gather) {
    gather_copy_kernel<<<4 * 148, 256, 0, s>>>(a.X, a.d, a.ids, a.count, a.n, p.allow_gather, xcap, a.xsel);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (launches) *launches += 1;
  }
  static unsigned long long *stats = nullptr;
  static const bool want_stats = getenv("VRS_STATS") != nullptr;
  if (want_stats && !stats) cudaMalloc(&stats, 64);
  p.stats = want_stats ? stats : nullptr;
  if (want_stats) cudaMemsetAsync(stats, 0, 64, s);
  static const bool no_ar = getenv("VRS_NO_AR") != nullptr;
  static const bool epi_skip = getenv("VRS_EPI_SKIP") != nullptr;
  p.epi_skip = epi_skip ? 1 : 0;
  const bool ar = p.nk <= 4 && !no_ar;
  const int cg = bn_rows == tc::BN / 2 ? 2 : 1;
  auto kern = cg == 2 ? (ar ? tc_topk_kernel<true, 2> : tc_topk_kernel<false, 2>)
                      : (ar ? tc_topk_kernel<true, 1> : tc_topk_kernel<false, 1>);
  // grid: (splits x query groups) work items, CG CTAs each (cluster of 2 for pairs)
  const int qgroups = (plan.qtiles + cg - 1) / cg;
  auto launch = [&](int splits, const TcParams &pr) -> cudaError_t {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(splits * qgroups * cg));
    cfg.blockDim = dim3(tc::THREADS);
    cfg.dynamicSmemBytes = tc::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cg;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (want_stats) cudaMemsetAsync(stats, 0, 64, s);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mq, mx, mg, pr);
    if (want_stats) {
      unsigned long long h[4];
      cudaMemcpyAsync(h, stats, 32, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      fprintf(stderr, "[vrs stats] part=%d dense=%d grid=%d chunks=%llu slow=%llu (%.3f) lane0-accepts=%llu compactions=%llu\n",
              pr.part, pr.dense ? 1 : 0, (int)cfg.gridDim.x, h[0], h[1], h[0] ? (double)h[1] / h[0] : 0.0, h[2], h[3]);
    }
    return e;
  };
  // sample pass: raw keys of the first SAMPLE_TILES row tiles for every query ->
  // per-query kp-th best -> initial shared threshold (no per-item warm-up)
  constexpr int SAMPLE_TILES = 4096 / tc::BN;   // 4096 sampled rows
  p.dense = nullptr;
  p.ldd = 0;
  p.dense_tiles = 0;
  p.tile_step = 1;
  static const bool no_sample = getenv("VRS_NO_SAMPLE") != nullptr;
  static const bool no_probe = getenv("VRS_NO_PROBE") != nullptr;
  if (p.row_tiles_max >= 8 && !no_sample) {
    TcParams ps = p;
    ps.P = std::max(1, std::min(SAMPLE_TILES, 148 / (qgroups * cg)));
    ps.dense = p.dense_buf;
    ps.ldd = SAMPLE_TILES * tc::BN;
    ps.dense_tiles = SAMPLE_TILES;
    cudaError_t e = cudaMemsetAsync(ps.dense, 0xff, (size_t)a.q * ps.ldd * 4, s);   // NaN fill = no row
    if (e != cudaSuccess) return e;
    e = launch(ps.P, ps);
    if (e != cudaSuccess) return e;
    SampleArgs sa{ps.dense, ps.ldd, a.q, p.kp, p.gtau};
    e = launch_sample_threshold(sa, s);
    if (e != cudaSuccess) return e;
    if (launches) *launches += 2;
  }
  // Threshold refinement before the main pass (masked full tiles only; the kernel
  // switches the probe off on gathered selections):
  //  default: probe pass over every PROBE_STEP-th row tile -> per-query kp-th best
  //  VRS_TWO_PART=1: main pass split 1/8 + 7/8 with a refinement over every list in between
  p.tile_step = 1;
  p.part = 0;
  static const bool two_part_env = getenv("VRS_TWO_PART") != nullptr;
  constexpr int PROBE_STEP = 16;
  if (two_part_env && p.row_tiles_max / plan.P >= 16) {
    p.part = 1;
    cudaError_t e = launch(plan.P, p);
    if (e != cudaSuccess) return e;
    RefineArgs ra{p.cand_key, p.cand_id, p.cnt_state, plan.P * 2, p.cap, a.q, p.kp, p.gtau};
    e = launch_refine_threshold(ra, s);
    if (e != cudaSuccess) return e;
    p.part = 2;
    if (launches) *launches += 2;
  } else if (p.row_tiles_max / plan.P >= 8 && !no_probe) {
    // each probe list keeps only its best kp/4 (>= 8): the union over all lists
    // still holds >= kp entries, so its kp-th best remains a valid lower bound
    TcParams pp = p;
    pp.tile_step = PROBE_STEP;
    pp.kp = std::max(8, p.kp / 4);
    pp.cap = std::max(pp.kp * tc::CAP_FACTOR, pp.kp + 96);   // room for >= 96 appends between compactions
    cudaError_t e = launch(plan.P, pp);
    if (e != cudaSuccess) return e;
    ProbeArgs pa{pp.cand_key, pp.cand_id, plan.P * 2, pp.cap, pp.kp, a.q, p.kp, p.gtau};
    e = launch_probe_threshold(pa, s);
    if (e != cudaSuccess) return e;
    if (launches) *launches += 2;
  }
  {
    cudaError_t el = launch(plan.P, p);
    if (el != cudaSuccess) return el;
  }
  if (launches) *launches += 1;
  return cudaGetLastError();
}

// Where the finalize pass reads the GEMM candidate lists.
void gemm_lists(const GemmArgs &a, const GemmPlan &plan, void *scratch, const float **key, const int32_t **id,
                int32_t *stride, int32_t *kread, int32_t *nlists, const float **list_tau) {
  *nlists = plan.P * 2;
  const int kp = kp_of(a.kprime);
  const int cap = kp * tc::CAP_FACTOR;
  *key = static_cast<const float *>(scratch);
  *id = reinterpret_cast<const int32_t *>(static_cast<const float *>(scratch) + (size_t)plan.P * 2 * a.q * cap);
  *stride = cap;
  *kread = kp;
  const uint32_t *gt = reinterpret_cast<const uint32_t *>(*id + (size_t)plan.P * 2 * a.q * cap);
  *list_tau = reinterpret_cast<const float *>(gt + ((a.q + 63) / 64) * 64);
}

}  // namespace vrs
