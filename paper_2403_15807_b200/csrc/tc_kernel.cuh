// tc_kernel.cuh -- the tcgen05 tensor-core pass (kernel template shared by
// gemm_tc.cu: top-k probe / main modes, and gemm_range.cu: range count / fill
// modes).  See gemm_tc.cu for the design notes.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "vrs_kernels.cuh"

namespace vrs {

namespace tc {
constexpr int BM = 128;         // queries per tile (TMEM lanes)
#ifndef VRS_BN
#define VRS_BN 256
#endif
constexpr int BN = VRS_BN;      // rows per tile (TMEM columns, MMA N)
constexpr int BK = 32;          // fp32 per K block = 128 bytes = one swizzle span (bf16: 64)
constexpr int PIPE_BYTES = 192 * 1024;   // shared-memory pipeline region (A resident and/or stages)
constexpr int MAX_STAGES = 8;
constexpr int A_BYTES = BM * BK * 4;   // 16 KB
constexpr int B_BYTES = BN * BK * 4;   // 32 KB at BN = 256
constexpr int ACC_STAGES = 512 / BN;   // accumulator tiles in TMEM (all 512 columns)
constexpr int TMEM_COLS = 512;
constexpr int EPI_WARP0 = 4;
constexpr int LPS = kListsPerSplit;   // lists per split = epilogue warps per TMEM lane quadrant
constexpr int EPI_WARPS = 4 * LPS;    // each owns BN / LPS columns of a quadrant's 32 rows (queries)
constexpr int EPI_COLS = BN / LPS;
static_assert(EPI_COLS % 32 == 0, "whole 32-column chunks per epilogue warp");
constexpr int THREADS = (EPI_WARP0 + EPI_WARPS) * 32;
constexpr int CAP_FACTOR = 4;   // candidate buffer = CAP_FACTOR * KP entries per (list, query)
constexpr int BIAS_STAGES = 4;
constexpr int STAGE_COLS = 8;   // per-warp key staging: one private row of 8 fp32 (a group's keys) per lane
constexpr int SLOTS = 32;       // probe: row slots per lane (column index mod 32)
constexpr int PROBE_STEP = 16;  // probe pass: every 16th row tile (8 / 32 for large / small batches)
constexpr int GROUPS = BN / 8;  // 8-column key-bound groups per tile
// dynamic smem: [pipeline region] + bias a/b/id [BIAS_STAGES][BN] + group bounds
// max b / max a / min a [3][BIAS_STAGES][GROUPS] + per-warp key staging (doubles as
// the compaction histogram)
constexpr size_t SMEM_BYTES = 1024 + (size_t)PIPE_BYTES + BIAS_STAGES * BN * 12 + 3 * BIAS_STAGES * GROUPS * 4 +
                              EPI_WARPS * 32 * STAGE_COLS * 4 + 256;
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
// Four rows (r0..r3) of one 128-byte K block into consecutive 128-byte smem rows
// (swizzled like a 4-row box): the late-materialisation load of gathered rows.
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int r0, int r1,
                                            int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}
// cp.async of 16 bytes (zero-filled when !valid) and an mbarrier arrival that fires
// when all of this thread's earlier cp.async have landed (pending count +1 now,
// -1 on completion: the barrier's expected count is unchanged)
__device__ __forceinline__ void cpa16(uint32_t dst, const void *src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cpa_mbar_arrive(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// ---- CTA pair (cta_group::2): cluster of two CTAs on one TPC --------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(const void *p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  // (default semantics, release at CTA scope, as CUTLASS's ClusterBarrier::arrive: a
  // .release.cluster arrival compiles to a GPU-scope MEMBAR per call -- measured: the pair's
  // main pass at 33 % tensor-pipe activity, membar / long-scoreboard stalls)
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA load into this CTA's shared memory whose completion (bytes) is counted on the
// barrier at cluster address `bar` -- the pair leader's stage barrier
__device__ __forceinline__ void tma_load_2d_pair(void *dst, const CUtensorMap *map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
// commit of the pair's MMAs: arrives on the barrier at this offset in both CTAs
__device__ __forceinline__ void tc_commit_pair(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"((uint16_t)3)
               : "memory");
}
// D[tmem of both CTAs] (+)= A[smem, 128 rows per CTA] . B[smem, N / 2 rows per CTA]^T, M = 256
__device__ __forceinline__ void tc_mma_f16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// three-input maximum (sm_100: one FMNMX3); NaN-free inputs (raw fp32 dot products)
__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
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

// D[tmem] (+)= A[smem] . B[smem]^T, kind::f16 (fp16 or bf16 inputs per idesc, fp32 accumulate), both K-major.
__device__ __forceinline__ void tc_mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
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

// The same with stride byte offset 0: every 8-row group of the operand reads the same
// 8 rows (AR8: a query tile of <= 8 queries held as 8 rows per K block; accumulator rows
// 8..127 repeat rows 0..7 and belong to no query)
__device__ __forceinline__ uint64_t sw128_desc_rows8(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor: D fp32, A/B format ab (kind::f16: 0 fp16, 1 bf16;
// kind::tf32: 2 tf32), both K-major, N = BN, M = BM.
__host__ __device__ constexpr uint32_t mma_idesc(int M, int N, uint32_t ab) {
  return (1u << 4) | (ab << 7) | (ab << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
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

#define TMEM_LD_32x32b_X64(taddr, r)                                                                              \
  asm volatile(                                                                                                   \
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19," \
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,"   \
      "%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"                            \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),  \
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),      \
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),     \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]),     \
        "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]),     \
        "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),     \
        "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]),     \
        "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])                  \
      : "r"(taddr))

// Wait for this thread's outstanding tcgen05.ld; the registers are tied to the
// wait so no use of them can be scheduled above it.
#define TMEM_LD_WAIT(r)                                                                                           \
  asm volatile("tcgen05.wait::ld.sync.aligned;"                                                                   \
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),   \
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),            \
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),          \
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),          \
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])                                                             \
               :                                                                                                  \
               : "memory")

// ---------------------------------------------------------------- kernel
struct TcParams {
  int64_t n_rows;          // rows of the index (identity / masked row space)
  const int32_t *ids;      // compacted ascending selection (nullptr: no predicate)
  const int64_t *count;    // device count of ids
  int32_t allow_gather;    // 0 never, 1 selectivity switch on the device, 2 forced
  int32_t d;
  int32_t nk;              // K blocks = ceil(d / 32)
  int64_t q;
  int32_t qtiles;
  int32_t P;               // splits
  int32_t tile_step;       // 1: every tile; PROBE_STEP: probe pass
  int32_t probe_div;       // probe: > 0 => step = clamp(main span / probe_div, 2, tile_step) (device-side span)
  int32_t probe_rows;      // probe with rows by cp.async: > 0 => only the first probe_rows (a multiple of 8) rows of
                           // each probed tile are fetched and scored (the others: zero-filled, masked) -- a
                           // one-tile-per-CTA probe lasts as long as one SM needs to fetch the tile
  int32_t P_main, min_p_main;   // probe: the main pass's splits (its span sets the density); 0 = P
  int32_t g4;              // gather mode: 1 = TMA gather4 from X by id (tmap_g), 2 = cp.async from X by id
                           // (xrows), 0 = TMA tiles from the X_sel copy
  const void *xrows;       // g4 == 2: the rows' base (fp32 corpus or its 16-bit shadow), row_bytes each
  int32_t row_bytes;
  int64_t cp_min_bytes;    // g4 == 2: cp.async only when the selection holds >= this many row bytes ...
  int64_t cp_min_rows;     // ... or >= this many rows (cp_fetch)
                           // (below it gather_copy_kernel made X_sel and TMA tiles stream it)
  int32_t min_span;        // used splits span >= this many row tiles (splits_used) ...
  int32_t min_p;           // ... unless that leaves fewer than min_p splits
  const uint32_t *bitmap;  // nullptr => every row qualifies
  const float *nx2;
  const float *inv_nx;
  int32_t metric;
  int32_t kp;              // entries kept by a compaction (pow2 >= k')
  int32_t cap;             // buffer capacity per (list, query)
  float *cand_key;         // [2P][q][cap]
  int32_t *cand_id;
  int32_t *cand_cnt;       // [2P][q] entries per list (MAIN, RCOUNT)
  const int64_t *coff;     // RFILL: [q][2P] start of each (query, list) segment in cand_id
  float *probe_max;        // [q][2P][SLOTS] probe slot maxima
  int64_t xsel_cap;        // rows of the materialised-selection buffer
  const float *xsel_norm;  // [xsel_cap] the gathered rows' norm term (L2 |x|^2, COS 1/|x|)
  uint32_t *gtau;          // [q] ordered-u32 threshold shared by all lists of a query (0 = none)
  unsigned long long *stats;  // optional counters: chunks, slow chunks, appends, compactions
  uint32_t idesc;          // MMA instruction descriptor (operand format)
  const int32_t *qexp;     // 16-bit operands: [q] per-query exponents e_q (nullptr: TF32, no scaling)
  int32_t xexp;            // the shadow's exponent e_x
  // refine pass: K runs over nseg = 3 segments -- q_hi.x_hi, q_hi.x_lo (x_lo
  // through tmap_gl gathered / tmap_xl masked / xrows_lo by id), q_lo.x_hi (q_lo at column
  // a_lo_off of the query map); the grid folds onto the *qcount compacted queries' tiles
  int32_t nseg = 1;
  int32_t a_lo_off = 0;
  const int32_t *qcount = nullptr;
  const void *xrows_lo = nullptr;   // cp.async gather, segment 1: x_lo's base
  int32_t no_helpers = 0;           // (A/B, VRS_NO_HELPERS) no helper producer warps
};

// Warp-cooperative compaction of one lane's candidate buffer to its best KP
// entries (key desc, then buffer order = ascending row id).  Returns the new
// threshold key (the KP-th best).  All 32 lanes call it with the same `owner`.
static __device__ __noinline__ float compact_lane(float *key, int32_t *id, int cnt, int kp, uint32_t *hist) {
  const int lane = threadIdx.x & 31;
  uint32_t prefix = 0, mask = 0;
  int rem = kp;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = lane; b < 256; b += 32) hist[b] = 0;
    __syncwarp();
    for (int i0 = 0; i0 < cnt; i0 += 32) {
      const int i = i0 + lane;
      const uint32_t ok = i < cnt ? ordered_u32(key[i]) : 0u;
      hist_add_warp(hist, (i < cnt && (ok & mask) == prefix) ? (ok >> shift) & 255u : 256u);
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

constexpr int MODE_MAIN = 0;    // fused top-k candidates
constexpr int MODE_PROBE = 1;   // slot maxima for the threshold
constexpr int MODE_RCOUNT = 2;  // range search: count keys >= the query's threshold per list
constexpr int MODE_RFILL = 3;   // range search: write those rows' ids to the list's segment

// AR: the query tile stays resident in shared memory (d <= 128).
// MODE: MAIN (fused top-k candidates) or PROBE (slot maxima for the threshold).
// ROWSCALE: per-row key scale (COSINE 1/|x|); otherwise a constant (L2: 2, IP: 1).
// BF: operands are bf16 (shadow corpus, kind::f16) instead of fp32 (kind::tf32).
#define TC_TL(slot) TL_STAMP(MODE & 3, slot)   // (thread-0-only stamps are filtered in TL_STAMP)
// PAIR: a cluster of two CTAs -- query tiles 2i and 2i + 1 of one row split -- runs
// each tile's MMA as one cta_group::2 M = 256 MMA: each CTA stages its own 128 queries
// and half (128) of the tile's rows, so every row is fetched once per query-tile pair
// (the one-query-tile-per-CTA kernel fetches it per query tile); the leader (rank 0)
// issues the MMAs, the accumulator (128 queries x 256 rows) lands in each CTA's TMEM
// and each CTA's epilogue is unchanged.  MODE_MAIN, 16-bit operands, streamed A only.
// ARM: 0 the query tile streams with every stage; 1 (AR) it stays resident, 16 KB per K
// block (nk <= 4); 2 (AR8) it stays resident as 8 rows per K block, 1 KB each (<= 8
// queries, nk <= 32), read by the MMA with stride 0 -- the stages hold rows only, so a
// small batch keeps 5 stages of rows in flight instead of 4 (A and B) per SM.
template <int ARM, int MODE, bool ROWSCALE, bool BF, bool PAIR>
__global__ void __launch_bounds__(tc::THREADS, 1)
    tc_topk_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_x,
                   const __grid_constant__ CUtensorMap tmap_g, const __grid_constant__ CUtensorMap tmap_xl,
                   const __grid_constant__ CUtensorMap tmap_gl, TcParams p) {
  using namespace tc;
  constexpr bool AR = ARM != 0;
  constexpr int ABLK = ARM == 2 ? 1024 : A_BYTES;           // resident bytes per K block
  constexpr int ARES = ARM == 2 ? 32 * 1024 : 4 * A_BYTES;  // resident query region
  static_assert(!PAIR || (MODE == MODE_MAIN && !AR && BF), "CTA pairs: main pass, streamed 16-bit A");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment (128B swizzle atoms) by pointer arithmetic on the shared
  // array itself, so the compiler keeps the shared address space (LDS, not LD)
  uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // pipeline region: AR ? [A: nk x 16 KB][B stages of 32 KB] : [stages of (A 16 KB | B 32 KB)]
  constexpr int BROWS = PAIR ? BN / 2 : BN;               // rows of a tile this CTA stages
  constexpr int BSTAGE = BROWS * BK * 4;                    // their bytes per K block
  constexpr int SSTRIDE = AR ? B_BYTES : A_BYTES + BSTAGE;   // bytes per pipeline stage
  constexpr int NST = ((PIPE_BYTES - (AR ? ARES : 0)) / SSTRIDE) < MAX_STAGES
                          ? ((PIPE_BYTES - (AR ? ARES : 0)) / SSTRIDE)
                          : MAX_STAGES;
  constexpr int BOFF = AR ? 0 : A_BYTES;                 // B offset within a stage
  constexpr int KE = BF ? 2 * BK : BK;                   // elements per 128-byte K block
  uint8_t *a_res = smem;                                 // AR: resident query tile
  uint8_t *b_base = AR ? smem + ARES : smem;
  float *bias_a = reinterpret_cast<float *>(smem + PIPE_BYTES);               // [BIAS_STAGES][BN]
  float *bias_b = bias_a + BIAS_STAGES * BN;                                    // [BIAS_STAGES][BN]
  int32_t *row_id = reinterpret_cast<int32_t *>(bias_b + BIAS_STAGES * BN);     // [BIAS_STAGES][BN]
  // per 8-row group: max b, max a, min a over its rows (the group's key upper bound)
  float *g_bmax = reinterpret_cast<float *>(row_id + BIAS_STAGES * BN);        // [BIAS_STAGES][GROUPS]
  float *g_amax = g_bmax + BIAS_STAGES * GROUPS;
  float *g_amin = g_amax + BIAS_STAGES * GROUPS;
  float *kstage = g_amin + BIAS_STAGES * GROUPS;                                // [EPI_WARPS][32][STAGE_COLS]

  __shared__ __align__(8) uint64_t full_bar[MAX_STAGES], empty_bar[MAX_STAGES];
  __shared__ __align__(8) uint64_t tfull_bar[ACC_STAGES], tempty_bar[ACC_STAGES];
  __shared__ __align__(8) uint64_t bfull_bar[BIAS_STAGES], bempty_bar[BIAS_STAGES];
  __shared__ __align__(8) uint64_t afull_bar;
  __shared__ uint32_t tmem_base_s;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int qtile = blockIdx.x % p.qtiles;
  int split = blockIdx.x / p.qtiles;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0u;   // (PAIR: qtile & 1)
  const bool leader = rank == 0;
  // Helper producers: the epilogue warps of TMEM lane quadrants that hold no query of this
  // tile (a batch of <= 96 queries) skip the epilogue; with cp.async row delivery they fetch
  // rows beside warps 0 and 3 -- each warp keeps ~55 loads in flight, so two producer warps
  // capped the by-id fetch near 40 GB/s per SM.  (Not in pairs / the refine / range passes.)
  const int64_t q_tile = p.q - (int64_t)qtile * BM;   // queries of this tile (<= BM when not the last)
  const int act_quads = (int)(((q_tile < BM ? q_tile : (int64_t)BM) + 31) / 32);
  const bool hp_ok = !PAIR && p.qcount == nullptr && (MODE == MODE_MAIN || MODE == MODE_PROBE) && act_quads >= 1 &&
                     act_quads < 4 && !p.no_helpers;
  const int epi_arrivals = hp_ok ? LPS * act_quads : EPI_WARPS;   // epilogue warps releasing a tile
  const bool helper = hp_ok && warp >= EPI_WARP0 && (warp & 3) >= act_quads;
  if (threadIdx.x == 0) TC_TL(0);
  if (threadIdx.x == 0) {
    // (PAIR: the leader's stage barrier also counts the peer's relay, its accumulator-empty
    // barrier both CTAs' epilogue warps)
    for (int s = 0; s < NST; ++s) { mbar_init(&full_bar[s], PAIR && leader ? 2 : 1); mbar_init(&empty_bar[s], 1); }
    mbar_init(&afull_bar, 1);
    for (int s = 0; s < ACC_STAGES; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], PAIR && leader ? 2 * EPI_WARPS : epi_arrivals);
    }
    for (int s = 0; s < BIAS_STAGES; ++s) {
      mbar_init(&bfull_bar[s], 32);
      mbar_init(&bempty_bar[s], epi_arrivals);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_q);
    prefetch_tmap(&tmap_x);
    prefetch_tmap(&tmap_g);
    if (p.nseg > 1) { prefetch_tmap(&tmap_xl); prefetch_tmap(&tmap_gl); }
  }
  if (warp == 1) {
    if (PAIR) {
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
  __syncthreads();
  if (PAIR) cluster_sync_all();   // both CTAs' barriers initialised and TMEM allocated
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;
  // (the prologue above overlaps the predecessor kernel's tail; global memory from here on)
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) TC_TL(1);
  // the refine pass (qcount: its compacted query count, on the device): the grid folds
  // onto the active query tiles, P F row splits per tile (refine_fold); split s writes
  // list split s mod P at list rows (s / P) Qa + query
  int64_t P_rows = p.P, lrow = 0;
  int lsplit = split;
  bool q_idle = false, fold_out = false;
  if (p.qcount != nullptr) {
    const int64_t qc = __ldg(p.qcount);
    const RefineFold rf = refine_fold(qc, p.qtiles, p.q);
    qtile = blockIdx.x % rf.tiles;
    split = blockIdx.x / rf.tiles;
    P_rows = (int64_t)p.P * rf.F;
    fold_out = split >= P_rows;
    lsplit = split % p.P;
    lrow = (int64_t)(split / p.P) * rf.Qa;
    q_idle = qc == 0 || fold_out;
  }
  // Selectivity-driven row delivery (decided on the device, no host sync):
  //  gather: the selection was materialised densely (gather_copy_kernel, late
  //          materialization) and streams by TMA from X_sel; ids map rows back
  //  masked: every row streams by TMA, unqualified rows are masked by the bitmap
  const int64_t n_sel = p.ids ? *p.count : p.n_rows;
  const bool gather = gather_mode(p.ids, p.allow_gather, n_sel, p.xsel_cap);
  // rows fetched by cp.async (see the producer): large one-query-tile selections, where
  // the X_sel copy's extra pass costs more than cp.async's lower streaming rate
  const bool cpg = gather && p.g4 == 2 && cp_fetch(n_sel, p.row_bytes, p.cp_min_bytes, p.cp_min_rows);
  const bool direct = cpg || (gather && p.g4 == 1);   // rows by id from X (no X_sel)
  const int prow_lim = cpg && p.probe_rows > 0 ? p.probe_rows : BN;   // rows of a tile that count (probe_rows)
  const int64_t n_space = gather ? n_sel : p.n_rows;
  const int64_t row_tiles = (n_space + BN - 1) / BN;
  // splits actually used (splits_used): >= 4 row tiles per item when the
  // (device-side) row space allows; CTAs of unused splits publish empty lists
  const int64_t p_eff = used_splits(row_tiles, P_rows, p.min_span, p.min_p);
  const int64_t t_begin = split < p_eff ? (row_tiles * split) / p_eff : 0;
  const int64_t t_end = split < p_eff ? (row_tiles * (split + 1)) / p_eff : 0;
  const int64_t span = t_end - t_begin;
  // probe: every step-th tile of the item (the first tile of a shorter item).  With
  // probe_div, short items (small selections) probe densely: their main pass is
  // slow-path bound, so a tighter threshold pays more than the denser probe costs
  int64_t step_cap = p.tile_step;
  if (p.probe_div > 0) {   // density from the main pass's span (the probe may use fewer, longer splits)
    const int64_t main_span = p.P_main > 0 ? row_tiles / used_splits(row_tiles, p.P_main, p.min_span, p.min_p_main) : span;
    step_cap = std::min<int64_t>(step_cap, std::max<int64_t>(2, main_span / p.probe_div));
  }
  const int step = MODE == MODE_PROBE ? (int)std::min<int64_t>(step_cap, std::max<int64_t>(1, span)) : 1;
  const int ntiles = q_idle ? 0 : (int)((span + step - 1) / step);
  const int nkb = p.nk * p.nseg;   // K blocks per tile (3 segments in the refine pass)
  auto tile_of = [&](int t) -> int64_t { return t_begin + (int64_t)t * step; };


  // cp.async producer warps: warps 0 and 3, plus (helpers, above) 2 or 6 epilogue warps of
  // query-less TMEM quadrants -- 2, 4 or 8 warps, each fetching a contiguous share of the
  // tile's rows.  Two warps: C4 s = 50 % Q = 1 2.06 -> 1.89 ms (r02_cp_warps_ab.txt);
  // the helpers: r02_helpers_ab.txt
  const int n_help = hp_ok ? (act_quads == 1 ? 6 : 2) : 0;
  int hidx = -1;   // helper index (epilogue warps of query-less quadrants, in warp order)
  if (helper) {
    hidx = 0;
    for (int w2 = EPI_WARP0; w2 < warp; ++w2) hidx += (w2 & 3) >= act_quads ? 1 : 0;
    if (hidx >= n_help) hidx = -1;   // (a third / fourth helper when two suffice: idle)
  }
  if ((warp == 0 || warp == 3 || hidx >= 0) && cpg) {
    // ------------------------------------------------ cp.async producers, gathered rows
    // (late materialisation without a copy: NPW warps each fetch a contiguous share of the
    // tile's rows straight from X by id -- each row's 128-byte K-block segment as 8 x 16 B,
    // placed in the 128B-swizzled layout the MMA descriptors expect (what a TMA box load
    // would write); the stage's barrier completes when every lane's copies land: each lane's
    // cp.async.mbarrier.arrive adds a pending arrival that its copies retire, and warp 0's
    // lane 0 arrives only after every producer warp registered its own)
    const bool lead = warp == 0;
    const int pidx = warp == 0 ? 0 : (warp == 3 ? 1 : 2 + hidx);
    auto produce = [&](auto npw_c) {
      constexpr int NPW = decltype(npw_c)::value;
      const int hrow = pidx * (BROWS / NPW);   // this warp's first row of the CTA's rows of the tile
      int stage = 0;
      uint32_t phase = 0;
      if (lead && AR && ntiles > 0 && lane == 0) {
        mbar_expect_tx(&afull_bar, p.nk * ABLK);
        for (int kb = 0; kb < p.nk; ++kb) tma_load_2d(a_res + kb * ABLK, &tmap_q, &afull_bar, kb * KE, qtile * BM);
      }
      constexpr int GR = BROWS / (32 * NPW);   // rows per lane per warp
      static_assert(GR >= 1, "at least one row per lane");
      const char *xb = static_cast<const char *>(p.xrows);
      const int64_t rb = p.row_bytes;
      const int32_t pad_row = n_sel > 0 ? __ldg(p.ids + n_sel - 1) : 0;
      auto load_ids = [&](int t, int32_t (&r)[GR]) {
#pragma unroll
        for (int u = 0; u < GR; ++u) {
          const int64_t pos = tile_of(t) * BN + rank * BROWS + hrow + lane + 32 * u;
          r[u] = pos < n_sel ? __ldg(p.ids + pos) : pad_row;
        }
      };
      int32_t rid[GR], rnext[GR];
      if (ntiles > 0) load_ids(0, rid);
      for (int t = 0; t < ntiles; ++t) {
        if (t + 1 < ntiles) load_ids(t + 1, rnext);
        for (int kb = 0; kb < nkb; ++kb) {
          const int seg = kb / p.nk, kk = kb - seg * p.nk;   // (refine: 3 segments, x_lo in segment 1)
          const char *xs = seg == 1 ? static_cast<const char *>(p.xrows_lo) : xb;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t *st = b_base + stage * SSTRIDE;
          const uint32_t bdst = smem_u32(st + BOFF);
          const int64_t koff = (int64_t)kk * 128;
          // coalesced: 8 lanes copy one row's 128-byte segment (16 B each), a warp
          // instruction 4 whole rows; the row ids (lane j holds rows j + 32v) by shuffle
          const int c = lane & 7;
          const bool cvalid = koff + c * 16 < rb;
#pragma unroll
          for (int u = 0; u < BROWS / (4 * NPW); ++u) {
            const int rl = 4 * u + (lane >> 3);   // row within this warp's part of the tile
            const int32_t id = __shfl_sync(0xffffffffu, rid[(4 * u) >> 5], rl & 31);   // (rl >> 5 == 4u >> 5)
            const int r = hrow + rl;
            cpa16(bdst + r * 128 + ((c ^ (r & 7)) << 4), xs + (int64_t)id * rb + koff + c * 16,
                  cvalid && rank * BROWS + r < prow_lim);
          }
          cpa_mbar_arrive(&full_bar[stage]);
          asm volatile("bar.sync 1, %0;" ::"n"(32 * NPW) : "memory");   // every producer warp registered its arrivals
          if (lead && lane == 0) {
            if (!AR) {
              mbar_expect_tx(&full_bar[stage], A_BYTES);
              tma_load_2d(st, &tmap_q, &full_bar[stage], (seg == 2 ? p.a_lo_off : 0) + kk * KE, qtile * BM);
            } else {
              mbar_arrive(&full_bar[stage]);
            }
          }
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
#pragma unroll
        for (int u = 0; u < GR; ++u) rid[u] = rnext[u];
      }
    };
    if constexpr (PAIR) {   // (no helpers in pairs: half a tile per CTA)
      produce(std::integral_constant<int, 2>{});
    } else {
      if (n_help == 6) produce(std::integral_constant<int, 8>{});
      else if (n_help == 2) produce(std::integral_constant<int, 4>{});
      else produce(std::integral_constant<int, 2>{});
    }
  } else if (warp == 0 && gather && p.g4 == 1) {
    // ------------------------------------------------ TMA producer, gathered rows
    // (late materialisation without a copy: each lane loads the ids of its 8 rows
    // of the tile one tile ahead and issues BN / 128 gather4 per K block)
    int stage = 0;
    uint32_t phase = 0;
    if (AR && ntiles > 0 && lane == 0) {
      mbar_expect_tx(&afull_bar, p.nk * ABLK);
      for (int kb = 0; kb < p.nk; ++kb) tma_load_2d(a_res + kb * ABLK, &tmap_q, &afull_bar, kb * KE, qtile * BM);
    }
    constexpr int GR = BN / 32;   // rows per lane (whole gather4 groups)
    static_assert(GR % 4 == 0, "gather4 groups per lane");
    const int32_t pad_row = n_sel > 0 ? __ldg(p.ids + n_sel - 1) : 0;   // tail rows: any valid row (masked)
    auto load_ids = [&](int t, int32_t (&r)[GR]) {
      const int64_t pos0 = tile_of(t) * BN + lane * GR;
      if (pos0 + GR <= n_sel) {
#pragma unroll
        for (int v = 0; v < GR / 4; ++v) {
          const int4 a0 = __ldg(reinterpret_cast<const int4 *>(p.ids + pos0) + v);
          r[4 * v] = a0.x; r[4 * v + 1] = a0.y; r[4 * v + 2] = a0.z; r[4 * v + 3] = a0.w;
        }
      } else {
#pragma unroll
        for (int u = 0; u < GR; ++u) r[u] = pos0 + u < n_sel ? __ldg(p.ids + pos0 + u) : pad_row;
      }
    };
    int32_t rid[GR], rnext[GR];
    if (ntiles > 0) load_ids(0, rid);
    for (int t = 0; t < ntiles; ++t) {
      if (t + 1 < ntiles) load_ids(t + 1, rnext);
      for (int kb = 0; kb < p.nk; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t *st = b_base + stage * SSTRIDE;
        if (lane == 0) {
          mbar_expect_tx(&full_bar[stage], AR ? B_BYTES : A_BYTES + B_BYTES);
          if (!AR) tma_load_2d(st, &tmap_q, &full_bar[stage], kb * KE, qtile * BM);
        }
        __syncwarp();
        uint8_t *dst = st + BOFF + lane * GR * 128;
#pragma unroll
        for (int v = 0; v < GR / 4; ++v)
          tma_gather4(dst + v * 4 * 128, &tmap_g, &full_bar[stage], kb * KE, rid[4 * v], rid[4 * v + 1],
                      rid[4 * v + 2], rid[4 * v + 3]);
        if (++stage == NST) { stage = 0; phase ^= 1; }
      }
#pragma unroll
      for (int u = 0; u < GR; ++u) rid[u] = rnext[u];
    }
  } else if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      if (AR && ntiles > 0) {
        mbar_expect_tx(&afull_bar, p.nk * ABLK);
        for (int kb = 0; kb < p.nk; ++kb) tma_load_2d(a_res + kb * ABLK, &tmap_q, &afull_bar, kb * KE, qtile * BM);
      }
      for (int t = 0; t < ntiles; ++t) {
        const int row0 = (int)(tile_of(t) * BN);
        for (int kb = 0; kb < nkb; ++kb) {
          const int seg = kb / p.nk, kk = kb - seg * p.nk;   // (refine: 3 segments; else seg = 0)
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t *st = b_base + stage * SSTRIDE;
          // (refine: x_lo in segment 1 -- gathered into its own X_sel copy, or masked over the full x_lo)
          const CUtensorMap *bmap = seg == 1 ? (gather ? &tmap_gl : &tmap_xl) : (gather ? &tmap_g : &tmap_x);
          if (PAIR) {   // both CTAs' loads complete on the leader's barrier; the peer adds one arrival
            const uint32_t lbar = mapa_rank(&full_bar[stage], 0);
            if (leader) mbar_expect_tx(&full_bar[stage], 2 * (A_BYTES + BSTAGE));
            tma_load_2d_pair(st, &tmap_q, lbar, kk * KE, qtile * BM);
            tma_load_2d_pair(st + BOFF, bmap, lbar, kk * KE, row0 + (int)rank * BROWS);   // (box BN / 2)
            if (!leader) mbar_arrive_cluster(lbar);
          } else {
            mbar_expect_tx(&full_bar[stage], AR ? B_BYTES : A_BYTES + BSTAGE);
            if (!AR) tma_load_2d(st, &tmap_q, &full_bar[stage], (seg == 2 ? p.a_lo_off : 0) + kk * KE, qtile * BM);
            tma_load_2d(st + BOFF, bmap, &full_bar[stage], kk * KE, row0);
          }
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && PAIR && !leader && cpg) {
    // ------------------------------------------------ the pair's peer: stage relay
    // (cp.async rows: this CTA's half of a stage has landed -- A by TMA, rows by cp.async -- ->
    // one arrival on the leader's barrier of that stage; the generic-proxy cp.async
    // writes are fenced to the async proxy first, as the leader's MMA warp does for its own)
    int stage = 0;
    uint32_t phase = 0;
    for (int t = 0; t < ntiles; ++t) {
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        if (cpg) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_rank(&full_bar[stage], 0));
        if (++stage == NST) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1 && (!PAIR || leader)) {
    // ------------------------------------------------ MMA issuer
    const uint32_t idesc = p.idesc;
    int stage = 0;
    uint32_t phase = 0;
    if (AR && ntiles > 0) mbar_wait(&afull_bar, 0);
    for (int t = 0; t < ntiles; ++t) {
      const int acc = t % ACC_STAGES;
      const uint32_t acc_phase = (t / ACC_STAGES) & 1;
      if (PAIR) mbar_wait_cluster(&tempty_bar[acc], acc_phase ^ 1);   // (both CTAs' epilogues)
      else mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < nkb; ++kb) {
        if (PAIR) mbar_wait_cluster(&full_bar[stage], phase);   // (own half + the peer's relay)
        else mbar_wait(&full_bar[stage], phase);
        if (t == 0 && kb == 0 && lane == 0) TL_STAMP_ANY(MODE & 3, 2);
        if (cpg) fence_proxy_async_smem();   // cp.async (generic proxy) writes -> the MMA's async-proxy reads
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sb = smem_u32(b_base + stage * SSTRIDE + BOFF);
          const uint32_t sa = AR ? smem_u32(a_res + kb * ABLK) : sb - A_BYTES;
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // K = 8 tf32 / 16 bf16 = 32 bytes per instruction
            const uint64_t da = ARM == 2 ? sw128_desc_rows8(sa + k * 32) : sw128_desc(sa + k * 32);
            if (PAIR) tc_mma_f16_pair(d_tmem, da, sw128_desc(sb + k * 32), idesc, (kb | k) != 0);
            else if (BF) tc_mma_bf16(d_tmem, da, sw128_desc(sb + k * 32), idesc, (kb | k) != 0);
            else tc_mma_tf32(d_tmem, da, sw128_desc(sb + k * 32), idesc, (kb | k) != 0);
          }
          // frees the smem slot when these MMAs finish; accumulator ready after the last K block
          // (PAIR: in both CTAs)
          if (PAIR) {
            tc_commit_pair(&empty_bar[stage]);
            if (kb == nkb - 1) tc_commit_pair(&tfull_bar[acc]);
          } else {
            tc_commit(&empty_bar[stage]);
            if (kb == nkb - 1) tc_commit(&tfull_bar[acc]);
          }
        }
        __syncwarp();
        if (++stage == NST) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------ per-row epilogue terms
    // Loads for tile t + PF are issued before tile t is written out: the warp is
    // memory-latency bound otherwise (one ~us round trip per tile).
    constexpr int PF = 2;
    // norm terms: L2 |x|^2, COS 1/|x|; the inner product needs none (no loads).  Gathered
    // rows read them contiguously from the gather's norm copy (no dependent load).
    const bool need_norm = p.metric != VRS_IP;
    const float *src_rows = p.metric == VRS_L2 ? p.nx2 : p.inv_nx;   // by row id
    const float *src = gather && !direct ? p.xsel_norm : src_rows;
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
        if (lane * RPL >= prow_lim) {   // (probe_rows: rows past the limit were not fetched)
#pragma unroll
          for (int u = 0; u < RPL; ++u) i8[u] = -1;
        }
        if (need_norm && direct) {   // by row id (dependent loads; the bias warp runs PF tiles ahead)
#pragma unroll
          for (int u = 0; u < RPL; ++u) n8[u] = i8[u] >= 0 ? __ldg(src_rows + i8[u]) : 0.f;
        } else if (need_norm && pos0 + RPL <= n_sel) {
#pragma unroll
          for (int v = 0; v < RPL / 4; ++v) {
            const float4 v0 = __ldg(reinterpret_cast<const float4 *>(src + pos0) + v);
            n8[4 * v] = v0.x; n8[4 * v + 1] = v0.y; n8[4 * v + 2] = v0.z; n8[4 * v + 3] = v0.w;
          }
        } else {
#pragma unroll
          for (int u = 0; u < RPL; ++u) n8[u] = need_norm && pos0 + u < n_sel ? __ldg(src + pos0 + u) : 0.f;
        }
        w = 0xffffffffu;
      } else {
        w = 0xffffffffu;
        if (p.bitmap && pos0 < p.n_rows) w = __ldg(p.bitmap + (pos0 >> 5));
        if (need_norm && pos0 + RPL <= p.n_rows) {
#pragma unroll
          for (int v = 0; v < RPL / 4; ++v) {
            const float4 v0 = __ldg(reinterpret_cast<const float4 *>(src + pos0) + v);
            n8[4 * v] = v0.x; n8[4 * v + 1] = v0.y; n8[4 * v + 2] = v0.z; n8[4 * v + 3] = v0.w;
          }
        } else {
#pragma unroll
          for (int u = 0; u < RPL; ++u) n8[u] = need_norm && pos0 + u < p.n_rows ? __ldg(src + pos0 + u) : 0.f;
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
          if (ROWSCALE)
            reinterpret_cast<float4 *>(bias_a + s * BN + lane * RPL)[v] =
                make_float4(av[4 * v], av[4 * v + 1], av[4 * v + 2], av[4 * v + 3]);
          reinterpret_cast<float4 *>(bias_b + s * BN + lane * RPL)[v] =
              make_float4(bv[4 * v], bv[4 * v + 1], bv[4 * v + 2], bv[4 * v + 3]);
          if (MODE == MODE_MAIN || MODE == MODE_RFILL)
            reinterpret_cast<int4 *>(row_id + s * BN + lane * RPL)[v] =
                make_int4(iv[u][4 * v], iv[u][4 * v + 1], iv[u][4 * v + 2], iv[u][4 * v + 3]);
        }
        // group bounds over 8-row groups (8 / RPL lanes each)
        static_assert(RPL <= 8 && 8 % RPL == 0, "8-row groups of whole lanes");
        // (without a per-row scale the third slot holds min b instead of min a: the
        // probe's raw-dot fast path needs to know that a group's bias is uniformly 0)
        float bmx = bv[0], amx = av[0], amn = ROWSCALE ? av[0] : bv[0];
#pragma unroll
        for (int k = 1; k < RPL; ++k) {
          bmx = fmaxf(bmx, bv[k]);
          amx = fmaxf(amx, av[k]);
          amn = fminf(amn, ROWSCALE ? av[k] : bv[k]);
        }
#pragma unroll
        for (int o = 1; o < 8 / RPL; o <<= 1) {
          bmx = fmaxf(bmx, __shfl_xor_sync(0xffffffffu, bmx, o));
          amx = fmaxf(amx, __shfl_xor_sync(0xffffffffu, amx, o));
          amn = fminf(amn, __shfl_xor_sync(0xffffffffu, amn, o));
        }
        if ((lane & (8 / RPL - 1)) == 0) {
          g_bmax[s * GROUPS + lane / (8 / RPL)] = bmx;
          g_amin[s * GROUPS + lane / (8 / RPL)] = amn;
          if (ROWSCALE) g_amax[s * GROUPS + lane / (8 / RPL)] = amx;
        }
        mbar_arrive(&bfull_bar[s]);
        fetch(t + PF, nv[u], iv[u], wv[u]);
      }
    }
  } else if (warp >= EPI_WARP0 && !helper) {
    // ------------------------------------------------ epilogue
    const int ew = warp - EPI_WARP0;
    const int quad = warp & 3;                     // TMEM lane quadrant this warp may access
    const int half = ew >> 2;                      // which BN / LPS of the tile's columns
    const int m = quad * 32 + lane;                // query row within the tile
    const int64_t qg = (int64_t)qtile * BM + m;    // global query index
    const bool active = qg < p.q && !fold_out;
    const int list = lsplit * LPS + half;          // candidate list index
    // key scale: L2 keys are natural units, 2<q,x> - |x|^2, so the 16-bit pass undoes its
    // power-of-two operand scales 2^(e_q + e_x) here (exact); IP / COS keys stay in the
    // query's scaled domain D = 2^(e_q + e_x) -- the order per query is unchanged, and
    // the threshold, the lists and the finalize compare keys of one query only
    // ("key domain")
    const float sc = p.metric == VRS_L2 ? (p.qexp != nullptr && active ? ldexpf(2.f, -(__ldg(p.qexp + qg) + p.xexp)) : 2.f)
                                        : 1.f;
    const int64_t cbase = MODE == MODE_RFILL ? (active ? p.coff[qg * (LPS * p.P) + list] : 0)
                                             : ((int64_t)list * p.q + (active ? lrow + qg : 0)) * p.cap;
    float *ckey = p.cand_key + (MODE == MODE_RFILL ? 0 : cbase);
    int32_t *cid = p.cand_id + cbase;
    float *wst = kstage + ew * 32 * STAGE_COLS;
    uint32_t *whist = reinterpret_cast<uint32_t *>(wst);   // compaction histogram aliases the staging area
    float thr = active ? -INFINITY : INFINITY;     // accept iff key > thr (inactive lanes never accept)
    int cnt = 0;
    // epilogue counters (VRS_STATS=1 prints them) exist only in builds with
    // -DVRS_TC_STATS: the hot loop carries no runtime debug state otherwise
#ifdef VRS_TC_STATS
#define TC_STAT(x) (x)
#else
#define TC_STAT(x) ((void)0)
#endif
    uint32_t st_chunks = 0, st_slow = 0, st_app = 0, st_comp = 0;
    float smax[SLOTS];
#pragma unroll
    for (int i = 0; i < SLOTS; ++i) smax[i] = -INFINITY;
    // Shared threshold (probe): the k'-th best key over all rows is >= gtau, so
    // keys below it can never be in the result; keys equal to it are kept.
    // (range modes: gtau is the query's key threshold, margin included)
    if (MODE != MODE_PROBE && active) {
      const uint32_t o = __ldcg(p.gtau + qg);
      if (o != 0) {
        const uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
        thr = nextafterf(__uint_as_float(u), -INFINITY);
      }
    }
    // own list: after a compaction to the KP best, a later row (larger id) must
    // beat the KP-th best strictly
    auto compact_needed = [&](int threshold) {
      uint32_t need = __ballot_sync(0xffffffffu, cnt > threshold);
      while (need) {
        const int owner = __ffs(need) - 1;
        need &= need - 1;
        const int oc = __shfl_sync(0xffffffffu, cnt, owner);
        const int64_t ob = ((int64_t)list * p.q + lrow + (int64_t)qtile * BM + quad * 32 + owner) * p.cap;
        const float nt = compact_lane(p.cand_key + ob, p.cand_id + ob, oc, p.kp, whist);
        TC_STAT(++st_comp);
        if (lane == owner) {
          cnt = p.kp;
          thr = fmaxf(thr, nt);
        }
      }
    };
    auto f4 = [](const float4 &v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; };
    // one 32-column chunk: r holds the raw dot products; gb/ga/gn: the chunk's 4
    // group bounds (max b, max a, min a)
    auto chunk = [&](uint32_t (&r)[32], const float *ba, const float *bb, const int32_t *rid, const float *gb,
                     const float *ga, const float *gn) {
      if (MODE == MODE_PROBE) {   // exact keys -> running slot maxima
        if (!ROWSCALE && p.metric == VRS_IP) {
          // inner product with every row of the chunk selected: key = dot exactly
          const float4 bx = *reinterpret_cast<const float4 *>(gb), bn = *reinterpret_cast<const float4 *>(gn);
          if (bx.x == 0.f && bx.y == 0.f && bx.z == 0.f && bx.w == 0.f && bn.x == 0.f && bn.y == 0.f && bn.z == 0.f &&
              bn.w == 0.f) {
#pragma unroll
            for (int i = 0; i < 32; ++i) smax[i] = fmaxf(smax[i], __uint_as_float(r[i]));
            return;
          }
        }
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 b4 = *reinterpret_cast<const float4 *>(bb + i);
          float4 a4 = make_float4(sc, sc, sc, sc);
          if (ROWSCALE) a4 = *reinterpret_cast<const float4 *>(ba + i);
          smax[i] = fmaxf(smax[i], fmaf(__uint_as_float(r[i]), a4.x, b4.x));
          smax[i + 1] = fmaxf(smax[i + 1], fmaf(__uint_as_float(r[i + 1]), a4.y, b4.y));
          smax[i + 2] = fmaxf(smax[i + 2], fmaf(__uint_as_float(r[i + 2]), a4.z, b4.z));
          smax[i + 3] = fmaxf(smax[i + 3], fmaf(__uint_as_float(r[i + 3]), a4.w, b4.w));
        }
        return;
      }
      // fast path: per 8-column group an upper bound of its keys from the group's
      // largest raw dot and its bias / scale range -- fma is monotone in each
      // argument (scale > 0), so no key of the group can exceed it
      const float4 b4 = *reinterpret_cast<const float4 *>(gb);
      float4 ax4 = b4, an4 = b4;
      if (ROWSCALE) { ax4 = *reinterpret_cast<const float4 *>(ga); an4 = *reinterpret_cast<const float4 *>(gn); }
      float dmg[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) {   // (three-input FMNMX3: 4 instructions per group instead of 7)
        const float *x = reinterpret_cast<const float *>(r + g * 8);
        dmg[g] = fmax3f(fmax3f(x[0], x[1], x[2]), fmax3f(x[3], x[4], x[5]), fmaxf(x[6], x[7]));
      }
      TC_STAT(++st_chunks);
      uint32_t pass = 0;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const float dm = dmg[g];
        const float kb = ROWSCALE ? fmaf(dm, dm >= 0.f ? f4(ax4, g) : f4(an4, g), f4(b4, g)) : fmaf(dm, sc, f4(b4, g));
        pass |= (kb > thr ? 1u : 0u) << g;
      }
      if (!__any_sync(0xffffffffu, pass != 0)) return;
      // rare once the threshold is in place: exact keys of the flagged groups, make
      // room (<= 8 appends follow; the compaction histogram aliases the staging
      // rows), then each lane appends its accepted columns in row order from its
      // private staging row
      TC_STAT(++st_slow);
      if (MODE == MODE_MAIN && __any_sync(0xffffffffu, cnt + 32 > p.cap)) compact_needed(p.cap - 32);
#ifdef VRS_SLOW_GROUPS_VOTE
#pragma unroll
      for (int g = 0; g < 4; ++g) {   // (unrolled: r must stay in registers)
        if (!__any_sync(0xffffffffu, (pass >> g) & 1u)) continue;
        float kk[8];
#pragma unroll
        for (int i = 0; i < 8; i += 4) {
          const float4 bq = *reinterpret_cast<const float4 *>(bb + g * 8 + i);
          float4 aq = make_float4(sc, sc, sc, sc);
          if (ROWSCALE) aq = *reinterpret_cast<const float4 *>(ba + g * 8 + i);
          kk[i] = fmaf(__uint_as_float(r[g * 8 + i]), aq.x, bq.x);
          kk[i + 1] = fmaf(__uint_as_float(r[g * 8 + i + 1]), aq.y, bq.y);
          kk[i + 2] = fmaf(__uint_as_float(r[g * 8 + i + 2]), aq.z, bq.z);
          kk[i + 3] = fmaf(__uint_as_float(r[g * 8 + i + 3]), aq.w, bq.w);
        }
        uint32_t msk = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) msk |= (kk[i] > thr ? 1u : 0u) << i;
        if (MODE == MODE_RCOUNT) { cnt += __popc(msk); continue; }
        if (MODE == MODE_RFILL) {   // the list's segment, rows in ascending order
          while (msk) {
            const int i = __ffs(msk) - 1;
            msk &= msk - 1;
            cid[cnt++] = rid[g * 8 + i];
          }
          continue;
        }
        if (!__any_sync(0xffffffffu, msk != 0)) continue;
        float *myrow = wst + lane * STAGE_COLS;
        if (msk) {
          *reinterpret_cast<float4 *>(myrow) = make_float4(kk[0], kk[1], kk[2], kk[3]);
          *reinterpret_cast<float4 *>(myrow + 4) = make_float4(kk[4], kk[5], kk[6], kk[7]);
          TC_STAT(st_app += __popc(msk));
          while (msk) {
            const int i = __ffs(msk) - 1;
            msk &= msk - 1;
            ckey[cnt] = myrow[i];
            cid[cnt] = rid[g * 8 + i];
            ++cnt;
          }
        }
        __syncwarp();
      }
    #else
      // each lane walks only its own flagged groups (the warp runs max-over-lanes
      // iterations, ~1 per slow chunk, instead of every group any lane flagged);
      // the group's 8 raw dots are picked from the unrolled registers by selects
      uint32_t pm = pass;
      float *myrow = wst + lane * STAGE_COLS;
      while (__any_sync(0xffffffffu, pm != 0)) {
        if (pm) {
          const int g = __ffs(pm) - 1;
          pm &= pm - 1;
          float kk[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t lo = g == 0 ? r[i] : r[8 + i], hi = g == 2 ? r[16 + i] : r[24 + i];
            kk[i] = __uint_as_float(g < 2 ? lo : hi);
          }
#pragma unroll
          for (int i = 0; i < 8; i += 4) {
            const float4 bq = *reinterpret_cast<const float4 *>(bb + g * 8 + i);
            float4 aq = make_float4(sc, sc, sc, sc);
            if (ROWSCALE) aq = *reinterpret_cast<const float4 *>(ba + g * 8 + i);
            kk[i] = fmaf(kk[i], aq.x, bq.x);
            kk[i + 1] = fmaf(kk[i + 1], aq.y, bq.y);
            kk[i + 2] = fmaf(kk[i + 2], aq.z, bq.z);
            kk[i + 3] = fmaf(kk[i + 3], aq.w, bq.w);
          }
          uint32_t msk = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) msk |= (kk[i] > thr ? 1u : 0u) << i;
          if (MODE == MODE_RCOUNT) {
            cnt += __popc(msk);
          } else if (MODE == MODE_RFILL) {   // the list's segment, rows in ascending order
            while (msk) {
              const int i = __ffs(msk) - 1;
              msk &= msk - 1;
              cid[cnt++] = rid[g * 8 + i];
            }
          } else if (msk) {
            *reinterpret_cast<float4 *>(myrow) = make_float4(kk[0], kk[1], kk[2], kk[3]);
            *reinterpret_cast<float4 *>(myrow + 4) = make_float4(kk[4], kk[5], kk[6], kk[7]);
            TC_STAT(st_app += __popc(msk));
            while (msk) {
              const int i = __ffs(msk) - 1;
              msk &= msk - 1;
              ckey[cnt] = myrow[i];
              cid[cnt] = rid[g * 8 + i];
              ++cnt;
            }
          }
        }
      }
      __syncwarp();   // (the next compaction's histogram aliases the staging rows)
#endif
    };

    for (int t = 0; t < ntiles; ++t) {
      const int acc = t % ACC_STAGES;
      const int bs = t % BIAS_STAGES;
      mbar_wait(&bfull_bar[bs], (t / BIAS_STAGES) & 1);
      mbar_wait(&tfull_bar[acc], (t / ACC_STAGES) & 1);
      if (t == 0 && ew == 0 && lane == 0) TL_STAMP_ANY(MODE & 3, 3);
      tc_fence_after();
      const float *ba = bias_a + bs * BN + half * EPI_COLS;
      const float *bb = bias_b + bs * BN + half * EPI_COLS;
      const int32_t *rid = row_id + bs * BN + half * EPI_COLS;
      const int g0 = bs * GROUPS + half * (EPI_COLS / 8);   // this warp's first group
      const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * BN + half * EPI_COLS);
#if !defined(VRS_EPI_SKIP_BUILD) && !defined(VRS_EPI_X64)
      {   // one chunk in flight per warp (the other warps hide the TMEM load latency)
        uint32_t ra[32];
#pragma unroll 1
        for (int c = 0; c < EPI_COLS / 32; ++c) {
          TMEM_LD_32x32b_X32(tbase + c * 32, ra);
          TMEM_LD_WAIT(ra);
#ifdef VRS_EPI_READOUT_ONLY   // debug build: read-out only (keeps the loads live)
          {
            uint32_t x = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) x ^= ra[i];
            if (x == 0x9e3779b9u && p.stats) atomicAdd(p.stats + 3, 1ull);
            continue;
          }
#endif
          chunk(ra, ba + c * 32, bb + c * 32, rid + c * 32, g_bmax + g0 + c * 4, g_amax + g0 + c * 4, g_amin + g0 + c * 4);
        }
      }
#elif !defined(VRS_EPI_SKIP_BUILD)
      {   // A/B (VRS_EPI_X64): two chunks per tcgen05.ld (32x32b.x64) -- measured equal
        static_assert((EPI_COLS / 32) % 2 == 0, "pairs of chunks");
        uint32_t ra[64];
#pragma unroll 1
        for (int c = 0; c < EPI_COLS / 32; c += 2) {
          TMEM_LD_32x32b_X64(tbase + c * 32, ra);
          TMEM_LD_WAIT(ra);
          TMEM_LD_WAIT(reinterpret_cast<uint32_t(&)[32]>(ra[32]));
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int cc = c + h;
            chunk(reinterpret_cast<uint32_t(&)[32]>(ra[32 * h]), ba + cc * 32, bb + cc * 32, rid + cc * 32,
                  g_bmax + g0 + cc * 4, g_amax + g0 + cc * 4, g_amin + g0 + cc * 4);
          }
        }
      }
#endif
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR && !leader) mbar_arrive_cluster(mapa_rank(&tempty_bar[acc], 0));   // (the leader's MMA waits)
        else mbar_arrive(&tempty_bar[acc]);
        mbar_arrive(&bempty_bar[bs]);
      }
    }
    if (ew == 0 && lane == 0) TL_STAMP_ANY(MODE & 3, 4);
    if (p.stats && lane == 0) {
      atomicAdd(p.stats + 0, (unsigned long long)st_chunks);
      atomicAdd(p.stats + 1, (unsigned long long)st_slow);
      atomicAdd(p.stats + 2, (unsigned long long)st_app);
      atomicAdd(p.stats + 3, (unsigned long long)st_comp);
    }
    if (active) {
      if (MODE == MODE_PROBE) {
        float4 *dst = reinterpret_cast<float4 *>(p.probe_max + ((qg * (LPS * p.P)) + list) * SLOTS);
#pragma unroll
        for (int i = 0; i < SLOTS; i += 4) dst[i / 4] = make_float4(smax[i], smax[i + 1], smax[i + 2], smax[i + 3]);
      } else if (MODE != MODE_RFILL) {
        p.cand_cnt[(int64_t)list * p.q + lrow + qg] = cnt;
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();   // no remote arrival / MMA into this CTA's smem or TMEM is pending
  if (threadIdx.x == 0) {
    TC_TL(5);
#ifdef VRS_TC_TIMING
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (blockIdx.x < 4096) { g_tl[MODE & 3][blockIdx.x][6] = smid; g_tl[MODE & 3][blockIdx.x][7] = (unsigned long long)ntiles; }
#endif
  }
  if (warp == 1) {
    tc_fence_after();
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS) : "memory");
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS) : "memory");
  }
}

// Minimum row tiles per used split (VRS_MIN_SPAN overrides; default 4).
static int tc_min_span() {
  static const int v = getenv("VRS_MIN_SPAN") ? std::max(1, atoi(getenv("VRS_MIN_SPAN"))) : 4;
  return v;
}

// ---------------------------------------------------------------- launch plumbing
// Everything a tensor-core pass launch needs: the tensor maps (queries, rows, gathered
// rows; the refine pass's x_lo rows and gathered x_lo rows -- copies of mx otherwise),
// the mode-independent parameters and the variant flags.
struct TcLaunch {
  CUtensorMap mq, mx, mg, ml, mlg;
  TcParams p;
  bool bf, ar, rowscale;
  bool pair = false;   // main pass as CTA pairs (mx / mg then have boxes of BN / 2 rows)
  bool ar8 = false;    // <= 8 queries resident as 8 rows per K block (mq then has boxes of 8 rows)
};
// Queries -> bf16 (padded tiles), tensor maps, parameters, and the gather copy
// when the selection is materialised (gemm_tc.cu).
cudaError_t tc_prepare(const GemmArgs &a, const GemmPlan &plan, cudaStream_t s, int *launches, TcLaunch *L);

typedef void (*TcKernel)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, TcParams);
template <int ARM, int MODE, bool ROWSCALE, bool BF, bool PAIR>
__global__ void tc_topk_kernel(const __grid_constant__ CUtensorMap tmap_q, const __grid_constant__ CUtensorMap tmap_x,
                               const __grid_constant__ CUtensorMap tmap_g, const __grid_constant__ CUtensorMap tmap_xl,
                               const __grid_constant__ CUtensorMap tmap_gl, TcParams p);
template <int MODE, bool BF>
static TcKernel pick_kernel(bool ar, bool rowscale, bool pair = false, bool ar8 = false) {
  if constexpr (MODE == MODE_MAIN && BF) {
    if (pair) return rowscale ? tc_topk_kernel<0, MODE, true, BF, true> : tc_topk_kernel<0, MODE, false, BF, true>;
  }
  if constexpr ((MODE == MODE_MAIN || MODE == MODE_PROBE) && BF) {
    if (ar8) return rowscale ? tc_topk_kernel<2, MODE, true, BF, false> : tc_topk_kernel<2, MODE, false, BF, false>;
  }
  return ar ? (rowscale ? tc_topk_kernel<1, MODE, true, BF, false> : tc_topk_kernel<1, MODE, false, BF, false>)
            : (rowscale ? tc_topk_kernel<0, MODE, true, BF, false> : tc_topk_kernel<0, MODE, false, BF, false>);
}

// One launch of the pass in MODE (the kernels of a mode are instantiated in the
// translation unit that calls this).  VRS_STATS=1 prints the epilogue counters (they count only in
// builds with -DVRS_TC_STATS).
template <int MODE>
static cudaError_t tc_launch_mode(const TcLaunch &L, const TcParams &pr, cudaStream_t s) {
  static size_t attr[32] = {};   // per variant (AR8, PAIR, AR, ROWSCALE, BF)
  const TcKernel kern = L.bf ? pick_kernel<MODE, true>(L.ar, L.rowscale, L.pair, L.ar8)
                             : pick_kernel<MODE, false>(L.ar, L.rowscale, L.pair, L.ar8);
  cudaError_t e = ensure_smem_attr(kern, tc::SMEM_BYTES,
                                   attr[(L.ar8 ? 16 : 0) | (L.pair ? 8 : 0) | (L.ar ? 4 : 0) | (L.rowscale ? 2 : 0) |
                                        (L.bf ? 1 : 0)]);
  if (e != cudaSuccess) return e;
  static unsigned long long *stats = nullptr;
  static const bool want_stats = getenv("VRS_STATS") != nullptr;   // (debug counters, single-threaded use)
  if (want_stats && !stats) cudaMalloc(&stats, 64);
  TcParams p2 = pr;
  p2.stats = want_stats ? stats : nullptr;
  if (want_stats) cudaMemsetAsync(stats, 0, 64, s);
  e = launch_k_cluster(kern, dim3((unsigned)(pr.P * pr.qtiles)), dim3(tc::THREADS), tc::SMEM_BYTES, s, L.pair ? 2 : 1,
                       L.mq, L.mx, L.mg, L.ml, L.mlg, p2);
  if (want_stats) {
    unsigned long long h[4];
    cudaMemcpyAsync(h, stats, 32, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "[vrs stats] mode=%d grid=%d chunks=%llu slow=%llu (%.3f) appends=%llu compactions=%llu\n", MODE,
            pr.P * pr.qtiles, h[0], h[1], h[0] ? (double)h[1] / h[0] : 0.0, h[2], h[3]);
  }
  return e;
}

// ---------------------------------------------------------------- tensor maps
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

// 2-D map over a row-major [rows x d] matrix of fp32 or 16-bit values (fmt16: 0
// fp16, 1 bf16), boxes of one 128-byte K block x box_rows rows, 128-byte swizzle
// (box_rows = 1: the gather4 map, four such rows per instruction).
static bool make_map(CUtensorMap *m, const void *base, int64_t rows, int32_t d, int box_rows, bool h16, int fmt16 = 1) {
  auto fn = encode_fn();
  if (!fn) return false;
  const int esz = h16 ? 2 : 4;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * esz};
  cuuint32_t box[2] = {(cuuint32_t)(128 / esz), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, !h16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : (fmt16 == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16), 2,
                  const_cast<void *>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace vrs
