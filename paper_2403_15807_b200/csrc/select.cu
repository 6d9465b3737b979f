// select.cu -- K4'/K5': relational predicate scan -> selection bitmap, count and
// compacted ascending row ids, in ONE pass (PAPER.md L283-L288 predicate
// pushdown; L319 "first staging the fast relational predicate filtering, then
// collecting the vectors that satisfy the condition").
//
// Integer work, bit-exact by construction.  Each warp evaluates theta_R on 32
// consecutive rows (coalesced 128 B / 32 B column loads), __ballot_sync gives
// the bitmap word, __popc its count.  Tiles of 1024 rows get their output
// offset through a single-pass decoupled look-back prefix scan (tiles are
// numbered by an atomic ticket, so a tile only ever waits on tiles that are
// already running: no forward-progress assumption on block scheduling).
//
// Algorithmic bytes per row: sum of attribute widths read + 1/8 (bitmap) +
// 4 * selectivity (ids).  HBM-bound.
#include "vrs_kernels.cuh"

namespace vrs {

constexpr int kSelThreads = 256;
constexpr int kSelWordsPerWarp = 4;
constexpr int kSelWords = (kSelThreads / 32) * kSelWordsPerWarp;  // 32 words
constexpr int kSelRows = kSelWords * 32;                           // 1024 rows per tile

constexpr uint64_t kFlagAgg = 1ull << 62;   // tile aggregate published
constexpr uint64_t kFlagIncl = 2ull << 62;  // inclusive prefix published
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ void st_volatile_u64(uint64_t *p, uint64_t v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(PredDev pred, int64_t n, uint32_t *__restrict__ bitmap,
                                                             int32_t *__restrict__ ids, int64_t *__restrict__ count,
                                                             uint64_t *__restrict__ tile_state,
                                                             uint32_t *__restrict__ ticket, uint32_t ntiles) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_words[kSelWords];
  __shared__ uint32_t s_wexcl[kSelWords];
  __shared__ uint64_t s_prefix;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t base = (int64_t)tile * kSelRows;

  // 1. theta_R per row, one bitmap word per 32 rows
#pragma unroll
  for (int w = 0; w < kSelWordsPerWarp; ++w) {
    const int widx = warp * kSelWordsPerWarp + w;
    const int64_t row = base + (int64_t)widx * 32 + lane;
    const bool sel = (row < n) && eval_pred(pred, row);
    const uint32_t word = __ballot_sync(0xffffffffu, sel);
    if (lane == 0) {
      s_words[widx] = word;
      if (base + (int64_t)widx * 32 < n) bitmap[(base >> 5) + widx] = word;
    }
  }
  __syncthreads();

  // 2. tile-local exclusive scan of word popcounts + decoupled look-back
  if (warp == 0) {
    const uint32_t c = __popc(s_words[lane]);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    s_wexcl[lane] = incl - c;
    const uint64_t total = __shfl_sync(0xffffffffu, incl, 31);
    // warp-parallel decoupled look-back: lane i inspects tile (look - i); the
    // nearest inclusive prefix ends the walk, aggregates before it are summed
    uint64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) st_volatile_u64(tile_state, kFlagIncl | total);
    } else {
      if (lane == 0) st_volatile_u64(tile_state + tile, kFlagAgg | total);
      int64_t look = (int64_t)tile - 1;
      while (true) {
        const int64_t i = look - lane;
        uint64_t st = kFlagIncl;  // before tile 0: inclusive prefix 0
        if (i >= 0) {
          do {
            st = ld_volatile_u64(tile_state + i);
          } while ((st >> 62) == 0);
        }
        const uint32_t incl_mask = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        const int first = incl_mask ? __ffs(incl_mask) - 1 : 32;
        uint64_t v = (lane <= first) ? (st & kValMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (incl_mask) break;
        look -= 32;
      }
      if (lane == 0) {
        __threadfence();
        st_volatile_u64(tile_state + tile, kFlagIncl | (excl + total));
      }
    }
    if (lane == 0) {
      s_prefix = excl;
      if (tile == ntiles - 1) *count = (int64_t)(excl + total);
    }
  }
  __syncthreads();

  // 3. scatter ascending ids (late materialization's selection vector)
  if (ids != nullptr) {
    const uint64_t prefix = s_prefix;
#pragma unroll
    for (int w = 0; w < kSelWordsPerWarp; ++w) {
      const int widx = warp * kSelWordsPerWarp + w;
      const uint32_t word = s_words[widx];
      if ((word >> lane) & 1u) {
        const uint64_t pos = prefix + s_wexcl[widx] + __popc(word & lanemask_lt());
        ids[pos] = (int32_t)(base + (int64_t)widx * 32 + lane);
      }
    }
  }
}

// Host launcher.  Scratch: tile_state uint64[ntiles] + ticket uint32 (zeroed here).
cudaError_t launch_select(const PredDev &pred, int64_t n, uint32_t *bitmap, int32_t *ids, int64_t *count,
                          void *scratch, cudaStream_t stream, int *launches) {
  const uint32_t ntiles = (uint32_t)((n + kSelRows - 1) / kSelRows);
  uint64_t *tile_state = static_cast<uint64_t *>(scratch);
  uint32_t *ticket = reinterpret_cast<uint32_t *>(tile_state + ntiles);
  cudaError_t e = cudaMemsetAsync(scratch, 0, (size_t)ntiles * 8 + 8, stream);
  if (e != cudaSuccess) return e;
  select_kernel<<<ntiles, kSelThreads, 0, stream>>>(pred, n, bitmap, ids, count, tile_state, ticket, ntiles);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

size_t select_scratch_bytes(int64_t n) { return (size_t)((n + kSelRows - 1) / kSelRows) * 8 + 8; }

}  // namespace vrs
