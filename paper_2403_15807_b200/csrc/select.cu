// select.cu -- K4'/K5': relational predicate scan -> selection bitmap, count and
// compacted ascending row ids (PAPER.md L283-L288 predicate pushdown; L319
// "first staging the fast relational predicate filtering, then collecting the
// vectors that satisfy the condition").
//
// Integer work, bit-exact by construction.  Two short passes:
//   select_count_kernel: each warp evaluates theta_R on 32 consecutive rows per
//     step (coalesced 128 B / 32 B column loads), __ballot_sync gives the
//     bitmap word and __popc its count; one block covers a contiguous chunk of
//     8192 rows and publishes the chunk count.
//   select_scatter_kernel: each block sums the counts of the chunks before it
//     (a parallel reduction over <= 4096 values; larger corpora get the
//     prefix from one select_prefix_kernel block instead), re-reads its 256
//     bitmap words (n/8 bytes in total, L2-resident) and scatters ascending row
//     ids with a warp prefix of popcounts; the last block writes the count.
// (A single-pass decoupled look-back was measured slower here: with the whole
// grid resident at once, tiles walk back through hundreds of aggregate-only
// predecessors.)
//
// Algorithmic bytes per row: sum of attribute widths read + 1/8 (bitmap) +
// 4 * selectivity (ids).  HBM-bound.
#include "convert16.cuh"

namespace vrs {

constexpr int kSelThreads = 256;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSelWordsPerWarp = 32;
constexpr int kSelWords = kSelWarps * kSelWordsPerWarp;  // 256 words
constexpr int kSelRows = kSelWords * 32;                 // 8192 rows per block

static_assert(kSelRows == kSelChunkRows, "chunk size shared with select_finish");

__global__ void __launch_bounds__(kSelThreads) select_count_kernel(PredDev pred, int64_t n,
                                                                   uint32_t *__restrict__ bitmap,
                                                                   uint32_t *__restrict__ chunk_count,
                                                                   SelectFuse fz, int32_t *__restrict__ ids_local) {
  TL_SCOPE(0);
  __shared__ uint32_t s_cnt[kSelWarps];
  pdl_wait();
  TL_WAITED(0);
  pdl_trigger();
  if (fz.q_out) {   // folded in: the 16-bit query operand, one warp per query row (convert16.cuh)
    for (int64_t row = (int64_t)blockIdx.x * kSelWarps + (threadIdx.x >> 5); row < fz.rows;
         row += (int64_t)gridDim.x * kSelWarps)
      query_row_to16(fz, row);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t base = (int64_t)blockIdx.x * kSelRows + (int64_t)warp * kSelWordsPerWarp * 32;
  // lane l owns row base + 32w + l for w = 0..31: per clause, all 32 column loads
  // are issued before any is used (one memory latency per clause, not 32)
  uint32_t selbits = 0xffffffffu;   // bit w: row base + 32w + lane qualifies
#pragma unroll
  for (int w = 0; w < kSelWordsPerWarp; ++w)
    if (base + (int64_t)w * 32 + lane >= n) selbits &= ~(1u << w);
  if (pred.empty) selbits = 0;
#pragma unroll 1
  for (int c = 0; c < pred.n; ++c) {
    const ClauseDev cl = pred.c[c];
    int32_t v[kSelWordsPerWarp];
    if (cl.type == VRS_ATTR_I32) {
      const int32_t *col = static_cast<const int32_t *>(cl.col);
#pragma unroll
      for (int w = 0; w < kSelWordsPerWarp; ++w) {
        const int64_t row = base + (int64_t)w * 32 + lane;
        v[w] = row < n ? __ldg(col + row) : 0;
      }
    } else {
      const uint8_t *col = static_cast<const uint8_t *>(cl.col);
#pragma unroll
      for (int w = 0; w < kSelWordsPerWarp; ++w) {
        const int64_t row = base + (int64_t)w * 32 + lane;
        v[w] = row < n ? (int32_t)__ldg(col + row) : 0;
      }
    }
#pragma unroll
    for (int w = 0; w < kSelWordsPerWarp; ++w)
      if (!(cl.lo <= v[w] && v[w] <= cl.hi)) selbits &= ~(1u << w);
  }
  uint32_t my_word = 0;
#pragma unroll
  for (int w = 0; w < kSelWordsPerWarp; ++w) {
    const uint32_t word = __ballot_sync(0xffffffffu, (selbits >> w) & 1u);
    if (lane == w) my_word = word;
  }
  const int64_t wrow = base + (int64_t)lane * 32;
  if (wrow < n) bitmap[wrow >> 5] = my_word;
  uint32_t c = __popc(my_word);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) s_cnt[warp] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
#pragma unroll
    for (int i = 0; i < kSelWarps; ++i) t += s_cnt[i];
    chunk_count[blockIdx.x] = t;
  }
  if (ids_local != nullptr) {
    // chunk-local ids (no global prefix needed): warp-cooperative, coalesced, as in
    // select_scatter_kernel but relative to this chunk's slot range
    uint32_t wpre = 0;
    for (int i = 0; i < warp; ++i) wpre += s_cnt[i];
    const uint32_t pc = __popc(my_word);
    uint32_t incl = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int32_t *out = ids_local + (int64_t)blockIdx.x * kSelRows + wpre;
#pragma unroll 4
    for (int w = 0; w < 32; ++w) {
      const uint32_t ww = __shfl_sync(0xffffffffu, my_word, w);
      const uint32_t before = __shfl_sync(0xffffffffu, incl - pc, w);
      if ((ww >> lane) & 1u) out[before + __popc(ww & lanemask_lt())] = (int32_t)(base + w * 32 + lane);
    }
  }
}

// Corpora of more than kSelDirectChunks chunks: the exclusive prefix of the chunk counts
// by one block (a contiguous segment per thread, a block scan of the segment sums), so
// that select_scatter's prefix stays O(1) per block -- summing every earlier chunk in
// each block is O(chunks^2) in total (fine at C3's 1221 chunks, not toward n ~ 2^31).
constexpr uint32_t kSelDirectChunks = 4096;
constexpr int kSelPrefixThreads = 1024;
__global__ void __launch_bounds__(kSelPrefixThreads) select_prefix_kernel(const uint32_t *__restrict__ chunk_count,
                                                                          uint32_t nchunks,
                                                                          uint64_t *__restrict__ prefix) {
  __shared__ uint64_t s_w[kSelPrefixThreads / 32];
  pdl_wait();
  pdl_trigger();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t per = (nchunks + kSelPrefixThreads - 1) / kSelPrefixThreads;
  const uint32_t b0 = min(nchunks, tid * per), b1 = min(nchunks, b0 + per);
  uint64_t mine = 0;
  for (uint32_t b = b0; b < b1; ++b) mine += chunk_count[b];
  uint64_t incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  uint64_t run = incl - mine;
  for (int i = 0; i < warp; ++i) run += s_w[i];
  for (uint32_t b = b0; b < b1; ++b) {
    prefix[b] = run;
    run += chunk_count[b];
  }
}

__global__ void __launch_bounds__(kSelThreads) select_scatter_kernel(int64_t n, const uint32_t *__restrict__ bitmap,
                                                                     const uint32_t *__restrict__ chunk_count,
                                                                     const uint64_t *__restrict__ prefix,
                                                                     int32_t *__restrict__ ids,
                                                                     int64_t *__restrict__ count) {
  TL_SCOPE(1);
  __shared__ uint64_t s_red[kSelWarps];
  pdl_wait();
  TL_WAITED(1);
  pdl_trigger();
  __shared__ uint32_t s_wsum[kSelWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // prefix over the chunks before this block (select_prefix_kernel's, or summed here)
  uint64_t pre = 0;
  if (prefix == nullptr)
    for (uint32_t b = threadIdx.x; b < blockIdx.x; b += kSelThreads) pre += chunk_count[b];
  else if (threadIdx.x == 0)
    pre = prefix[blockIdx.x];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
  if (lane == 0) s_red[warp] = pre;
  // this thread's word and its rank within the block
  const int64_t word_idx = (int64_t)blockIdx.x * kSelWords + threadIdx.x;
  const uint32_t word = (word_idx * 32 < n) ? bitmap[word_idx] : 0u;
  const uint32_t c = __popc(word);
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  uint64_t base = 0;
#pragma unroll
  for (int i = 0; i < kSelWarps; ++i) base += s_red[i];
  uint32_t wpre = 0;
  for (int i = 0; i < warp; ++i) wpre += s_wsum[i];
  if (ids != nullptr) {
    // warp-cooperative, coalesced: for each of the warp's 32 words, lane l emits bit l
    const uint64_t wbase = base + wpre;
    const int64_t row0 = ((int64_t)blockIdx.x * kSelWords + warp * 32) * 32;
#pragma unroll 4
    for (int w = 0; w < 32; ++w) {
      const uint32_t ww = __shfl_sync(0xffffffffu, word, w);
      const uint32_t before = __shfl_sync(0xffffffffu, incl - c, w);
      if ((ww >> lane) & 1u) ids[wbase + before + __popc(ww & lanemask_lt())] = (int32_t)(row0 + w * 32 + lane);
    }
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kSelThreads - 1) *count = (int64_t)(base + wpre + incl);
}

// scratch: chunk counts uint32[nchunks] (+ 8), then the chunk prefix uint64[nchunks] (8-byte aligned)
static size_t select_prefix_offset(int64_t n) { return ((size_t)((n + kSelRows - 1) / kSelRows) * 4 + 8 + 7) & ~size_t(7); }
size_t select_scratch_bytes(int64_t n) { return select_prefix_offset(n) + (size_t)((n + kSelRows - 1) / kSelRows) * 8; }

// Host launcher.  Scratch: chunk counts uint32[nchunks].  ids may be nullptr
// (bitmap + count only).
cudaError_t launch_select(const PredDev &pred, int64_t n, uint32_t *bitmap, int32_t *ids, int64_t *count,
                          void *scratch, cudaStream_t stream, int *launches, const SelectFuse *fuse) {
  const SelectFuse fz = fuse ? *fuse : SelectFuse{};
  const uint32_t nchunks = (uint32_t)((n + kSelRows - 1) / kSelRows);
  uint32_t *chunk_count = static_cast<uint32_t *>(scratch);
  cudaError_t e0 = launch_k(select_count_kernel, dim3(nchunks), dim3(kSelThreads), 0, stream, pred, n, bitmap, chunk_count, fz,
                            (int32_t *)nullptr);
  if (e0 != cudaSuccess) return e0;
  if (launches) *launches += 1;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  static const uint32_t direct_max = getenv("VRS_SELECT_DIRECT_MAX") ? (uint32_t)atoi(getenv("VRS_SELECT_DIRECT_MAX"))
                                                                     : kSelDirectChunks;   // (tests: force the prefix kernel)
  uint64_t *prefix = nullptr;
  if (nchunks > direct_max) {
    prefix = reinterpret_cast<uint64_t *>(static_cast<char *>(scratch) + select_prefix_offset(n));
    e = launch_k(select_prefix_kernel, dim3(1), dim3(kSelPrefixThreads), 0, stream, (const uint32_t *)chunk_count,
                 nchunks, prefix);
    if (e != cudaSuccess) return e;
    if (launches) *launches += 1;
  }
  e = launch_k(select_scatter_kernel, dim3(nchunks), dim3(kSelThreads), 0, stream, n, (const uint32_t *)bitmap,
               (const uint32_t *)chunk_count, (const uint64_t *)prefix, ids, count);
  if (e != cudaSuccess) return e;
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_select_local(const PredDev &pred, int64_t n, uint32_t *bitmap, int32_t *ids_local, void *scratch,
                                cudaStream_t stream, int *launches, const SelectFuse *fuse) {
  const SelectFuse fz = fuse ? *fuse : SelectFuse{};
  const uint32_t nchunks = (uint32_t)((n + kSelRows - 1) / kSelRows);
  cudaError_t e = launch_k(select_count_kernel, dim3(nchunks), dim3(kSelThreads), 0, stream, pred, n, bitmap,
                           static_cast<uint32_t *>(scratch), fz, ids_local);
  if (e != cudaSuccess) return e;
  if (launches) *launches += 1;
  return cudaGetLastError();
}


}  // namespace vrs

#ifdef VRS_TC_TIMING
namespace vrs {
int tl_read_select(unsigned long long *host) { return tl_read(host); }
}
#endif
