// TMEM read-out bandwidth on this GPU (B200, sm_100a): W warps per CTA, one CTA
// per SM, each warp repeatedly loads 32 lanes x NCOL columns (tcgen05.ld
// 32x32b.xNCOL) from its TMEM lane quadrant and waits; bytes / SM clock cycles.
// The secondary roofline of the fused top-k epilogue (every fp32 accumulator is
// read out of TMEM once) uses this number.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu && ./tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define LD32(taddr, r)                                                                                            \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16," \
               "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                           \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),       \
                 "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),     \
                 "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),     \
                 "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                          \
               : "r"(taddr))
#define WAIT(r)                                                                                                  \
  asm volatile("tcgen05.wait::ld.sync.aligned;"                                                                 \
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]), \
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),       \
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),     \
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),     \
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])                                                          \
               :                                                                                                 \
               : "memory")

// inflight: loads issued before each wait (1 = load, wait, use; 2 = two buffers)
template <int INFLIGHT>
__global__ void tmem_read(int iters, unsigned long long *cycles, uint32_t *sink) {
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tbase_s))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tbase_s + ((uint32_t)((warp & 3) * 32) << 16);
  const int colw = (warp >> 2) * 32 * INFLIGHT;   // warps of one quadrant read different columns
  uint32_t acc = 0;
  uint32_t r[INFLIGHT][32];
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int col = (colw + it * 32 * INFLIGHT) & 511 & ~31;
#pragma unroll
    for (int b = 0; b < INFLIGHT; ++b) LD32(tb + ((col + 32 * b) & 511), r[b]);
#pragma unroll
    for (int b = 0; b < INFLIGHT; ++b) WAIT(r[b]);
#pragma unroll
    for (int b = 0; b < INFLIGHT; ++b)
#pragma unroll
      for (int i = 0; i < 32; ++i) acc ^= r[b][i];
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase_s) : "memory");
}

template <int INFLIGHT>
static void run(int warps, int sms) {
  const int iters = 20000;
  unsigned long long *cyc;
  uint32_t *sink;
  cudaMalloc(&cyc, sms * 8);
  cudaMalloc(&sink, 4);
  tmem_read<INFLIGHT><<<sms, warps * 32>>>(100, cyc, sink);   // warm-up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  tmem_read<INFLIGHT><<<sms, warps * 32>>>(iters, cyc, sink);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[1024];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double bytes_sm = (double)warps * iters * INFLIGHT * 32 * 32 * 4;
  printf("warps %2d inflight %d: %.1f B/clk/SM (clock64), %.2f TB/s chip (%d SMs, events %.3f ms)\n", warps, INFLIGHT,
         bytes_sm / mx, bytes_sm * sms / (ms * 1e-3) / 1e12, sms, ms);
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 16}) {
    run<1>(w, sms);
    run<2>(w, sms);
  }
  return 0;
}
