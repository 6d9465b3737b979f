// Standalone check of TMA tile::gather4 on sm_100a: gathers 8 rows (2 instructions) of a
// [n x 32] fp32 matrix by index into 128B-swizzled shared memory and reports the layout.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap map, const int *rows, float *out) {
  __shared__ __align__(1024) float tile[8 * 32];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(8 * 128));
    for (int g = 0; g < 2; ++g) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::
              "r"(smem_u32(tile + g * 4 * 32)), "l"(&map), "r"(0), "r"(rows[4 * g]), "r"(rows[4 * g + 1]), "r"(rows[4 * g + 2]),
          "r"(rows[4 * g + 3]), "r"(smem_u32(&bar))
          : "memory");
    }
  }
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)));
  for (int i = threadIdx.x; i < 8 * 32; i += blockDim.x) out[i] = tile[i];
}

int main() {
  const int n = 64, d = 32;
  float h[n * d];
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < d; ++c) h[r * d + c] = r * 100 + c;
  float *dX, *dO;
  int *dR;
  int rows[8] = {5, 9, 2, 63, 17, 0, 40, 33};
  cudaMalloc(&dX, sizeof h);
  cudaMalloc(&dO, 8 * 32 * 4);
  cudaMalloc(&dR, sizeof rows);
  cudaMemcpy(dX, h, sizeof h, cudaMemcpyHostToDevice);
  cudaMemcpy(dR, rows, sizeof rows, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &qr);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n};
  cuuint64_t str[1] = {(cuuint64_t)d * 4};
  cuuint32_t box[2] = {32, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dX, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode box{32,1}: %d\n", (int)r);
  k<<<1, 128>>>(map, dR, dO);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  float o[8 * 32];
  cudaMemcpy(o, dO, sizeof o, cudaMemcpyDeviceToHost);
  int ok_sw = 1, ok_lin = 1;
  for (int rr = 0; rr < 8; ++rr)
    for (int c = 0; c < 32; ++c) {
      const float want = rows[rr] * 100 + c;
      const int chunk = c / 4, sw = ((chunk ^ (rr & 7)) * 4) + (c % 4);
      if (o[rr * 32 + sw] != want) ok_sw = 0;
      if (o[rr * 32 + c] != want) ok_lin = 0;
    }
  printf("swizzled layout match: %d, linear layout match: %d\n", ok_sw, ok_lin);
  printf("row0: ");
  for (int c = 0; c < 32; ++c) printf("%g ", o[c]);
  printf("\nrow1: ");
  for (int c = 0; c < 32; ++c) printf("%g ", o[32 + c]);
  printf("\n");
  return 0;
}
