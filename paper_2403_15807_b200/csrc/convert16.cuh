// convert16.cuh -- fp32 -> 16-bit (fp16 / bf16) operand conversion with a
// power-of-two scale and an exact fp64 residual.  Shared by
// the shadow kernel at load (gemm_tc.cu) and the per-search query conversion
// (standalone in gemm_tc.cu, folded into select_count_kernel in select.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "vrs_kernels.cuh"

namespace vrs {

__device__ __forceinline__ uint32_t pack16x2(float a, float b, int fmt) {
  if (fmt == 0) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t *>(&h);
  }
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t *>(&h);
}
__device__ __forceinline__ float2 unpack16x2(uint32_t w, int fmt) {
  if (fmt == 0) return __half22float2(*reinterpret_cast<const __half2 *>(&w));
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&w));
}
// exponent that puts max|v| into [2^14, 2^15) (fp16), 0 for bf16 or a zero row
__device__ __forceinline__ int scale_exp16(float amax, int fmt) {
  if (fmt != 0 || !(amax > 0.f) || !(amax < INFINITY)) return 0;
  return max(-120, min(120, 14 - ilogbf(amax)));
}

// One row of d values (d % 4 == 0, 16-byte aligned) -> 16-bit with exponent e, by
// one warp; returns |converted * 2^-e - v|^2 (fp64) on every lane.
__device__ __forceinline__ double row_to16(const float *__restrict__ in, uint16_t *__restrict__ out, int d, int e, int fmt) {
  const int lane = threadIdx.x & 31;
  double r2 = 0.0;
  for (int t = 4 * lane; t < d; t += 128) {
    const float4 v = __ldg(reinterpret_cast<const float4 *>(in + t));
    uint2 w;
    w.x = pack16x2(ldexpf(v.x, e), ldexpf(v.y, e), fmt);
    w.y = pack16x2(ldexpf(v.z, e), ldexpf(v.w, e), fmt);
    *reinterpret_cast<uint2 *>(out + t) = w;
    const float2 a = unpack16x2(w.x, fmt), b = unpack16x2(w.y, fmt);
    const double d0 = ldexp((double)a.x, -e) - v.x, d1 = ldexp((double)a.y, -e) - v.y;
    const double d2 = ldexp((double)b.x, -e) - v.z, d3 = ldexp((double)b.y, -e) - v.w;
    r2 += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
  return r2;
}

// One row -> a 16-bit pair (fp16 only): hi = fp16(v 2^e), lo = fp16(v 2^e - hi) (the
// difference is exact in fp32), by one warp; returns |hi 2^-e - v|^2 in .x and
// |(hi + lo) 2^-e - v|^2 in .y (fp64) on every lane.  The refine pass multiplies
// q_hi.x_hi + q_hi.x_lo + q_lo.x_hi ("Refine").
__device__ __forceinline__ double2 row_to16x2(const float *__restrict__ in, uint16_t *__restrict__ hi,
                                              uint16_t *__restrict__ lo, int d, int e) {
  const int lane = threadIdx.x & 31;
  double r1 = 0.0, r2 = 0.0;
  for (int t = 4 * lane; t < d; t += 128) {
    const float4 v = __ldg(reinterpret_cast<const float4 *>(in + t));
    const float s0 = ldexpf(v.x, e), s1 = ldexpf(v.y, e), s2 = ldexpf(v.z, e), s3 = ldexpf(v.w, e);
    uint2 wh;
    wh.x = pack16x2(s0, s1, 0);
    wh.y = pack16x2(s2, s3, 0);
    const float2 h01 = unpack16x2(wh.x, 0), h23 = unpack16x2(wh.y, 0);
    uint2 wl;
    wl.x = pack16x2(s0 - h01.x, s1 - h01.y, 0);
    wl.y = pack16x2(s2 - h23.x, s3 - h23.y, 0);
    *reinterpret_cast<uint2 *>(hi + t) = wh;
    if (lo) *reinterpret_cast<uint2 *>(lo + t) = wl;
    const float2 l01 = unpack16x2(wl.x, 0), l23 = unpack16x2(wl.y, 0);
    const double a0 = ldexp((double)h01.x, -e) - v.x, a1 = ldexp((double)h01.y, -e) - v.y;
    const double a2 = ldexp((double)h23.x, -e) - v.z, a3 = ldexp((double)h23.y, -e) - v.w;
    r1 += a0 * a0 + a1 * a1 + a2 * a2 + a3 * a3;
    const double b0 = ldexp((double)h01.x + l01.x, -e) - v.x, b1 = ldexp((double)h01.y + l01.y, -e) - v.y;
    const double b2 = ldexp((double)h23.x + l23.x, -e) - v.z, b3 = ldexp((double)h23.y + l23.y, -e) - v.w;
    r2 += b0 * b0 + b1 * b1 + b2 * b2 + b3 * b3;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    r1 += __shfl_xor_sync(0xffffffffu, r1, o);
    r2 += __shfl_xor_sync(0xffffffffu, r2, o);
  }
  return make_double2(r1, r2);
}

// One query row (warp): per-row exponent, 16-bit row, exponent and residual
// (rounded up) to qexp / rq.  Rows q..rows-1 are zero padding (whole 128-row tiles).
__device__ __forceinline__ void query_row_to16(const QueryFuse &f, int64_t row) {
  const int lane = threadIdx.x & 31;
  uint16_t *out = static_cast<uint16_t *>(f.q_out) + row * f.d;
  if (row >= f.q) {
    for (int t = 4 * lane; t < f.d; t += 128) *reinterpret_cast<uint2 *>(out + t) = make_uint2(0u, 0u);
    return;
  }
  const float *in = f.q_in + row * f.d;
  float am = 0.f;
  for (int t = 4 * lane; t < f.d; t += 128) {
    const float4 v = __ldg(reinterpret_cast<const float4 *>(in + t));
    am = fmaxf(am, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
  const int e = scale_exp16(am, f.fmt);
  const double r2 = row_to16(in, out, f.d, e, f.fmt);
  if (lane == 0) {
    f.qexp[row] = e;
    f.rq[row] = __double2float_ru(sqrt(r2) * (1.0 + 0x1p-50));
  }
}

}  // namespace vrs
