// swiglu.cu -- A5: fused SwiGLU + 1x128 power-of-two E4M3 quantization.
//
// Paper: P:380-381 ("we fuse the SwiGLU activation and quantization steps into a single kernel"),
// BF16 input from the first BF16 boundary, tile scale Eq. 2, codes Eq. 3.
// Readings: R18 a = h[:, :F] is gated (silu), b = h[:, F:] linear; R20 the
// reference value is a*b / (1 + e^-a) evaluated in fp64 and rounded once to fp32 (oracle C10);
// acceptance: codes within 1 E4M3 ULP on <= 1e-4 of elements, scale bytes identical.
//
// Kernel: the A1 work decomposition (warp item = 32 rows x 256 output columns, half-warp per
// 1x128 tile, 32-byte MN-major scale runs) with the activation evaluated in fp32 using the MUFU
// fast path y' = (a*b) / (1 + 2^(-a*log2e)) (a*b is exact: two 8-bit significands).  |y' - y| is
// bounded by ~70 fp32 ulp for |a| <= 64, so every decision the fp32 value takes is checked with
// a +-2^-16 relative bracket and re-taken from an fp64 evaluation when the bracket straddles it:
//   * the tile scale: amax' within the bracket of a boundary 448 * 2^T -> the elements that can
//     be the true max are recomputed in fp64 before the scale is chosen;
//   * each code: if cvt(u (1 - 2^-16)) != cvt(u (1 + 2^-16)) the element is recomputed in fp64.
// Elements with |a| > 64 (exp overflow range) or |a*b| < 2^-100 (subnormal range) always take
// the fp64 path.
#include "common.cuh"
#include "kernels.h"

namespace fp8flow {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kBracketLo = 1.0f - 1.52587890625e-05f;  // 1 - 2^-16
constexpr float kBracketHi = 1.0f + 1.52587890625e-05f;  // 1 + 2^-16

__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float swiglu_fast(float ab, float a) {
  return __fdividef(ab, 1.0f + ex2_approx(-a * kLog2e));  // MUFU.EX2 + MUFU.RCP
}
__device__ __noinline__ float swiglu_exact(float a, float b) {
  const double ad = static_cast<double>(a), bd = static_cast<double>(b);
  return static_cast<float>(ad * bd / (1.0 + exp(-ad)));
}

__global__ void __launch_bounds__(256) swiglu_quant_kernel(const __nv_bfloat16* __restrict__ h, int64_t rows_max,
                                                           const int32_t* __restrict__ rows_dev, int64_t F,
                                                           uint8_t* __restrict__ q, uint8_t* __restrict__ s,
                                                           int64_t ld_s) {
  const int lane = threadIdx.x & 31, half = lane >> 4, sub = lane & 15;
  const int64_t rows = rows_dev != nullptr ? static_cast<int64_t>(*rows_dev) : rows_max;
  const int64_t col_pairs = (F + 255) / 256;
  const int64_t n_items = ((rows + 31) / 32) * col_pairs;
  const int64_t warp_global = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t warp_stride = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t ld_h = 2 * F;

  for (int64_t item = warp_global; item < n_items; item += warp_stride) {
    const int64_t rg = item / col_pairs;
    const int64_t cp = item - rg * col_pairs;
    const int64_t row0 = rg * 32;
    const int64_t col = cp * 256 + half * 128 + sub * 8;
    const bool col_ok = col < F;
    const int nrows = static_cast<int>(min64(32, rows - row0));
    uint32_t sc0 = 0, sc1 = 0;

#pragma unroll 1
    for (int rb = 0; rb < 32; rb += 4) {
      uint4 va[4], vb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        va[i] = vb[i] = make_uint4(0, 0, 0, 0);
        if (rb + i < nrows && col_ok) {
          const __nv_bfloat16* p = h + (row0 + rb + i) * ld_h + col;
          va[i] = ld_nc_v4(p);
          vb[i] = ld_nc_v4(p + F);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = rb + i;
        const uint32_t wa[4] = {va[i].x, va[i].y, va[i].z, va[i].w};
        const uint32_t wb[4] = {vb[i].x, vb[i].y, vb[i].z, vb[i].w};
        float a[8], b[8], y[8];
        bool wild = false;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          a[2 * j] = bf16lo_to_f32(wa[j]);
          a[2 * j + 1] = bf16hi_to_f32(wa[j]);
          b[2 * j] = bf16lo_to_f32(wb[j]);
          b[2 * j + 1] = bf16hi_to_f32(wb[j]);
        }
        uint32_t mag = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float ab = a[j] * b[j];  // exact unless it underflows
          y[j] = swiglu_fast(ab, a[j]);
          wild |= fabsf(a[j]) > 64.0f || (ab != 0.0f && fabsf(ab) < 7.888609052210118e-31f);  // 2^-100
          mag = max(mag, __float_as_uint(y[j]) & 0x7FFFFFFFu);
        }
        if (wild) {  // exp overflow range: exact evaluation
#pragma unroll
          for (int j = 0; j < 8; ++j) y[j] = swiglu_exact(a[j], b[j]);
          mag = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) mag = max(mag, __float_as_uint(y[j]) & 0x7FFFFFFFu);
        }
        mag = halfwarp_max_u32(mag);
        // scale decision: near the boundary amax = 1.75 * 2^e (mantissa field 0x600000)?
        const int32_t dm = static_cast<int32_t>(mag & 0x7FFFFFu) - 0x600000;
        const bool near = (mag >> 23) != 0u && dm >= -512 && dm <= 512;
        if (__any_sync(0xffffffffu, near)) {
          if (near) {
            const float thr = __uint_as_float(mag) * (1.0f - 6.103515625e-05f);  // 1 - 2^-14
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (fabsf(y[j]) >= thr) y[j] = swiglu_exact(a[j], b[j]);
            uint32_t m2 = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) m2 = max(m2, __float_as_uint(y[j]) & 0x7FFFFFFFu);
            mag = m2;
          }
          mag = halfwarp_max_u32(mag);
        }
        const uint32_t sb = scale_byte_from_f32_mag(mag);
        const float inv = inv_scale_from_byte(sb);
        uint32_t c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float u0 = y[2 * j] * inv, u1 = y[2 * j + 1] * inv;
          uint32_t cc = cvt_e4m3x2_f32(u0, u1);
          const uint32_t lo = cvt_e4m3x2_f32(u0 * kBracketLo, u1 * kBracketLo);
          const uint32_t hi = cvt_e4m3x2_f32(u0 * kBracketHi, u1 * kBracketHi);
          if (lo != hi) {  // a rounding boundary lies inside the error bracket: decide in fp64
            u0 = swiglu_exact(a[2 * j], b[2 * j]) * inv;
            u1 = swiglu_exact(a[2 * j + 1], b[2 * j + 1]) * inv;
            cc = cvt_e4m3x2_f32(u0, u1);
          }
          c[j] = cc;
        }
        if (r < nrows && col_ok) st_v2(q + (row0 + r) * F + col, c[0] | (c[1] << 16), c[2] | (c[3] << 16));
        const uint32_t s0 = __shfl_sync(0xffffffffu, sb, 0);
        const uint32_t s1 = __shfl_sync(0xffffffffu, sb, 16);
        if (lane == r) {
          sc0 = s0;
          sc1 = s1;
        }
      }
    }
    if (lane < nrows) {
      const int64_t t0 = cp * 2;
      s[t0 * ld_s + row0 + lane] = static_cast<uint8_t>(sc0);
      if ((t0 + 1) * 128 < F) s[(t0 + 1) * ld_s + row0 + lane] = static_cast<uint8_t>(sc1);
    }
  }
}

cudaError_t launch_swiglu_quant(const void* h, int64_t rows_max, const int32_t* rows_dev, int64_t ffn, uint8_t* q,
                                uint8_t* s, int64_t ld_s, cudaStream_t stream, int num_sms) {
  const int64_t n_items = ((rows_max + 31) / 32) * ((ffn + 255) / 256);
  int64_t blocks = (n_items + 7) / 8;
  const int64_t cap = static_cast<int64_t>(num_sms) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  swiglu_quant_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(h), rows_max, rows_dev, ffn, q, s, ld_s);
  return cudaGetLastError();
}

}  // namespace fp8flow
