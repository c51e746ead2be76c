// swiglu.cu -- A5: fused SwiGLU + 1x128 power-of-two E4M3 quantization.
//
// Paper: P:380-381 ("we fuse the SwiGLU activation and quantization steps into a single kernel"),
// BF16 input from the first BF16 boundary, tile scale Eq. 2, codes Eq. 3.
// Readings: R18 a = h[:, :F] is gated (silu), b = h[:, F:] linear; R20 the
// reference value is a*b / (1 + e^-a) evaluated in fp64 and rounded once to fp32 (oracle C10);
// acceptance: codes within 1 E4M3 ULP on <= 1e-4 of elements, scale bytes identical.
//
// Kernel: the A1 work decomposition (warp item = 4 rows x 256 output columns, half-warp per 1x128
// tile, warp-item schedules as in A1) with the activation evaluated in fp32 using the MUFU
// fast path y' = (a*b) / (1 + 2^(-a*log2e)) (a*b is exact: two 8-bit significands).  |y' - y| is
// bounded by ~70 fp32 ulp for |a| <= 64, so every decision the fp32 value takes is checked with
// a +-2^-16 relative bracket and re-taken from an fp64 evaluation when the bracket straddles it:
//   * the tile scale: amax' within the bracket of a boundary 448 * 2^T -> the elements that can
//     be the true max are recomputed in fp64 before the scale is chosen;
//   * each code: if cvt(u (1 - 2^-16)) != cvt(u (1 + 2^-16)) the element is recomputed in fp64.
// Tile-rows outside the fast path's domain (|a| > 64: exp overflow range; tile amax above 2^100:
// a*b may overflow; tile amax below 2^-60: subnormal intermediates) are evaluated in fp64.
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
                                                           int64_t ld_s, int sched) {
  const int lane = threadIdx.x & 31, half = lane >> 4, sub = lane & 15;
  const int64_t rows = rows_dev != nullptr ? static_cast<int64_t>(*rows_dev) : rows_max;
  const int64_t col_pairs = (F + 255) / 256;
  const int64_t n_items = ((rows + 3) / 4) * col_pairs;  // warp item = 4 rows x 256 output columns
  const int64_t ld_h = 2 * F;
  for (ItemIter it = warp_item_iter(n_items, sched); it.cur < it.end; it.cur += it.step) {
    const int64_t item = it.cur;
    const int64_t rg = item / col_pairs;
    const int64_t cp = item - rg * col_pairs;
    const int64_t row0 = rg * 4;
    const int64_t col = cp * 256 + half * 128 + sub * 8;
    const bool col_ok = col < F;
    const int nrows = static_cast<int>(min64(4, rows - row0));
    uint32_t packed = 0;  // scale bytes of rows row0..row0+3 for this half's tile
    {
      uint4 va[4], vb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        va[i] = vb[i] = make_uint4(0, 0, 0, 0);
        if (i < nrows && col_ok) {
          const __nv_bfloat16* p = h + (row0 + i) * ld_h + col;
          va[i] = ld_nc_v4(p);
          vb[i] = ld_nc_v4(p + F);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = i;
        const uint32_t wa[4] = {va[i].x, va[i].y, va[i].z, va[i].w};
        const uint32_t wb[4] = {vb[i].x, vb[i].y, vb[i].z, vb[i].w};
        float a[8], b[8], y[8];
        uint32_t abig = 0;  // SWAR: bit 15 / 31 set where |a| > 64 (BF16 magnitude > 0x4280)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          a[2 * j] = bf16lo_to_f32(wa[j]);
          a[2 * j + 1] = bf16hi_to_f32(wa[j]);
          b[2 * j] = bf16lo_to_f32(wb[j]);
          b[2 * j + 1] = bf16hi_to_f32(wb[j]);
          abig |= (wa[j] & 0x7FFF7FFFu) + 0x3D7F3D7Fu;
        }
        // fast fp32 path; the domain where its error bound holds is checked per tile-row below
        float ymax = 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          y[j] = swiglu_fast(a[j] * b[j], a[j]);
          ymax = fmaxf(ymax, fabsf(y[j]));
        }
        uint32_t mag = halfwarp_max_u32(__float_as_uint(ymax));
        // outside |a| <= 64 and 2^-60 <= tile amax <= 2^100 (or amax exactly 0) the fp32 bound may
        // not hold (exp overflow, overflowing a*b, subnormal intermediates): the whole tile-row is
        // then evaluated in fp64
        const bool exotic = (abig & 0x80008000u) != 0u || mag > 0x71800000u || (mag != 0u && mag < 0x21800000u);
        const uint32_t exb = __ballot_sync(0xffffffffu, exotic);
        if (exb != 0u) {
          if ((exb >> (16 * half)) & 0xFFFFu) {
            float m2 = 0.0f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              y[j] = swiglu_exact(a[j], b[j]);
              m2 = fmaxf(m2, fabsf(y[j]));
            }
            mag = __float_as_uint(m2);
          }
          mag = halfwarp_max_u32(mag);
        }
        // scale decision: near the boundary amax = 1.75 * 2^e (mantissa field 0x600000)?
        const int32_t dm = static_cast<int32_t>(mag & 0x7FFFFFu) - 0x600000;
        const bool near = (mag >> 23) != 0u && dm >= -512 && dm <= 512;
        if (__any_sync(0xffffffffu, near)) {
          if (near) {
            const float thr = __uint_as_float(mag) * (1.0f - 6.103515625e-05f);  // 1 - 2^-14
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (fabsf(y[j]) >= thr) y[j] = swiglu_exact(a[j], b[j]);
            float m2 = 0.0f;
#pragma unroll
            for (int j = 0; j < 8; ++j) m2 = fmaxf(m2, fabsf(y[j]));
            mag = __float_as_uint(m2);
          }
          mag = halfwarp_max_u32(mag);
        }
        const uint32_t sb = scale_byte_from_f32_mag(mag);
        const float inv = inv_scale_from_byte(sb);
        uint32_t c[4];
        uint32_t need = 0;  // pairs whose rounding decision lies inside the error bracket
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float u0 = y[2 * j] * inv, u1 = y[2 * j + 1] * inv;
          c[j] = cvt_e4m3x2_f32(u0, u1);
          const uint32_t lo = cvt_e4m3x2_f32(u0 * kBracketLo, u1 * kBracketLo);
          const uint32_t hi = cvt_e4m3x2_f32(u0 * kBracketHi, u1 * kBracketHi);
          need |= (lo != hi ? 1u : 0u) << j;
        }
        if (__any_sync(0xffffffffu, need != 0u)) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if ((need >> j) & 1u) {  // decide in fp64
              c[j] = cvt_e4m3x2_f32(swiglu_exact(a[2 * j], b[2 * j]) * inv,
                                    swiglu_exact(a[2 * j + 1], b[2 * j + 1]) * inv);
            }
          }
        }
        if (r < nrows && col_ok) st_v2(q + (row0 + r) * F + col, c[0] | (c[1] << 16), c[2] | (c[3] << 16));
        packed |= sb << (8 * r);
      }
    }
    if (sub == 0 && col_ok) {
      uint8_t* sp = s + (cp * 2 + half) * ld_s + row0;
      if (nrows == 4) {
        *reinterpret_cast<uint32_t*>(sp) = packed;  // row0 % 4 == 0, ld_s % 16 == 0: aligned
      } else {
        for (int r = 0; r < nrows; ++r) sp[r] = static_cast<uint8_t>(packed >> (8 * r));
      }
    }
  }
}

cudaError_t launch_swiglu_quant(const void* h, int64_t rows_max, const int32_t* rows_dev, int64_t ffn, uint8_t* q,
                                uint8_t* s, int64_t ld_s, cudaStream_t stream, int num_sms) {
  static const int occ = occupancy_of(swiglu_quant_kernel, 256, 0);
  const int64_t n_items = ((rows_max + 3) / 4) * ((ffn + 255) / 256);
  const int sched = sched_for("A5", kSchedInterleaved);
  const int64_t grid = sched_grid(sched, n_items, 8, occ, num_sms);
  swiglu_quant_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(h), rows_max,
                                                                       rows_dev, ffn, q, s, ld_s, sched);
  return cudaGetLastError();
}

}  // namespace fp8flow
