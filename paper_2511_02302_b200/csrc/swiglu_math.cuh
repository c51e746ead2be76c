// swiglu_math.cuh -- the SwiGLU + 1x128 quantization arithmetic of A5 (fp32 MUFU fast path,
// certified scale bytes, fp64 fallback), shared by the A5 kernel (swiglu.cu) and the dual-output
// kernel (dual.cu) so that both emit identical codes.  See swiglu.cu for the error analysis.
#pragma once

#include "common.cuh"

namespace fp8flow {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float max_nan(float x, float y) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(x), "f"(y));
  return r;
}
static __device__ __noinline__ float swiglu_exact(float a, float b) {
  const double ad = static_cast<double>(a), bd = static_cast<double>(b);
  return static_cast<float>(ad * bd / (1.0 + exp(-ad)));
}

// one warp-row (lane: 4 elements) evaluated exactly; amax ignores NaN like the oracle.
// returns {codes, scale byte}
static __device__ __noinline__ uint2 swiglu_row_exact(uint2 wa, uint2 wb) {
  const float a[4] = {bf16lo_to_f32(wa.x), bf16hi_to_f32(wa.x), bf16lo_to_f32(wa.y), bf16hi_to_f32(wa.y)};
  const float b[4] = {bf16lo_to_f32(wb.x), bf16hi_to_f32(wb.x), bf16lo_to_f32(wb.y), bf16hi_to_f32(wb.y)};
  float y[4], m = 0.0f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    y[j] = swiglu_exact(a[j], b[j]);
    m = fmaxf(m, fabsf(y[j]));
  }
  const uint32_t sb = scale_byte_from_f32_mag(__reduce_max_sync(0xffffffffu, __float_as_uint(m)));
  const float inv = inv_scale_from_byte(sb);
  return make_uint2(cvt_e4m3x2_f32(y[0] * inv, y[1] * inv) | (cvt_e4m3x2_f32(y[2] * inv, y[3] * inv) << 16), sb);
}

// N warp-rows (lane l: elements 4l..4l+3 of each 128-element tile row; wa/wb = the a and b
// parts as packed BF16).  Returns the lane's packed codes of every warp-row in c[], and in the
// return value the scale byte of warp-row (lane % N) -- the N decisions are taken in parallel by
// lanes 0..N-1 and broadcast with shuffles.  Warp-uniform control flow only.
template <int N>
__device__ __forceinline__ uint32_t swiglu_quant_rows(const uint2 (&wa)[N], const uint2 (&wb)[N], uint32_t (&c)[N]) {
  static_assert(N == 4 || N == 8 || N == 16, "N warp-rows, lanes 0..N-1 decide");
  constexpr int kSwSub = N;
  const int lane = threadIdx.x & 31;
  // phase 1: fp32 values, the warp maximum |y'| of every warp-row, and whether any denominator
  // of the warp-row reaches 2^92 (a < -63.8: outside the fast path's domain).  Every decision is
  // per warp-row, so the result does not depend on how warp-rows are grouped (A5 and the
  // dual-output kernel group them differently and must agree bit for bit).
  float2 y[kSwSub][2];
  uint32_t mY[kSwSub], dom = 0;
#pragma unroll
  for (int i = 0; i < kSwSub; ++i) {
    const uint32_t aw[2] = {wa[i].x, wa[i].y}, bw[2] = {wb[i].x, wb[i].y};
    float ym = 0.0f, dm = 0.0f;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float2 a = make_float2(bf16lo_to_f32(aw[j]), bf16hi_to_f32(aw[j]));
      const float2 b = make_float2(bf16lo_to_f32(bw[j]), bf16hi_to_f32(bw[j]));
      const float2 x = __fmul2_rn(a, make_float2(-kLog2e, -kLog2e));
      const float2 d = __fadd2_rn(make_float2(ex2_approx(x.x), ex2_approx(x.y)), make_float2(1.0f, 1.0f));
      y[i][j] = __fmul2_rn(__fmul2_rn(a, b), make_float2(rcp_approx(d.x), rcp_approx(d.y)));
      ym = max_nan(ym, max_nan(fabsf(y[i][j].x), fabsf(y[i][j].y)));
      dm = max_nan(dm, max_nan(d.x, d.y));
    }
    mY[i] = __reduce_max_sync(0xffffffffu, __float_as_uint(ym));
    dom |= (__any_sync(0xffffffffu, !(dm < 4.951760157141521e27f)) ? 1u : 0u) << i;  // NaN: via amax'
  }
  // phase 2: lanes 0..N-1 take the N scale decisions (lane k: warp-row k), then broadcast
  const int r = lane & (kSwSub - 1);
  uint32_t my = mY[0];
#pragma unroll
  for (int i = 1; i < kSwSub; ++i) my = r == i ? mY[i] : my;
  // domain: amax 0 or in [2^-60, 2^100] (NaN fails), denominators < 2^92
  const bool exotic = ((dom >> r) & 1u) != 0u || (my != 0u && my - 0x21800000u > 0x50000000u);
  // near a scale boundary amax = 1.75 * 2^e (mantissa field 0x600000) within 2^-14?
  const int32_t dmant = static_cast<int32_t>(my & 0x7FFFFFu) - 0x600000;
  const bool sure = !exotic && !(dmant >= -512 && dmant <= 512);
  uint32_t sbyte = scale_byte_from_f32_mag(my);
  const float inv = inv_scale_from_byte(sbyte);
#pragma unroll
  for (int i = 0; i < kSwSub; ++i) {
    const float iv = __shfl_sync(0xffffffffu, inv, i);
    const float2 u0 = __fmul2_rn(y[i][0], make_float2(iv, iv)), u1 = __fmul2_rn(y[i][1], make_float2(iv, iv));
    c[i] = cvt_e4m3x2_f32(u0.x, u0.y) | (cvt_e4m3x2_f32(u1.x, u1.y) << 16);
  }
  const uint32_t unsure = __ballot_sync(0xffffffffu, !sure) & ((1u << kSwSub) - 1u);
  if (unsure != 0u) {  // rare, warp-uniform: whole warp-rows in fp64
#pragma unroll
    for (int i = 0; i < kSwSub; ++i) {
      if ((unsure >> i) & 1u) {
        const uint2 x = swiglu_row_exact(wa[i], wb[i]);
        c[i] = x.x;
        if (r == i) sbyte = x.y;
      }
    }
  }
  return sbyte;
}

}  // namespace fp8flow
