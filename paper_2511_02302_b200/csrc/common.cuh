// common.cuh -- device helpers shared by the sm_100a kernels of libfp8flow.
//
// Numeric contract (readings R3/R8-R13): E4M3 codes with RNE + satfinite + signed
// zero (the hardware cvt.rn.satfinite behaviour); UE8M0 scale bytes = T + 127 where T is the
// least integer with amax <= 448 * 2^T, clamped to [-127, 127]; amax = 0 -> byte 0.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace fp8flow {

constexpr int kTile = 128;  // 1x128 scaling tiles and 128x128 transpose blocks

// ------------------------------------------------------------------------------------------
// E4M3 conversions (PTX cvt; SASS F2FP).  In the e4m3x2 packing the first-listed source lands in
// the UPPER byte, so (lo, hi) are swapped on the way in to keep memory order = element order.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cvt_e4m3x2_f32(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t cvt_f16x2_from_e4m3x2(uint32_t two_codes) {
  uint32_t r;
  uint16_t v = static_cast<uint16_t>(two_codes);
  asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(r) : "h"(v));
  return r;
}
__device__ __forceinline__ uint32_t cvt_e4m3x2_from_f16x2(uint32_t h2) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f16x2 %0, %1;" : "=h"(r) : "r"(h2));
  return r;
}

// UE8M0 scale byte from the bit pattern of a non-negative amax.
//   BF16 amax (15-bit magnitude):  byte = expfield - 8 + [mant7 > 0x60], clamped at 0
//   fp32 amax (31-bit magnitude):  byte = expfield - 8 + [mant23 > 0x600000], clamped at 0
// (T = e - 8 + [m > 0.75]: amax <= 1.75 * 2^e = 448 * 2^(e-8); zero/subnormal -> T = -127.)
__device__ __forceinline__ uint32_t scale_byte_from_bf16_mag(uint32_t mag) {
  int ef = static_cast<int>(mag >> 7);
  int b = ef - 8 + ((mag & 0x7Fu) > 0x60u ? 1 : 0);
  b = ef == 0 ? 0 : b;
  return static_cast<uint32_t>(b < 0 ? 0 : b);
}
__device__ __forceinline__ uint32_t scale_byte_from_f32_mag(uint32_t mag) {
  int ef = static_cast<int>(mag >> 23);
  int b = ef - 8 + ((mag & 0x7FFFFFu) > 0x600000u ? 1 : 0);
  b = ef == 0 ? 0 : b;
  b = b > 254 ? 254 : b;
  return static_cast<uint32_t>(b < 0 ? 0 : b);
}
// 2^-T as fp32 for a scale byte (T = byte - 127); exact for bytes 0..253.
__device__ __forceinline__ float inv_scale_from_byte(uint32_t byte) {
  return __uint_as_float((254u - byte) << 23);
}
// 2^T as fp32 for a scale byte; byte 0 (T = -127) is the fp32 subnormal 2^-127.
__device__ __forceinline__ float scale_from_byte(uint32_t byte) {
  return byte == 0 ? __uint_as_float(0x00400000u) : __uint_as_float(byte << 23);
}

__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// half-warp (16 lanes) max reduction; every lane of the half receives the result
__device__ __forceinline__ uint32_t halfwarp_max_u32(uint32_t v) {
  v = max(v, __shfl_xor_sync(0xffffffffu, v, 8));
  v = max(v, __shfl_xor_sync(0xffffffffu, v, 4));
  v = max(v, __shfl_xor_sync(0xffffffffu, v, 2));
  v = max(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return v;
}

// ------------------------------------------------------------------------------------------
// Exponent shift of 4 packed codes of one row by the same k >= 0 (derivation after Eq. 11,
// P:186-198): result = E4M3_RNE(decode(code) * 2^-k) -- the exponent edit E' = E - k whenever the
// result stays normal, RNE into the subnormal grid otherwise (R7).
// ------------------------------------------------------------------------------------------
// Branch-free, 8 instructions per 4 codes: the hardware decode e4m3x2 -> f16x2 (exact: E4M3 is a
// subset of f16, subnormals included), one HMUL2 by 2^-k per pair (exact whenever the E4M3 result
// can be nonzero: the product keeps its 4 significant bits down to 2^-21, far below the 2^-10
// rounding threshold of E4M3's smallest subnormal), the single RNE rounding by the hardware
// cvt.rn.satfinite f16x2 -> e4m3x2, and the sign bits OR-ed back (an underflow to zero keeps its
// sign, R10; a NaN code 0x7F / 0xFF comes back as the same byte, as in the oracle's shift).
__device__ __forceinline__ uint32_t f16x2_pow2(int e) {
  // f16x2 with both halves = 2^e, e in [-24, 15] (normal for e >= -14, subnormal below); 0 below
  const uint32_t h = e >= -14 ? static_cast<uint32_t>(e + 15) << 10 : (e >= -24 ? (1u << (e + 24)) : 0u);
  return h | (h << 16);
}
// multiplier for shift4: 2^-k as f16x2 (k > 24: 0, every result is +-0)
__device__ __forceinline__ uint32_t shift_multiplier(uint32_t k) {
  return f16x2_pow2(-static_cast<int>(k > 25u ? 25u : k));
}
__device__ __forceinline__ uint32_t shift4(uint32_t w, uint32_t m2) {
  uint32_t h01, h23, r;
  asm("{\n\t.reg .b16 lo, hi;\n\t"
      "mov.b32 {lo, hi}, %2;\n\t"
      "cvt.rn.f16x2.e4m3x2 %0, lo;\n\t"
      "cvt.rn.f16x2.e4m3x2 %1, hi;\n\t}"
      : "=r"(h01), "=r"(h23)
      : "r"(w));
  __half2 p01 = __hmul2(*reinterpret_cast<const __half2*>(&h01), *reinterpret_cast<const __half2*>(&m2));
  __half2 p23 = __hmul2(*reinterpret_cast<const __half2*>(&h23), *reinterpret_cast<const __half2*>(&m2));
  asm("{\n\t.reg .b16 lo, hi;\n\t"
      "cvt.rn.satfinite.e4m3x2.f16x2 lo, %1;\n\t"
      "cvt.rn.satfinite.e4m3x2.f16x2 hi, %2;\n\t"
      "mov.b32 %0, {lo, hi};\n\t}"
      : "=r"(r)
      : "r"(*reinterpret_cast<uint32_t*>(&p01)), "r"(*reinterpret_cast<uint32_t*>(&p23)));
  return r | (w & 0x80808080u);
}

// ------------------------------------------------------------------------------------------
// memory helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_v2(void* p, uint32_t a, uint32_t b) {
  asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}

__device__ __forceinline__ float bf16lo_to_f32(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi_to_f32(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// per bf16 half: max(|a|, |b|), sign bit = xor of the signs (callers mask it off)
__device__ __forceinline__ uint32_t absmax_bf16x2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// A1's arithmetic (Eq. 2-3, power-of-two scales P:173-175) for one 1x128 tile row held
// by 8 consecutive lanes (8k..8k+7), 16 BF16 per lane in w (any split of the row's columns): exact
// |amax| by 7 packed max.xorsign.abs, 3 butterfly shuffles on the 15-bit magnitude, scale byte
// T + 127 = max(((mag + 0x1F) >> 7) - 8, 0) (the +0x1F carries into the exponent exactly when the
// 7-bit mantissa exceeds 0x60), codes RNE(x * 2^-T) (the product is exact).  c[j]: the two codes of
// w[j] (low byte = low half).  Returns the scale byte (zero / subnormal amax -> 0, R11, R13).
__device__ __forceinline__ uint32_t a1_quant16(const uint32_t (&w)[8], uint32_t (&c)[8]) {
  const uint32_t m = absmax_bf16x2(absmax_bf16x2(absmax_bf16x2(w[0], w[1]), absmax_bf16x2(w[2], w[3])),
                                   absmax_bf16x2(absmax_bf16x2(w[4], w[5]), absmax_bf16x2(w[6], w[7])));
  uint32_t mag = max(m & 0x7FFFu, (m >> 16) & 0x7FFFu);
  mag = max(mag, __shfl_xor_sync(0xffffffffu, mag, 1));
  mag = max(mag, __shfl_xor_sync(0xffffffffu, mag, 2));
  mag = max(mag, __shfl_xor_sync(0xffffffffu, mag, 4));
  const int sb = max(static_cast<int>((mag + 0x1Fu) >> 7) - 8, 0);
  const float inv = __uint_as_float(static_cast<uint32_t>(254 - sb) << 23);
  const float2 iv = make_float2(inv, inv);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float2 p = __fmul2_rn(make_float2(bf16lo_to_f32(w[j]), bf16hi_to_f32(w[j])), iv);
    c[j] = cvt_e4m3x2_f32(p.x, p.y);
  }
  return static_cast<uint32_t>(sb);
}

}  // namespace fp8flow
