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
// P:186-198): result = E4M3_RNE(decode(c) * 2^-k) -- the exponent edit E' = E - k whenever the
// result stays normal, RNE into the subnormal grid otherwise (R7).
// ------------------------------------------------------------------------------------------
// Branch-free.  The 7 magnitude bits of an E4M3 code placed at bits 7..13 of an f16 are the f16
// whose value is decode(code) * 2^-8 -- for normal AND subnormal codes (E4M3's subnormal grid
// 2^-9 maps onto f16 multiples of 2^-17, which f16 represents exactly).  So the up-conversion is
// a mask + shift (bytes 0,2 and bytes 1,3 form two f16x2), the rescale by 2^(8-k) is one HMUL2
// per pair (exact whenever the E4M3 result can be nonzero), and the single RNE rounding is the
// hardware cvt.rn.satfinite f16x2 -> e4m3x2 on magnitudes; the sign bits are re-attached
// unchanged (so an underflow to zero keeps its sign, R10).
__device__ __forceinline__ uint32_t f16x2_pow2(int e) {
  // f16x2 with both halves = 2^e, e in [-24, 8] (normal for e >= -14, subnormal below)
  const uint32_t h = e >= -14 ? static_cast<uint32_t>(e + 15) << 10 : (1u << (e + 24));
  return h | (h << 16);
}
// multiplier for shift4: 2^(8-k) as f16x2, k >= 0 (k > 32 behaves like k = 32: all results +-0)
__device__ __forceinline__ uint32_t shift_multiplier(uint32_t k) {
  const int e = 8 - static_cast<int>(k > 32u ? 32u : k);
  return f16x2_pow2(e < -24 ? -24 : e);
}
// two f16x2 (bytes 0,2 and 1,3) -> 4 E4M3 codes in byte order 0,1,2,3
__device__ __forceinline__ uint32_t cvt_e4m3x4_from_f16x2_pairs(uint32_t p02, uint32_t p13) {
  uint32_t r;
  asm("{\n\t.reg .b16 lo, hi;\n\t"
      "cvt.rn.satfinite.e4m3x2.f16x2 lo, %1;\n\t"
      "cvt.rn.satfinite.e4m3x2.f16x2 hi, %2;\n\t"
      "mov.b32 %0, {lo, hi};\n\t}"
      : "=r"(r)
      : "r"(p02), "r"(p13));
  return __byte_perm(r, 0u, 0x3120);  // [c0, c2, c1, c3] -> [c0, c1, c2, c3]
}
// nan_acc accumulates the largest f16 magnitude half seen (u16x2 max): a code of magnitude 0x7F
// (E4M3 NaN) is the only one that maps to 0x3F80, so has_nan_code() tells a caller to patch the
// (rare) words holding NaN codes with keep_nan_codes() -- NaN propagates unchanged, as in the
// oracle's shift (the f16 path alone would turn it into a finite code).
__device__ __forceinline__ uint32_t shift4(uint32_t w, uint32_t m2, uint32_t& nan_acc) {
  const uint32_t lo02 = (w & 0x007F007Fu) << 7;            // bytes 0, 2 -> f16 halves (value * 2^-8)
  const uint32_t hi13 = (w >> 1) & 0x3F803F80u;            // bytes 1, 3
  nan_acc = __vmaxu2(nan_acc, __vmaxu2(lo02, hi13));
  __half2 p02 = __hmul2(*reinterpret_cast<const __half2*>(&lo02), *reinterpret_cast<const __half2*>(&m2));
  __half2 p13 = __hmul2(*reinterpret_cast<const __half2*>(&hi13), *reinterpret_cast<const __half2*>(&m2));
  return cvt_e4m3x4_from_f16x2_pairs(*reinterpret_cast<uint32_t*>(&p02), *reinterpret_cast<uint32_t*>(&p13)) |
         (w & 0x80808080u);
}
__device__ __forceinline__ bool has_nan_code(uint32_t nan_acc) {
  return (nan_acc & 0xFFFFu) == 0x3F80u || (nan_acc >> 16) == 0x3F80u;
}
// bytes of w whose magnitude is 0x7F (NaN) replace the corresponding bytes of `shifted`
__device__ __forceinline__ uint32_t keep_nan_codes(uint32_t shifted, uint32_t w) {
  const uint32_t t = ((w & 0x7F7F7F7Fu) + 0x01010101u) & 0x80808080u;  // bit 7 of every NaN byte
  const uint32_t m = (t >> 7) * 0xFFu;
  return (shifted & ~m) | (w & m);
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

}  // namespace fp8flow
