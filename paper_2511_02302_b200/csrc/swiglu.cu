// swiglu.cu -- A5: fused SwiGLU + 1x128 power-of-two E4M3 quantization.
//
// Paper: P:380-381 ("we fuse the SwiGLU activation and quantization steps into a single kernel"),
// BF16 input from the first BF16 boundary, tile scale Eq. 2, codes Eq. 3.
// Readings: R18 a = h[:, :F] is gated (silu), b = h[:, F:] linear; R20 the
// reference value is a*b / (1 + e^-a) evaluated in fp64 and rounded once to fp32 (oracle C10);
// acceptance: codes within 1 E4M3 ULP on <= 1e-4 of elements, scale bytes identical.
//
// Kernel: TMA-fed producer/consumer pipeline (below), half-warp per 1x128 output tile row, with the
// activation evaluated in fp32 using the MUFU
// fast path y' = (a*b) / (1 + 2^(-a*log2e)) (a*b is exact: two 8-bit significands).  |y' - y| is
// bounded by ~70 fp32 ulp for |a| <= 64, so every decision the fp32 value takes is checked with
// a +-2^-16 relative bracket and re-taken from an fp64 evaluation when the bracket straddles it:
//   * the tile scale: amax' within the bracket of a boundary 448 * 2^T -> the elements that can
//     be the true max are recomputed in fp64 before the scale is chosen;
//   * each code: if cvt(u (1 - 2^-16)) != cvt(u (1 + 2^-16)) the element is recomputed in fp64.
// Tile-rows outside the fast path's domain (|a| > 64: exp overflow range; tile amax above 2^100:
// a*b may overflow; tile amax below 2^-60: subnormal intermediates) are evaluated in fp64.
#include <cuda.h>

#include "async.cuh"
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
__device__ __noinline__ float swiglu_exact(float a, float b) {
  const double ad = static_cast<double>(a), bd = static_cast<double>(b);
  return static_cast<float>(ad * bd / (1.0 + exp(-ad)));
}

// ---------------------------------------------------------------------------------------------
// Kernel structure: one CTA per SM, warp 0 = TMA producer, warps 1-16 = consumers.
// A tile = 64 rows x 256 output columns: the a-part h[r][c..c+255] and the b-part
// h[r][F+c..F+c+255] arrive as two 2-D TMA boxes (32 KB each) in a 3-stage mbarrier ring, so up to
// 192 KB per SM are in flight while the consumers compute.  Consumer warp w owns rows 4w..4w+3 of
// the tile; a half-warp owns one 1x128 output tile row (16 lanes x 8 elements).
// ---------------------------------------------------------------------------------------------
constexpr int kSwCols = 256;  // output columns per TMA tile
constexpr int kSwStages = 3;

// CONS consumer warps (4 rows each) -> tiles of 4*CONS rows; CONS = 16: one CTA per SM (192 KB of
// stages), CONS = 8: two CTAs per SM (96 KB each) so that another kernel's CTA can co-reside
template <int CONS>
struct SwigluSmem {
  static constexpr int kRows = 4 * CONS;
  static constexpr int kBox = kRows * kSwCols * 2;  // bytes of one box (a or b part)
  uint8_t a[kSwStages][kBox];
  uint8_t b[kSwStages][kBox];
  uint64_t full[kSwStages];
  uint64_t empty[kSwStages];
};

__device__ __forceinline__ void swiglu_tile_row(const uint4& va, const uint4& vb, int lane, int half,
                                                uint32_t (&c)[4], uint32_t& sb_out) {
  const uint32_t wa[4] = {va.x, va.y, va.z, va.w};
  const uint32_t wb[4] = {vb.x, vb.y, vb.z, vb.w};
  float a[8], b[8], y[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    a[2 * j] = bf16lo_to_f32(wa[j]);
    a[2 * j + 1] = bf16hi_to_f32(wa[j]);
    b[2 * j] = bf16lo_to_f32(wb[j]);
    b[2 * j + 1] = bf16hi_to_f32(wb[j]);
  }
  // fast fp32 path: y' = a*b / (1 + 2^(-a log2e)); the domain where its error bound holds is
  // checked per tile-row below (the largest denominator flags a < -64)
  float ymax = 0.0f, dmax = 0.0f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float d = 1.0f + ex2_approx(-a[j] * kLog2e);
    y[j] = __fdividef(a[j] * b[j], d);
    ymax = fmaxf(ymax, fabsf(y[j]));
    dmax = fmaxf(dmax, d);
  }
  uint32_t mag = halfwarp_max_u32(__float_as_uint(ymax));
  // outside |a| <= 64 and 2^-60 <= tile amax <= 2^100 (or amax exactly 0) the fp32 bound may not
  // hold (exp overflow, overflowing a*b, subnormal intermediates): the tile-row is evaluated in fp64
  const bool exotic = !(dmax < 5.0e27f) || mag > 0x71800000u || (mag != 0u && mag < 0x21800000u);  // 2^92
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
  // codes: the true u = y * 2^-T lies in [y'(1-2^-16), y'(1+2^-16)] * 2^-T; if both ends round to
  // the same E4M3 code that code is exact, otherwise the pair is decided in fp64
  const float inv_lo = inv * kBracketLo, inv_hi = inv * kBracketHi;
  uint32_t need = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t lo = cvt_e4m3x2_f32(y[2 * j] * inv_lo, y[2 * j + 1] * inv_lo);
    const uint32_t hi = cvt_e4m3x2_f32(y[2 * j] * inv_hi, y[2 * j + 1] * inv_hi);
    c[j] = lo;
    need |= (lo != hi ? 1u : 0u) << j;
  }
  if (__any_sync(0xffffffffu, need != 0u)) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if ((need >> j) & 1u) {  // decide in fp64
        c[j] = cvt_e4m3x2_f32(swiglu_exact(a[2 * j], b[2 * j]) * inv, swiglu_exact(a[2 * j + 1], b[2 * j + 1]) * inv);
      }
    }
  }
  (void)lane;
  sb_out = sb;
}

template <int CONS>
__global__ void __launch_bounds__(32 * (1 + CONS), 1)
    swiglu_quant_kernel(const __grid_constant__ CUtensorMap tmap_h, int64_t rows_max,
                        const int32_t* __restrict__ rows_dev, int64_t F, uint8_t* __restrict__ q,
                        uint8_t* __restrict__ s, int64_t ld_s) {
  extern __shared__ __align__(1024) uint8_t smem_sw[];
  using Smem = SwigluSmem<CONS>;
  constexpr int kSwRows = Smem::kRows;
  constexpr int kSwBox = Smem::kBox;
  Smem& sm = *reinterpret_cast<Smem*>(smem_sw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rows = rows_dev != nullptr ? static_cast<int64_t>(*rows_dev) : rows_max;
  const int col_tiles = static_cast<int>((F + kSwCols - 1) / kSwCols);
  const int64_t n_tiles = ((rows + kSwRows - 1) / kSwRows) * col_tiles;
  if (tid == 0) {
    for (int i = 0; i < kSwStages; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], CONS);
    }
    mbar_init_fence();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_h)) : "memory");
  }
  __syncthreads();

  if (warp == 0) {  // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int st = 0;
      uint32_t parity = 0;
      int64_t n = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++n) {
        if (n >= kSwStages) mbar_wait(&sm.empty[st], parity ^ 1u);
        const int64_t rg = t / col_tiles;
        const int c0 = static_cast<int>(t - rg * col_tiles) * kSwCols;
        mbar_expect_tx(&sm.full[st], 2 * kSwBox);
        tma_load_2d(sm.a[st], &tmap_h, &sm.full[st], c0, static_cast<int32_t>(rg * kSwRows));
        tma_load_2d(sm.b[st], &tmap_h, &sm.full[st], static_cast<int32_t>(F) + c0, static_cast<int32_t>(rg * kSwRows));
        if (++st == kSwStages) {
          st = 0;
          parity ^= 1u;
        }
      }
    }
    return;
  }
  // ------------------------------------------------------------------------ consumers
  const int cw = warp - 1;  // rows 4cw..4cw+3 of each tile
  const int half = lane >> 4, sub = lane & 15;
  int st = 0;
  uint32_t parity = 0;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const int64_t rg = t / col_tiles;
    const int64_t c0 = (t - rg * col_tiles) * kSwCols;
    const int64_t col = c0 + half * 128 + sub * 8;
    const bool col_ok = col < F;
    const int64_t row0 = rg * kSwRows + 4 * cw;
    const int nrows = static_cast<int>(min64(4, rows - row0));
    mbar_wait(&sm.full[st], parity);
    uint4 va[4], vb[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int off = ((4 * cw + i) * kSwCols + half * 128 + sub * 8) * 2;
      va[i] = *reinterpret_cast<const uint4*>(&sm.a[st][off]);
      vb[i] = *reinterpret_cast<const uint4*>(&sm.b[st][off]);
    }
    fence_proxy_async_smem();  // reads (generic proxy) before the next TMA write (async proxy)
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[st]);  // stage data is in registers: release it
    if (++st == kSwStages) {
      st = 0;
      parity ^= 1u;
    }
    uint32_t packed = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t c[4], sb;
      swiglu_tile_row(va[i], vb[i], lane, half, c, sb);
      if (i < nrows && col_ok) st_v2(q + (row0 + i) * F + col, c[0] | (c[1] << 16), c[2] | (c[3] << 16));
      packed |= sb << (8 * i);
    }
    if (sub == 0 && col_ok && nrows > 0) {
      uint8_t* sp = s + (col / 128) * ld_s + row0;
      if (nrows == 4) {
        *reinterpret_cast<uint32_t*>(sp) = packed;  // row0 % 4 == 0, ld_s % 16 == 0: aligned
      } else {
        for (int r = 0; r < nrows; ++r) sp[r] = static_cast<uint8_t>(packed >> (8 * r));
      }
    }
  }
}

typedef CUresult (*PFN_encodeTiled_sw)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

cudaError_t launch_swiglu_quant(const void* h, int64_t rows_max, const int32_t* rows_dev, int64_t ffn, uint8_t* q,
                                uint8_t* s, int64_t ld_s, cudaStream_t stream, int num_sms) {
  static PFN_encodeTiled_sw encode = nullptr;
  if (!encode) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qres;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qres) != cudaSuccess ||
        qres != cudaDriverEntryPointSuccess)
      return cudaErrorNotSupported;
    encode = reinterpret_cast<PFN_encodeTiled_sw>(p);
    cudaFuncSetAttribute(swiglu_quant_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(SwigluSmem<16>)));
    cudaFuncSetAttribute(swiglu_quant_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(SwigluSmem<8>)));
  }
  const int ctas = tune_int("CTAS_PER_SM_A5", 1) >= 2 ? 2 : 1;
  const int rows_per_tile = ctas == 2 ? SwigluSmem<8>::kRows : SwigluSmem<16>::kRows;
  CUtensorMap map;
  const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(2 * ffn), static_cast<cuuint64_t>(rows_max)};
  const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(4 * ffn)};
  const cuuint32_t box[2] = {kSwCols, static_cast<cuuint32_t>(rows_per_tile)};
  const cuuint32_t estride[2] = {1, 1};
  if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(h), gdim, gstride, box, estride,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const int64_t tiles_ub = ((rows_max + rows_per_tile - 1) / rows_per_tile) * ((ffn + kSwCols - 1) / kSwCols);
  const int64_t max_grid = static_cast<int64_t>(num_sms) * ctas;
  int64_t grid = tiles_ub < max_grid ? tiles_ub : max_grid;
  if (grid < 1) grid = 1;
  if (ctas == 2)
    swiglu_quant_kernel<8><<<static_cast<unsigned>(grid), 32 * 9, sizeof(SwigluSmem<8>), stream>>>(
        map, rows_max, rows_dev, ffn, q, s, ld_s);
  else
    swiglu_quant_kernel<16><<<static_cast<unsigned>(grid), 32 * 17, sizeof(SwigluSmem<16>), stream>>>(
        map, rows_max, rows_dev, ffn, q, s, ld_s);
  return cudaGetLastError();
}

}  // namespace fp8flow
