// quantize.cu -- A1: entry BF16 -> E4M3 quantization with 1x128 power-of-two scales.
//
// Paper: Eq. 2 (tile scale), Eq. 3 (code = round(x / s)), power-of-two scales
// s = 2^T, "no explicit casting except at the entry point".
//
// Work decomposition (HBM-bound streaming op, 3.008 B/element):
//   warp item = 8 consecutive rows x 256 columns (two 1x128 tiles), one item per warp; the warp
//   issues its 8 row loads (8 x 16 B per lane) before using any.  A half-warp owns one tile row:
//   in-thread max over 8 BF16 magnitudes as packed 16-bit pairs, the tile amax by two full-warp
//   redux.sync (one per half), the scale byte from the amax bit pattern (exact integer rule),
//   x * 2^-T exact in fp32 (packed f32x2 multiplies), cvt.rn.satfinite packs the codes.  The 8
//   scale bytes of a warp's rows are contiguous in the MN-major layout s[tile][row] and leave as
//   two 32-bit stores per tile.
#include "common.cuh"
#include "kernels.h"

namespace fp8flow {

template <int ROWS>
__device__ __forceinline__ void a1_load(const __nv_bfloat16* __restrict__ x, int64_t rows, int64_t cols,
                                        int64_t col_pairs, int64_t item, int half, int sub, uint4 (&v)[ROWS]) {
  const int64_t rg = item / col_pairs;
  const int64_t cp = item - rg * col_pairs;
  const int64_t row0 = rg * ROWS;
  const int64_t col = cp * 256 + half * 128 + sub * 8;
  const bool col_ok = col < cols;
  const int nrows = static_cast<int>(min64(ROWS, rows - row0));
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    v[r] = make_uint4(0, 0, 0, 0);
    if (r < nrows && col_ok) v[r] = ld_nc_v4(x + (row0 + r) * cols + col);
  }
}

// v2 of the per-item math (the default): the tile max of a half-warp by two
// full-warp redux.sync (each half contributes to its own), magnitudes max'ed as packed 16-bit
// pairs (__vmaxu2 on w & 0x7FFF7FFF), x * 2^-T as packed f32x2 multiplies (FMUL2).  Same results:
// max over |bf16| bit patterns, exact power-of-two scaling, one RNE per element.
template <int ROWS>
__device__ __forceinline__ void a1_process_v2(int64_t rows, int64_t cols, int64_t col_pairs, int64_t item, int half,
                                              int sub, const uint4 (&v)[ROWS], uint8_t* __restrict__ q,
                                              uint8_t* __restrict__ s, int64_t ld_s) {
  const int64_t rg = item / col_pairs;
  const int64_t cp = item - rg * col_pairs;
  const int64_t row0 = rg * ROWS;
  const int64_t col = cp * 256 + half * 128 + sub * 8;
  const bool col_ok = col < cols;
  const int nrows = static_cast<int>(min64(ROWS, rows - row0));
  uint32_t packed[ROWS / 4];
#pragma unroll
  for (int i = 0; i < ROWS / 4; ++i) packed[i] = 0;
  uint8_t* qrow = q + row0 * cols + col;
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    const uint32_t w[4] = {v[r].x, v[r].y, v[r].z, v[r].w};
    uint32_t m2 = __vmaxu2(__vmaxu2(w[0] & 0x7FFF7FFFu, w[1] & 0x7FFF7FFFu),
                           __vmaxu2(w[2] & 0x7FFF7FFFu, w[3] & 0x7FFF7FFFu));
    const uint32_t m = max(m2 & 0xFFFFu, m2 >> 16);
    const uint32_t lo = __reduce_max_sync(0xffffffffu, half ? 0u : m);
    const uint32_t hi = __reduce_max_sync(0xffffffffu, half ? m : 0u);
    const uint32_t sb = scale_byte_from_bf16_mag(half ? hi : lo);
    const float inv = inv_scale_from_byte(sb);
    const float2 iv = make_float2(inv, inv);
    uint32_t c[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 p = __fmul2_rn(make_float2(bf16lo_to_f32(w[j]), bf16hi_to_f32(w[j])), iv);
      c[j] = cvt_e4m3x2_f32(p.x, p.y);
    }
    if (r < nrows && col_ok) st_v2(qrow + r * cols, c[0] | (c[1] << 16), c[2] | (c[3] << 16));
    packed[r / 4] |= sb << (8 * (r % 4));
  }
  if (sub == 0 && col_ok) {
    uint8_t* sp = s + (cp * 2 + half) * ld_s + row0;
    if (nrows == ROWS) {
#pragma unroll
      for (int i = 0; i < ROWS / 4; ++i) reinterpret_cast<uint32_t*>(sp)[i] = packed[i];
    } else {
      for (int r = 0; r < nrows; ++r) sp[r] = static_cast<uint8_t>(packed[r / 4] >> (8 * (r % 4)));
    }
  }
}

template <int ROWS, int WARPS = 8>
__global__ void __launch_bounds__(32 * WARPS) quantize_rowwise_v2_kernel(const __nv_bfloat16* __restrict__ x, int64_t rows,
                                                                   int64_t cols, uint8_t* __restrict__ q,
                                                                   uint8_t* __restrict__ s, int64_t ld_s) {
  const int lane = threadIdx.x & 31;
  const int half = lane >> 4;
  const int sub = lane & 15;
  const int64_t col_pairs = (cols + 255) / 256;
  const int64_t n_items = ((rows + ROWS - 1) / ROWS) * col_pairs;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * WARPS + (threadIdx.x >> 5);  // one item per warp
  if (item >= n_items) return;
  uint4 v[ROWS];
  a1_load<ROWS>(x, rows, cols, col_pairs, item, half, sub, v);
  a1_process_v2<ROWS>(rows, cols, col_pairs, item, half, sub, v, q, s, ld_s);
}

cudaError_t launch_quantize_rowwise(const void* x, int64_t rows, int64_t cols, uint8_t* q, uint8_t* s,
                                    int64_t ld_s, cudaStream_t stream, int num_sms) {
  // 8-row items, one per warp, 4 warps per CTA (DESIGN.md §6/§9)
  const int64_t n_items = ((rows + 7) / 8) * ((cols + 255) / 256);
  quantize_rowwise_v2_kernel<8, 4><<<static_cast<unsigned>((n_items + 3) / 4), 128, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(x), rows, cols, q, s, ld_s);
  return cudaGetLastError();
}

}  // namespace fp8flow
