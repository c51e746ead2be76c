// quantize.cu -- A1: entry BF16 -> E4M3 quantization with 1x128 power-of-two scales.
//
// Paper: Eq. 2 (tile scale), Eq. 3 (code = round(x / s)), power-of-two scales
// s = 2^T, "no explicit casting except at the entry point".
//
// HBM-bound streaming op (3.008 B/element).  The r01 kernel spent 707 warp-instructions per 2048
// elements (issue slots 72 % busy at 4096 x 7168); this one ~0.2 per element:
//   * a 1x128 tile row is held by 8 lanes, 16 consecutive BF16 per lane (two 128-bit loads), so
//     every scale decision is amortised over 16 elements per lane;
//   * warp item = 8 rows x 256 columns (lanes 8r..8r+7: rows r and r + 4 of two adjacent tiles),
//     all 8 loads (4 KB per warp) issued before any use; one item per warp, 4-warp CTAs, so the
//     hardware CTA scheduler sweeps the tensor in address order with ~128 KB in flight per SM
//     (r02 marginal cold-L2 times, tools/probe/marginal_a1.py: 4096 x 7168 16.2 -> 14.1 us,
//     16384 x 7168 53.4 -> 48.7 us, 65536 x 7168 209 -> 200 us; a persistent blocked or
//     interleaved schedule was 5-20 % slower at the large shapes);
//   * in-lane |max| by 7 packed bf16x2 `max.xorsign.abs` (HMNMX2), the 8-lane max by 3 butterfly
//     shuffles on the 15-bit magnitude;
//   * the scale byte and 2^-T straight from the amax bit pattern: T + 127 = max(((mag + 0x1F) >> 7)
//     - 8, 0) (the +0x1F carries into the exponent exactly when the 7-bit mantissa exceeds 0x60,
//     i.e. amax > 1.75 * 2^e = 448 * 2^(e-8)); zero / subnormal amax -> byte 0 (R11, R13);
//   * x * 2^-T exact in fp32 (packed f32x2 multiplies), cvt.rn.satfinite.e4m3x2 (the single RNE),
//     16 codes per lane leave as one 128-bit store, the row's scale byte from its first lane.
#include "common.cuh"
#include "kernels.h"

namespace fp8flow {

namespace {

constexpr int kA1Warps = 4;  // 128-thread CTAs (8-warp CTAs measured equal)

// one 1x128 tile row held by 8 lanes (16 BF16 each): common.cuh a1_quant16, then the stores
__device__ __forceinline__ void a1_tile_row(const uint4 (&v)[2], int lane, bool ok, uint8_t* pq, uint8_t* ps) {
  const uint32_t w[8] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y, v[1].z, v[1].w};
  uint32_t c[8];
  const uint32_t sb = a1_quant16(w, c);
  if (ok) {
    st_v4(pq, make_uint4(c[0] | (c[1] << 16), c[2] | (c[3] << 16), c[4] | (c[5] << 16), c[6] | (c[7] << 16)));
    if ((lane & 7) == 0) *ps = static_cast<uint8_t>(sb);
  }
}

// one warp = 8 rows x 256 columns: lanes 8r..8r+7 take rows r and r + 4 of two adjacent tiles
template <int WARPS>
__global__ void __launch_bounds__(32 * WARPS) quantize_rowwise_kernel(const __nv_bfloat16* __restrict__ x, int64_t rows,
                                                                 int64_t cols, uint8_t* __restrict__ q,
                                                                 uint8_t* __restrict__ s, int64_t ld_s) {
  const int lane = threadIdx.x & 31;
  const int r_in = lane >> 3, c16 = (lane & 7) * 16;
  const int64_t n_tiles = cols / kTile;
  const int64_t n_pairs = (n_tiles + 1) / 2;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * WARPS + (threadIdx.x >> 5);
  const int64_t rg = item / n_pairs;                 // 8-row group
  const int64_t tp = item - rg * n_pairs;
  const int64_t row0 = rg * 8 + r_in;
  if (rg * 8 >= rows) return;
  uint4 v[2][2][2];                                  // [row half][tile][2 loads]
  bool ok[2][2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int64_t row = row0 + 4 * h, tj = tp * 2 + t;
      ok[h][t] = row < rows && tj < n_tiles;
      const __nv_bfloat16* p = x + row * cols + tj * kTile + c16;
      if (ok[h][t]) {
        v[h][t][0] = ld_nc_v4(p);
        v[h][t][1] = ld_nc_v4(p + 8);
      }
    }
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int64_t row = row0 + 4 * h, tj = tp * 2 + t;
      a1_tile_row(v[h][t], lane, ok[h][t], q + row * cols + tj * kTile + c16, s + tj * ld_s + row);
    }
}

}  // namespace

cudaError_t launch_quantize_rowwise(const void* x, int64_t rows, int64_t cols, uint8_t* q, uint8_t* s,
                                    int64_t ld_s, cudaStream_t stream, int num_sms) {
  (void)num_sms;  // one warp item per warp; the hardware CTA scheduler balances and sweeps in order
  const int64_t n_items = ((rows + 7) / 8) * ((cols / kTile + 1) / 2);
  const int64_t grid = (n_items + kA1Warps - 1) / kA1Warps;
  if (grid > 0x7FFFFFFFLL) return cudaErrorInvalidValue;
  quantize_rowwise_kernel<kA1Warps><<<static_cast<unsigned>(grid), 32 * kA1Warps, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(x), rows, cols, q, s, ld_s);
  return cudaGetLastError();
}

}  // namespace fp8flow
