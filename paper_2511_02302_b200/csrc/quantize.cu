// quantize.cu -- A1: entry BF16 -> E4M3 quantization with 1x128 power-of-two scales.
//
// Paper: Eq. 2 (tile scale), Eq. 3 (code = round(x / s)), power-of-two scales
// s = 2^T, "no explicit casting except at the entry point".
//
// Work decomposition (HBM-bound streaming op, 3.008 B/element):
//   warp item = 4 consecutive rows x 256 columns (two 1x128 tiles); the warp issues its 4 row
//   loads (4 x 16 B per lane) before using any.  A half-warp owns one tile row:
//   in-thread max over 8 BF16 magnitudes, 4 xor-shuffles give the tile amax, the scale byte comes
//   from the amax bit pattern (exact integer rule), x * 2^-T is exact in fp32, and
//   cvt.rn.satfinite packs the codes.  The 4 scale bytes of a warp's rows are contiguous in the
//   MN-major layout s[tile][row] and leave as one 32-bit store per tile.  Items are scheduled per
//   warp (Sched in common.cuh; tuned default in the launcher).
#include "common.cuh"
#include "kernels.h"

namespace fp8flow {

constexpr int kQuantRows = 4;  // rows per warp item (a warp item = 4 rows x 256 columns)

__global__ void __launch_bounds__(256) quantize_rowwise_kernel(const __nv_bfloat16* __restrict__ x, int64_t rows,
                                                                int64_t cols, uint8_t* __restrict__ q,
                                                                uint8_t* __restrict__ s, int64_t ld_s, int sched) {
  const int lane = threadIdx.x & 31;
  const int half = lane >> 4;
  const int sub = lane & 15;
  const int64_t col_pairs = (cols + 255) / 256;
  const int64_t n_items = ((rows + kQuantRows - 1) / kQuantRows) * col_pairs;
  for (ItemIter it = warp_item_iter(n_items, sched); it.cur < it.end; it.cur += it.step) {
    const int64_t item = it.cur;
    const int64_t rg = item / col_pairs;
    const int64_t cp = item - rg * col_pairs;
    const int64_t row0 = rg * kQuantRows;
    const int64_t col = cp * 256 + half * 128 + sub * 8;
    const bool col_ok = col < cols;  // odd number of tiles: upper half idles on the last pair
    const int nrows = static_cast<int>(min64(kQuantRows, rows - row0));
    uint4 v[kQuantRows];
#pragma unroll
    for (int r = 0; r < kQuantRows; ++r) {
      v[r] = make_uint4(0, 0, 0, 0);
      if (r < nrows && col_ok) v[r] = ld_nc_v4(x + (row0 + r) * cols + col);
    }
    uint32_t packed = 0;  // scale bytes of rows row0..row0+3 for this half's tile
#pragma unroll
    for (int r = 0; r < kQuantRows; ++r) {
      const uint32_t w[4] = {v[r].x, v[r].y, v[r].z, v[r].w};
      uint32_t mag = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) mag = max(mag, max(w[j] & 0x7FFFu, (w[j] >> 16) & 0x7FFFu));
      mag = halfwarp_max_u32(mag);
      const uint32_t sb = scale_byte_from_bf16_mag(mag);
      const float inv = inv_scale_from_byte(sb);
      uint32_t c[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) c[j] = cvt_e4m3x2_f32(bf16lo_to_f32(w[j]) * inv, bf16hi_to_f32(w[j]) * inv);
      if (r < nrows && col_ok) st_v2(q + (row0 + r) * cols + col, c[0] | (c[1] << 16), c[2] | (c[3] << 16));
      packed |= sb << (8 * r);
    }
    if (sub == 0 && col_ok) {
      uint8_t* sp = s + (cp * 2 + half) * ld_s + row0;
      if (nrows == kQuantRows) {
        *reinterpret_cast<uint32_t*>(sp) = packed;  // row0 % 4 == 0 and ld_s % 16 == 0: aligned
      } else {
        for (int r = 0; r < nrows; ++r) sp[r] = static_cast<uint8_t>(packed >> (8 * r));
      }
    }
  }
}

cudaError_t launch_quantize_rowwise(const void* x, int64_t rows, int64_t cols, uint8_t* q, uint8_t* s,
                                    int64_t ld_s, cudaStream_t stream, int num_sms) {
  const int64_t n_items = ((rows + kQuantRows - 1) / kQuantRows) * ((cols + 255) / 256);
  static const int occ = occupancy_of(quantize_rowwise_kernel, 256, 0);
  const int sched = sched_for("A1", kSchedInterleaved);
  const int64_t grid = sched_grid(sched, n_items, 8, occ, num_sms);
  quantize_rowwise_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(x),
                                                                           rows, cols, q, s, ld_s, sched);
  return cudaGetLastError();
}

}  // namespace fp8flow
