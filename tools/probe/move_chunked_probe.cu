// Move probe (not product): the A3 move as a column-chunked row gather -- for each chunk of CH
// bytes of the hidden dimension (chunk-major), every output row r copies its CH bytes from token
// src_of_row[r] (PAD rows: zeros) and the chunk's scale bytes; a warp copies one row's chunk with
// 16-byte loads/stores.  Rows are walked in order, so each chunk pass writes X_perm rows
// sequentially while the tokens' CH-byte pieces (num_tokens x CH bytes) stay in L2.
#include <cstdint>
#include <cuda_runtime.h>

template <int CH>
__global__ void __launch_bounds__(256) move_chunked_kernel(const uint8_t* __restrict__ q_tok, const uint8_t* __restrict__ s_tok,
                                                           int64_t ld_s_tok, int64_t H, const int32_t* __restrict__ src_of_row,
                                                           int64_t R, int64_t max_rows, uint8_t* __restrict__ q_out,
                                                           uint8_t* __restrict__ s_out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t nch = H / CH;
  constexpr int kV = CH / 16 / 32;  // 16-byte vectors per lane per row chunk
  for (int64_t item = gw; item < nch * R; item += nw) {
    const int64_t q = item / R, r = item - q * R;
    const int src = __ldg(src_of_row + r);
    const uint4* sp = reinterpret_cast<const uint4*>(q_tok + static_cast<int64_t>(src < 0 ? 0 : src) * H + q * CH);
    uint4* dp = reinterpret_cast<uint4*>(q_out + r * H + q * CH);
    uint4 v[kV > 0 ? kV : 1];
#pragma unroll
    for (int k = 0; k < kV; ++k) v[k] = src >= 0 ? __ldg(sp + lane + 32 * k) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < kV; ++k) dp[lane + 32 * k] = v[k];
    if (lane < CH / 128) {  // the chunk's scale bytes
      const int64_t j = q * (CH / 128) + lane;
      s_out[j * max_rows + r] = src >= 0 ? __ldg(s_tok + j * ld_s_tok + src) : 0;
    }
  }
}

extern "C" int probe_move_chunked(const void* q_tok, const void* s_tok, int64_t ld_s_tok, int64_t H, const int32_t* src,
                                  int64_t R, int64_t max_rows, void* q_out, void* s_out, int ch, int grid, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto a = static_cast<const uint8_t*>(q_tok);
  auto b = static_cast<const uint8_t*>(s_tok);
  auto o = static_cast<uint8_t*>(q_out);
  auto so = static_cast<uint8_t*>(s_out);
  if (ch == 512) move_chunked_kernel<512><<<grid, 256, 0, st>>>(a, b, ld_s_tok, H, src, R, max_rows, o, so);
  else if (ch == 1024) move_chunked_kernel<1024><<<grid, 256, 0, st>>>(a, b, ld_s_tok, H, src, R, max_rows, o, so);
  else if (ch == 3584) move_chunked_kernel<3584><<<grid, 256, 0, st>>>(a, b, ld_s_tok, H, src, R, max_rows, o, so);
  else move_chunked_kernel<7168><<<grid, 256, 0, st>>>(a, b, ld_s_tok, H, src, R, max_rows, o, so);
  return static_cast<int>(cudaGetLastError());
}
