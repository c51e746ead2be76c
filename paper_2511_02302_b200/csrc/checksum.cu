// checksum.cu -- verification checksum of an output buffer (C11):
//   sum_i b_i * (i * 0x9E3779B97F4A7C15 + 1)  mod 2^64
// Order-independent (a sum mod 2^64) and position-sensitive, so per-rank checksums can be
// gathered with NCCL after the timed region and compared with the oracle's.
#include "common.cuh"
#include "kernels.h"

namespace fp8flow {

__global__ void __launch_bounds__(256) checksum64_kernel(const uint8_t* __restrict__ buf, int64_t nbytes,
                                                         unsigned long long* __restrict__ out) {
  constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ull;
  uint64_t acc = 0;
  const int64_t n16 = nbytes / 16;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t v = tid; v < n16; v += nth) {
    const uint4 w = ld_nc_v4(buf + v * 16);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    const uint64_t i0 = static_cast<uint64_t>(v) * 16;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint64_t b = (ws[k >> 2] >> (8 * (k & 3))) & 0xFFu;
      acc += b * ((i0 + k) * kPhi + 1ull);
    }
  }
  for (int64_t i = n16 * 16 + tid; i < nbytes; i += nth) acc += static_cast<uint64_t>(buf[i]) * (static_cast<uint64_t>(i) * kPhi + 1ull);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, static_cast<unsigned long long>(acc));
}

cudaError_t launch_checksum64(const void* buf, int64_t nbytes, uint64_t* out, cudaStream_t stream, int num_sms) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(uint64_t), stream);
  if (e != cudaSuccess) return e;
  int64_t blocks = (nbytes / 16 + 255) / 256;
  const int64_t cap = static_cast<int64_t>(num_sms) * 4;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  checksum64_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(static_cast<const uint8_t*>(buf), nbytes,
                                                                       reinterpret_cast<unsigned long long*>(out));
  return cudaGetLastError();
}

}  // namespace fp8flow
