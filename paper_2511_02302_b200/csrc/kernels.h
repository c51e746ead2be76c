// kernels.h -- internal launch functions of libfp8flow (not part of the public C ABI).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace fp8flow {

constexpr int kMaxRanks = 64;  // FP8FLOW_MAX_RANKS

// cuTensorMapEncodeTiled from the driver (resolved once through the runtime; no -lcuda)
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled tensor_map_encoder();
// A 2D tensor map of a row-major [rows][cols] tensor (element type dt, row pitch in bytes) with
// box {box_cols, box_rows}, no swizzle, 256-byte L2 promotion.  false if the driver rejects it.
bool encode_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t cols, uint64_t rows,
               uint64_t row_pitch_bytes, uint32_t box_cols, uint32_t box_rows,
               CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_NONE);

// resident CTAs per SM of a kernel
template <typename Kernel>
inline int occupancy_of(Kernel kernel, int threads, size_t smem) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem) != cudaSuccess || occ < 1) occ = 1;
  return occ;
}
// one full wave of CTAs (SMs x occupancy), capped by the work available
inline int64_t one_wave_grid(int occ, int num_sms, int64_t max_ctas) {
  int64_t g = static_cast<int64_t>(num_sms) * occ;
  if (g > max_ctas) g = max_ctas;
  return g < 1 ? 1 : g;
}

// Per-device launch setup of one kernel.  cudaFuncSetAttribute (the dynamic shared-memory opt-in)
// and the occupancy it implies apply to the CURRENT device only, so they are recorded per device
// id: a process that drives several GPUs prepares the kernel once on each.  Idempotent; the
// unsynchronised first use on two host threads only repeats the same calls.
constexpr int kMaxDevices = 64;
struct KernelSetup {
  int occ[kMaxDevices] = {};  // resident CTAs per SM on device d; 0 = not prepared yet
};
// Opts the kernel in to `attr_smem` bytes of dynamic shared memory (when above the 48 KB default)
// and returns its occupancy at (threads, occ_smem) on the current device; 0 if the device cannot
// be queried or the attribute is refused.
template <typename Kernel>
inline int prepare_kernel(KernelSetup& ks, Kernel kernel, int threads, size_t attr_smem, size_t occ_smem) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 0;
  int occ = __atomic_load_n(&ks.occ[dev], __ATOMIC_ACQUIRE);
  if (occ > 0) return occ;
  if (attr_smem > 48 * 1024 &&
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(attr_smem)) !=
          cudaSuccess)
    return 0;
  occ = occupancy_of(kernel, threads, occ_smem);
  __atomic_store_n(&ks.occ[dev], occ, __ATOMIC_RELEASE);
  return occ;
}

cudaError_t launch_quantize_rowwise(const void* x, int64_t rows, int64_t cols, uint8_t* q, uint8_t* s,
                                    int64_t ld_s, cudaStream_t stream, int num_sms);

cudaError_t launch_scaling_aware_transpose(const uint8_t* q, const uint8_t* s, int64_t ld_s, int64_t rows,
                                           int64_t cols, const int32_t* seg_offsets, int32_t num_segs,
                                           uint8_t* qT, uint8_t* sT, cudaStream_t stream, int num_sms);

size_t naive_workspace_bytes(int64_t rows, int64_t cols, int32_t num_segs);
cudaError_t launch_naive_transpose(const uint8_t* q, const uint8_t* s, int64_t ld_s, int64_t rows, int64_t cols,
                                   const int32_t* seg_offsets, int32_t num_segs, uint8_t* qT, uint8_t* sT,
                                   void* ws, cudaStream_t stream, int num_sms);

size_t permute_workspace_bytes(int64_t num_tokens, int32_t num_local_experts);
cudaError_t launch_permute_plan(const int32_t* topk_idx, int64_t num_tokens, int32_t top_k, int32_t expert_begin,
                                int32_t num_local_experts, int32_t align, int32_t* row_map, int32_t* src_of_row,
                                int64_t max_rows, int32_t* expert_offsets, void* ws, cudaStream_t stream);
cudaError_t launch_unpermute_unpad(const void* x, int64_t hidden, const int32_t* row_map, const float* probs,
                                   int64_t num_tokens, int32_t top_k, void* y, cudaStream_t stream, int num_sms);

cudaError_t launch_swiglu_quant(const void* h, int64_t rows_max, const int32_t* rows_dev, int64_t ffn, uint8_t* q,
                                uint8_t* s, int64_t ld_s, cudaStream_t stream, int num_sms);

cudaError_t launch_quantize_dual(const void* x, int64_t rows, int64_t cols, const int32_t* seg_offsets,
                                 int32_t num_segs, uint8_t* q, uint8_t* s, int64_t ld_s, uint8_t* qT, uint8_t* sT,
                                 cudaStream_t stream, int num_sms);
cudaError_t launch_swiglu_quant_dual(const void* h, int64_t rows_max, const int32_t* rows_dev, int64_t ffn,
                                     const int32_t* seg_offsets, int32_t num_segs, uint8_t* q, uint8_t* s,
                                     int64_t ld_s, uint8_t* qT, uint8_t* sT, cudaStream_t stream, int num_sms);
cudaError_t launch_permute_pad_dual(const uint8_t* q_tok, const uint8_t* s_tok, int64_t ld_s_tok, int64_t hidden,
                                    const int32_t* src_of_row, const int32_t* expert_offsets,
                                    int32_t num_local_experts, int64_t max_rows, uint8_t* q_out, uint8_t* s_out,
                                    uint8_t* qT, uint8_t* sT, cudaStream_t stream, int num_sms);
cudaError_t launch_gemm_blockscaled(const uint8_t* A, const uint8_t* sa, int64_t ld_sa, const uint8_t* B,
                                    const uint8_t* sb, int64_t ld_sb, int64_t M, int64_t N, int64_t K,
                                    const int32_t* seg_offsets, int32_t num_groups, void* D, int32_t d_f32,
                                    cudaStream_t stream, int num_sms);
cudaError_t launch_gemm_wgrad(const uint8_t* AT, const uint8_t* saT, int64_t Ma, const uint8_t* BT, const uint8_t* sbT,
                              int64_t Nb, const int32_t* seg_offsets, int32_t num_groups, void* D, int32_t d_f32,
                              void* workspace, cudaStream_t stream, int num_sms);
cudaError_t launch_swiglu_bwd_quant(const void* h, const void* dA, int64_t rows_max, const int32_t* rows_dev,
                                    int64_t ffn, uint8_t* q, uint8_t* s, int64_t ld_s, cudaStream_t stream,
                                    int num_sms);

cudaError_t launch_peer_gather(const void* const* peer_src, int32_t n, int64_t bytes_per_rank, void* dst,
                               const int32_t* gate, cudaStream_t stream, int num_sms);
cudaError_t launch_peer_barrier(void* const* peer_signal, int32_t rank, int32_t n, int32_t* status,
                                uint32_t timeout_ms, cudaStream_t stream);
cudaError_t launch_dispatch_permute_pad(const uint8_t* const* peer_q, const uint8_t* const* peer_s, int64_t ld_s_tok,
                                        int32_t n, int64_t tokens_per_rank, int64_t hidden, const int32_t* row_map,
                                        int32_t top_k, const int32_t* src_of_row, const int32_t* expert_offsets,
                                        int32_t num_local_experts, int64_t max_rows, uint8_t* q_out, uint8_t* s_out,
                                        int32_t kernel, const int32_t* gate, cudaStream_t stream, int num_sms);
cudaError_t launch_combine_unpermute(const void* const* peer_x, const int32_t* const* peer_row_map, int32_t n,
                                     int64_t hidden, const int32_t* topk_idx, int32_t experts_per_rank,
                                     const float* probs, int64_t token_begin, int64_t num_tokens, int32_t top_k,
                                     void* y, const int32_t* gate, cudaStream_t stream, int num_sms);

cudaError_t launch_checksum64(const void* buf, int64_t nbytes, uint64_t* out, cudaStream_t stream, int num_sms);

}  // namespace fp8flow
