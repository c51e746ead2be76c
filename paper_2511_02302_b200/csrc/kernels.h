// kernels.h -- internal launch functions of libfp8flow (not part of the public C ABI).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace fp8flow {

constexpr int kMaxRanks = 64;  // FP8FLOW_MAX_RANKS

struct DeviceInfo {
  int device;
  int num_sms;
  int cc_major, cc_minor;
};

// resident CTAs per SM of a kernel (query once per call site: `static const int occ = ...`)
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

// Work-item schedule of an op (see Sched in common.cuh): the tuned default, overridable for
// tuning experiments with FP8FLOW_SCHED_<OP> (0 one-item-per-warp, 1 blocked, 2 interleaved).
int sched_for(const char* op, int tuned_default);
// Integer tuning knob FP8FLOW_<name> (tuning experiments only), else the tuned default.
int tune_int(const char* name, int tuned_default);
// grid for a warp-item kernel under a schedule
inline int64_t sched_grid(int sched, int64_t n_items, int warps_per_cta, int occ, int num_sms) {
  const int64_t need = (n_items + warps_per_cta - 1) / warps_per_cta;
  if (sched == 0) return need < 1 ? 1 : need;
  return one_wave_grid(occ, num_sms, need);
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
cudaError_t launch_permute_pad(const uint8_t* q_tok, const uint8_t* s_tok, int64_t ld_s_tok, int64_t hidden,
                               const int32_t* src_of_row, const int32_t* expert_offsets, int32_t num_local_experts,
                               int64_t max_rows, uint8_t* q_out, uint8_t* s_out, cudaStream_t stream, int num_sms);
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
cudaError_t launch_gemm_blockscaled(const uint8_t* A, const uint8_t* sa, int64_t ld_sa, const uint8_t* B,
                                    const uint8_t* sb, int64_t ld_sb, int64_t M, int64_t N, int64_t K,
                                    const int32_t* seg_offsets, int32_t num_groups, void* D, int32_t d_f32,
                                    cudaStream_t stream, int num_sms);
cudaError_t launch_gemm_wgrad(const uint8_t* AT, const uint8_t* saT, int64_t Ma, const uint8_t* BT, const uint8_t* sbT,
                              int64_t Nb, const int32_t* seg_offsets, int32_t num_groups, void* D, int32_t d_f32,
                              cudaStream_t stream, int num_sms);
cudaError_t launch_swiglu_bwd_quant(const void* h, const void* dA, int64_t rows_max, const int32_t* rows_dev,
                                    int64_t ffn, uint8_t* q, uint8_t* s, int64_t ld_s, cudaStream_t stream,
                                    int num_sms);

cudaError_t launch_peer_gather(const void* const* peer_src, int32_t n, int64_t bytes_per_rank, void* dst,
                               cudaStream_t stream, int num_sms);
cudaError_t launch_peer_barrier(void* const* peer_signal, int32_t rank, int32_t n, int32_t* status,
                                uint32_t timeout_ms, cudaStream_t stream);
cudaError_t launch_dispatch_permute_pad(const uint8_t* const* peer_q, const uint8_t* const* peer_s, int64_t ld_s_tok,
                                        int32_t n, int64_t tokens_per_rank, int64_t hidden, const int32_t* row_map,
                                        int32_t top_k, const int32_t* src_of_row, const int32_t* expert_offsets,
                                        int32_t num_local_experts, int64_t max_rows, uint8_t* q_out, uint8_t* s_out,
                                        cudaStream_t stream, int num_sms);
cudaError_t launch_combine_unpermute(const void* const* peer_x, const int32_t* const* peer_row_map, int32_t n,
                                     int64_t hidden, const int32_t* topk_idx, int32_t experts_per_rank,
                                     const float* probs, int64_t token_begin, int64_t num_tokens, int32_t top_k,
                                     void* y, cudaStream_t stream, int num_sms);

cudaError_t launch_checksum64(const void* buf, int64_t nbytes, uint64_t* out, cudaStream_t stream, int num_sms);

}  // namespace fp8flow
