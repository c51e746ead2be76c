// kernels.h -- internal launch functions of libfp8flow (not part of the public C ABI).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace fp8flow {

struct DeviceInfo {
  int device;
  int num_sms;
  int cc_major, cc_minor;
};

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

cudaError_t launch_checksum64(const void* buf, int64_t nbytes, uint64_t* out, cudaStream_t stream, int num_sms);

}  // namespace fp8flow
