// api.cu -- the extern "C" boundary of libfp8flow (include/fp8flow.h): argument validation,
// architecture check, status codes, and dispatch to the sm_100a kernels.  No compute happens on
// the host and there is no fallback path.
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "../../include/fp8flow.h"
#include "kernels.h"

using namespace fp8flow;

PFN_encodeTiled fp8flow::tensor_map_encoder() {
  static PFN_encodeTiled fn = nullptr;  // a process-wide driver entry point (not device state)
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qres;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qres) == cudaSuccess &&
        qres == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

bool fp8flow::encode_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t cols, uint64_t rows,
                        uint64_t row_pitch_bytes, uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swizzle) {
  PFN_encodeTiled encode = tensor_map_encoder();
  if (!encode) return false;
  const cuuint64_t gdim[2] = {cols, rows};
  const cuuint64_t gstride[1] = {row_pitch_bytes};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estride[2] = {1, 1};
  return encode(map, dt, 2, const_cast<void*>(base), gdim, gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

thread_local int g_last_cuda_error = 0;

int g_dev_ok[kMaxDevices];   // 0 = unknown, 1 = sm_100, 2 = other
int g_dev_sms[kMaxDevices];

int fail_cuda(cudaError_t e) {
  g_last_cuda_error = static_cast<int>(e);
  return FP8FLOW_ERR_CUDA;
}

// resolves the current device; returns OK / ERR_ARCH / ERR_CUDA and the SM count
int device(int* num_sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail_cuda(e);
  if (dev < 0 || dev >= kMaxDevices) return FP8FLOW_ERR_ARCH;
  if (g_dev_ok[dev] == 0) {
    int major = 0, minor = 0, sms = 0;
    if ((e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev)) != cudaSuccess ||
        (e = cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev)) != cudaSuccess ||
        (e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
      return fail_cuda(e);
    g_dev_sms[dev] = sms;
    g_dev_ok[dev] = (major == 10 && minor == 0) ? 1 : 2;
  }
  if (g_dev_ok[dev] != 1) return FP8FLOW_ERR_ARCH;
  *num_sms = g_dev_sms[dev];
  return FP8FLOW_OK;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline int launched(cudaError_t e) { return e == cudaSuccess ? FP8FLOW_OK : fail_cuda(e); }

}  // namespace

extern "C" {

const char* fp8flow_status_string(int status) {
  switch (status) {
    case FP8FLOW_OK: return "FP8FLOW_OK";
    case FP8FLOW_ERR_NULL: return "FP8FLOW_ERR_NULL";
    case FP8FLOW_ERR_SHAPE: return "FP8FLOW_ERR_SHAPE";
    case FP8FLOW_ERR_ALIGN: return "FP8FLOW_ERR_ALIGN";
    case FP8FLOW_ERR_ARG: return "FP8FLOW_ERR_ARG";
    case FP8FLOW_ERR_WORKSPACE: return "FP8FLOW_ERR_WORKSPACE";
    case FP8FLOW_ERR_ARCH: return "FP8FLOW_ERR_ARCH";
    case FP8FLOW_ERR_CUDA: return "FP8FLOW_ERR_CUDA";
    default: return "FP8FLOW_UNKNOWN_STATUS";
  }
}

int fp8flow_last_cuda_error(void) { return g_last_cuda_error; }
int fp8flow_version(void) { return 100; }  // 0.1.0
const char* fp8flow_build_target(void) { return "sm_100a"; }
#ifndef FP8FLOW_SOURCE_HASH
#define FP8FLOW_SOURCE_HASH "unknown"
#endif
const char* fp8flow_source_hash(void) { return FP8FLOW_SOURCE_HASH; }

int fp8flow_device_check(void) {
  int sms = 0;
  return device(&sms);
}

int fp8flow_quantize_rowwise(const void* x_bf16, int64_t rows, int64_t cols, uint8_t* q, uint8_t* s, int64_t ld_s,
                             void* stream) {
  if (rows < 0 || cols <= 0 || cols % 128 != 0) return FP8FLOW_ERR_SHAPE;
  if (ld_s < rows || ld_s % 16 != 0) return FP8FLOW_ERR_SHAPE;
  if (rows == 0) return FP8FLOW_OK;
  if (!x_bf16 || !q || !s) return FP8FLOW_ERR_NULL;
  if (!aligned16(x_bf16) || !aligned16(q) || !aligned16(s)) return FP8FLOW_ERR_ALIGN;
  int sms = 0, st = device(&sms);
  if (st != FP8FLOW_OK) return st;
  return launched(launch_quantize_rowwise(x_bf16, rows, cols, q, s, ld_s, static_cast<cudaStream_t>(stream), sms));
}

static int check_transpose_args(const uint8_t* q, const uint8_t* s, int64_t ld_s, int64_t rows, int64_t cols,
                                const int32_t* seg_offsets, int32_t num_segs, const uint8_t* qT, const uint8_t* sT) {
  if (rows < 0 || cols <= 0 || cols % 128 != 0 || rows % 16 != 0) return FP8FLOW_ERR_SHAPE;
  if (rows > INT32_MAX - 128) return FP8FLOW_ERR_SHAPE;
  if (ld_s < rows || ld_s % 16 != 0) return FP8FLOW_ERR_SHAPE;
  if (seg_offsets && (num_segs < 1 || num_segs > 1024)) return FP8FLOW_ERR_ARG;
  if (!q || !s || !qT || !sT) return FP8FLOW_ERR_NULL;
  if (!aligned16(q) || !aligned16(s) || !aligned16(qT) || !aligned16(sT)) return FP8FLOW_ERR_ALIGN;
  return FP8FLOW_OK;
}

int fp8flow_scaling_aware_transpose(const uint8_t* q, const uint8_t* s, int64_t ld_s, int64_t rows, int64_t cols,
                                    const int32_t* seg_offsets, int32_t num_segs, uint8_t* qT, uint8_t* sT,
                                    void* stream) {
  if (rows == 0 && !seg_offsets) return FP8FLOW_OK;
  int st = check_transpose_args(q, s, ld_s, rows, cols, seg_offsets, num_segs, qT, sT);
  if (st != FP8FLOW_OK) return st;
  int sms = 0;
  if ((st = device(&sms)) != FP8FLOW_OK) return st;
  return launched(launch_scaling_aware_transpose(q, s, ld_s, rows, cols, seg_offsets, num_segs, qT, sT,
                                                 static_cast<cudaStream_t>(stream), sms));
}

size_t fp8flow_naive_workspace_bytes(int64_t rows, int64_t cols, int32_t num_segs) {
  if (rows < 0 || cols < 0 || num_segs < 0) return 0;
  return naive_workspace_bytes(rows, cols, num_segs < 1 ? 1 : num_segs);
}

int fp8flow_naive_transpose(const uint8_t* q, const uint8_t* s, int64_t ld_s, int64_t rows, int64_t cols,
                            const int32_t* seg_offsets, int32_t num_segs, uint8_t* qT, uint8_t* sT, void* ws,
                            size_t ws_bytes, void* stream) {
  if (rows == 0 && !seg_offsets) return FP8FLOW_OK;
  int st = check_transpose_args(q, s, ld_s, rows, cols, seg_offsets, num_segs, qT, sT);
  if (st != FP8FLOW_OK) return st;
  if (!ws) return FP8FLOW_ERR_NULL;
  if (!aligned16(ws)) return FP8FLOW_ERR_ALIGN;
  if (ws_bytes < naive_workspace_bytes(rows, cols, seg_offsets ? num_segs : 1)) return FP8FLOW_ERR_WORKSPACE;
  int sms = 0;
  if ((st = device(&sms)) != FP8FLOW_OK) return st;
  return launched(launch_naive_transpose(q, s, ld_s, rows, cols, seg_offsets, num_segs, qT, sT, ws,
                                         static_cast<cudaStream_t>(stream), sms));
}

size_t fp8flow_permute_workspace_bytes(int64_t num_tokens, int32_t top_k, int32_t num_local_experts) {
  (void)top_k;
  if (num_tokens < 0 || num_local_experts < 1) return 0;
  return permute_workspace_bytes(num_tokens, num_local_experts);
}

int fp8flow_permute_plan(const int32_t* topk_idx, int64_t num_tokens, int32_t top_k, int32_t expert_begin,
                         int32_t num_local_experts, int32_t align, int32_t* row_map, int32_t* src_of_row,
                         int64_t max_rows, int32_t* expert_offsets, void* ws, size_t ws_bytes, void* stream) {
  if (num_tokens < 0 || max_rows < 0) return FP8FLOW_ERR_SHAPE;
  if (top_k < 1 || top_k > 16 || num_local_experts < 1 || num_local_experts > 1024 || align < 1 || align > 1024 ||
      expert_begin < 0)
    return FP8FLOW_ERR_ARG;
  if (num_tokens > INT32_MAX / 16 || max_rows > INT32_MAX) return FP8FLOW_ERR_SHAPE;
  if (!expert_offsets || !ws || (num_tokens > 0 && (!topk_idx || !row_map)) || (max_rows > 0 && !src_of_row))
    return FP8FLOW_ERR_NULL;
  if (ws_bytes < permute_workspace_bytes(num_tokens, num_local_experts)) return FP8FLOW_ERR_WORKSPACE;
  if (!aligned16(ws)) return FP8FLOW_ERR_ALIGN;
  int sms = 0, st = device(&sms);
  if (st != FP8FLOW_OK) return st;
  return launched(launch_permute_plan(topk_idx, num_tokens, top_k, expert_begin, num_local_experts, align, row_map,
                                      src_of_row, max_rows, expert_offsets, ws, static_cast<cudaStream_t>(stream)));
}

int fp8flow_permute_pad(const uint8_t* q_tok, const uint8_t* s_tok, int64_t ld_s_tok, int64_t num_tokens,
                        int64_t hidden, const int32_t* row_map, int32_t top_k, const int32_t* src_of_row,
                        const int32_t* expert_offsets, int32_t num_local_experts, int64_t max_rows, uint8_t* q_out,
                        uint8_t* s_out, void* stream) {
  if (num_tokens < 0 || hidden <= 0 || hidden % 128 != 0 || max_rows < 0 || max_rows % 16 != 0)
    return FP8FLOW_ERR_SHAPE;
  if (ld_s_tok < num_tokens || num_tokens > INT32_MAX) return FP8FLOW_ERR_SHAPE;
  if (num_local_experts < 1 || num_local_experts > 1024 || top_k < 1 || top_k > 16) return FP8FLOW_ERR_ARG;
  if (max_rows == 0 || num_tokens == 0) return FP8FLOW_OK;  // no tokens: every expert is empty
  if (!row_map || !src_of_row || !expert_offsets || !q_out || !s_out || !q_tok || !s_tok) return FP8FLOW_ERR_NULL;
  if (!aligned16(q_tok) || !aligned16(q_out)) return FP8FLOW_ERR_ALIGN;
  int sms = 0, st = device(&sms);
  if (st != FP8FLOW_OK) return st;
  // the move is the one-rank case of the fused dispatch: each token is read once and written to all
  // of its local expert rows (bulk-copy engine; register copies when the engine's ring cannot fit)
  return launched(launch_dispatch_permute_pad(&q_tok, &s_tok, ld_s_tok, 1, num_tokens, hidden, row_map, top_k,
                                              src_of_row, expert_offsets, num_local_experts, max_rows, q_out, s_out,
                                              FP8FLOW_DISPATCH_AUTO, nullptr, static_cast<cudaStream_t>(stream), sms));
}

int fp8flow_unpermute_unpad(const void* x_bf16, int64_t hidden, const int32_t* row_map, const float* probs,
                            int64_t num_tokens, int32_t top_k, void* y_bf16, void* stream) {
  if (num_tokens < 0 || hidden <= 0 || hidden % 8 != 0) return FP8FLOW_ERR_SHAPE;
  if (top_k < 1 || top_k > 16) return FP8FLOW_ERR_ARG;
  if (num_tokens == 0) return FP8FLOW_OK;
  if (!x_bf16 || !row_map || !y_bf16) return FP8FLOW_ERR_NULL;
  if (!aligned16(x_bf16) || !aligned16(y_bf16) || (hidden * 2) % 16 != 0) return FP8FLOW_ERR_ALIGN;
  int sms = 0, st = device(&sms);
  if (st != FP8FLOW_OK) return st;
  return launched(launch_unpermute_unpad(x_bf16, hidden, row_map, probs, num_tokens, top_k, y_bf16,
                                         static_cast<cudaStream_t>(stream), sms));
}

int fp8flow_swiglu_quant(const void* h_bf16, int64_t rows_max, const int32_t* rows_dev, int64_t ffn, uint8_t* q,
                         uint8_t* s, int64_t ld_s, void* stream) {
  if (rows_max < 0 || ffn <= 0 || ffn % 128 != 0) return FP8FLOW_ERR_SHAPE;
  if (ld_s < rows_max || ld_s % 16 != 0) return FP8FLOW_ERR_SHAPE;
  if (rows_max == 0) return FP8FLOW_OK;
  if (!h_bf16 || !q || !s) return FP8FLOW_ERR_NULL;
  if (!aligned16(h_bf16) || !aligned16(q)) return FP8FLOW_ERR_ALIGN;
  int sms = 0, st = device(&sms);
  if (st != FP8FLOW_OK) return st;
  return launched(
      launch_swiglu_quant(h_bf16, rows_max, rows_dev, ffn, q, s, ld_s, static_cast<cudaStream_t>(stream), sms));
}

int fp8flow_swiglu_bwd_quant(const void* h_bf16, const void* dA_bf16, int64_t rows_max, const int32_t* rows_dev,
                             int64_t ffn, uint8_t* q, uint8_t* s, int64_t ld_s, void* stream) {
  if (rows_max < 0 || ffn <= 0 || ffn % 128 != 0) return FP8FLOW_ERR_SHAPE;
  if (ld_s < rows_max || ld_s % 16 != 0) return FP8FLOW_ERR_SHAPE;
  if (rows_max == 0) return FP8FLOW_OK;
  if (!h_bf16 || !dA_bf16 || !q || !s) return FP8FLOW_ERR_NULL;
  if (!aligned16(h_bf16) || !aligned16(dA_bf16) || !aligned16(q)) return FP8FLOW_ERR_ALIGN;
  int sms = 0, st = device(&sms);
  if (st != FP8FLOW_OK) return st;
  return launched(launch_swiglu_bwd_quant(h_bf16, dA_bf16, rows_max, rows_dev, ffn, q, s, ld_s,
                                          static_cast<cudaStream_t>(stream), sms));
}

int fp8flow_quantize_dual(const void* x_bf16, int64_t rows, int64_t cols, const int32_t* seg_offsets,
                          int32_t num_segs, uint8_t* q, uint8_t* s, int64_t ld_s, uint8_t* qT, uint8_t* sT,
                          void* stream) {
  if (rows == 0 && !seg_offsets) return FP8FLOW_OK;
  int st = check_transpose_args(q, s, ld_s, rows, cols, seg_offsets, num_segs, qT, sT);
  if (st != FP8FLOW_OK) return st;
  if (!x_bf16) return FP8FLOW_ERR_NULL;
  if (!aligned16(x_bf16)) return FP8FLOW_ERR_ALIGN;
  int sms = 0;
  if ((st = device(&sms)) != FP8FLOW_OK) return st;
  return launched(launch_quantize_dual(x_bf16, rows, cols, seg_offsets, num_segs, q, s, ld_s, qT, sT,
                                       static_cast<cudaStream_t>(stream), sms));
}

int fp8flow_swiglu_quant_dual(const void* h_bf16, int64_t rows_max, const int32_t* rows_dev, int64_t ffn,
                              const int32_t* seg_offsets, int32_t num_segs, uint8_t* q, uint8_t* s, int64_t ld_s,
                              uint8_t* qT, uint8_t* sT, void* stream) {
  if (rows_max == 0) return FP8FLOW_OK;
  int st = check_transpose_args(q, s, ld_s, rows_max, ffn, seg_offsets, num_segs, qT, sT);
  if (st != FP8FLOW_OK) return st;
  if (!h_bf16) return FP8FLOW_ERR_NULL;
  if (!aligned16(h_bf16)) return FP8FLOW_ERR_ALIGN;
  int sms = 0;
  if ((st = device(&sms)) != FP8FLOW_OK) return st;
  return launched(launch_swiglu_quant_dual(h_bf16, rows_max, rows_dev, ffn, seg_offsets, num_segs, q, s, ld_s, qT,
                                           sT, static_cast<cudaStream_t>(stream), sms));
}

int fp8flow_permute_pad_dual(const uint8_t* q_tok, const uint8_t* s_tok, int64_t ld_s_tok, int64_t num_tokens,
                             int64_t hidden, const int32_t* src_of_row, const int32_t* expert_offsets,
                             int32_t num_local_experts, int64_t max_rows, uint8_t* q_out, uint8_t* s_out, uint8_t* qT,
                             uint8_t* sT, void* stream) {
  if (num_tokens < 0 || hidden <= 0 || hidden % 128 != 0 || max_rows < 0 || max_rows % 16 != 0)
    return FP8FLOW_ERR_SHAPE;
  if (ld_s_tok < num_tokens || ld_s_tok % 4 != 0 || num_tokens > INT32_MAX || max_rows > INT32_MAX - 128)
    return FP8FLOW_ERR_SHAPE;
  if (num_local_experts < 1 || num_local_experts > 1024) return FP8FLOW_ERR_ARG;
  if (max_rows == 0 || num_tokens == 0) return FP8FLOW_OK;  // no tokens: every expert is empty
  if (!q_tok || !s_tok || !src_of_row || !expert_offsets || !q_out || !s_out || !qT || !sT) return FP8FLOW_ERR_NULL;
  if (!aligned16(q_tok) || !aligned16(s_tok) || !aligned16(q_out) || !aligned16(s_out) || !aligned16(qT) ||
      !aligned16(sT) || !aligned16(src_of_row))
    return FP8FLOW_ERR_ALIGN;
  int sms = 0, st = device(&sms);
  if (st != FP8FLOW_OK) return st;
  return launched(launch_permute_pad_dual(q_tok, s_tok, ld_s_tok, hidden, src_of_row, expert_offsets,
                                          num_local_experts, max_rows, q_out, s_out, qT, sT,
                                          static_cast<cudaStream_t>(stream), sms));
}

int fp8flow_gemm_blockscaled(const uint8_t* A, const uint8_t* sa, int64_t ld_sa, const uint8_t* B, const uint8_t* sb,
                             int64_t ld_sb, int64_t M, int64_t N, int64_t K, const int32_t* seg_offsets,
                             int32_t num_groups, void* D, int32_t d_f32, void* stream) {
  if (M < 0 || N <= 0 || K <= 0 || M % 16 != 0 || N % 256 != 0 || K % 128 != 0) return FP8FLOW_ERR_SHAPE;
  if (M > INT32_MAX - 128 || N > (1 << 24)) return FP8FLOW_ERR_SHAPE;
  if (ld_sa < M || ld_sa % 16 != 0 || ld_sb < N || ld_sb % 16 != 0) return FP8FLOW_ERR_SHAPE;
  if (seg_offsets && (num_groups < 1 || num_groups > 512)) return FP8FLOW_ERR_ARG;
  if (M == 0 && !seg_offsets) return FP8FLOW_OK;
  if (!A || !sa || !B || !sb || !D) return FP8FLOW_ERR_NULL;
  if (!aligned16(A) || !aligned16(sa) || !aligned16(B) || !aligned16(sb) || !aligned16(D)) return FP8FLOW_ERR_ALIGN;
  int sms = 0, st = device(&sms);
  if (st != FP8FLOW_OK) return st;
  return launched(launch_gemm_blockscaled(A, sa, ld_sa, B, sb, ld_sb, M, N, K, seg_offsets, num_groups, D, d_f32,
                                          static_cast<cudaStream_t>(stream), sms));
}

int64_t fp8flow_gemm_wgrad_workspace_bytes(int32_t num_groups) {
  return num_groups < 1 ? 0 : static_cast<int64_t>(num_groups) * 256;  // two 128-byte TMA maps per group
}

int fp8flow_gemm_wgrad(const uint8_t* AT, const uint8_t* saT, int64_t Ma, const uint8_t* BT, const uint8_t* sbT,
                       int64_t Nb, const int32_t* seg_offsets, int32_t num_groups, void* D, int32_t d_f32,
                       void* workspace, int64_t workspace_bytes, void* stream) {
  if (Ma <= 0 || Nb <= 0 || Ma % 128 != 0 || Nb % 256 != 0 || Ma > (1 << 24) || Nb > (1 << 24)) return FP8FLOW_ERR_SHAPE;
  if (num_groups < 1 || num_groups > 512) return FP8FLOW_ERR_ARG;
  if (!AT || !saT || !BT || !sbT || !D || !seg_offsets || !workspace) return FP8FLOW_ERR_NULL;
  if (workspace_bytes < fp8flow_gemm_wgrad_workspace_bytes(num_groups)) return FP8FLOW_ERR_WORKSPACE;
  if (!aligned16(AT) || !aligned16(saT) || !aligned16(BT) || !aligned16(sbT) || !aligned16(D) ||
      reinterpret_cast<uintptr_t>(workspace) % 128 != 0)
    return FP8FLOW_ERR_ALIGN;
  int sms = 0, st = device(&sms);
  if (st != FP8FLOW_OK) return st;
  return launched(launch_gemm_wgrad(AT, saT, Ma, BT, sbT, Nb, seg_offsets, num_groups, D, d_f32, workspace,
                                    static_cast<cudaStream_t>(stream), sms));
}

int fp8flow_checksum64(const void* buf, int64_t nbytes, uint64_t* out_dev, void* stream) {
  if (nbytes < 0) return FP8FLOW_ERR_SHAPE;
  if (!out_dev || (nbytes > 0 && !buf)) return FP8FLOW_ERR_NULL;
  if (nbytes > 0 && !aligned16(buf)) return FP8FLOW_ERR_ALIGN;
  int sms = 0, st = device(&sms);
  if (st != FP8FLOW_OK) return st;
  return launched(launch_checksum64(buf, nbytes, out_dev, static_cast<cudaStream_t>(stream), sms));
}

// ------------------------------------------------------------------------------------- NEXT-3
namespace {
typedef int (*PFN_cuMemGetAddressRange)(unsigned long long*, size_t*, unsigned long long);

int peer_table_ok(const void* const* tab, int32_t n, bool need16) {
  if (!tab) return FP8FLOW_ERR_NULL;
  for (int r = 0; r < n; ++r) {
    if (!tab[r]) return FP8FLOW_ERR_NULL;
    if (need16 && !aligned16(tab[r])) return FP8FLOW_ERR_ALIGN;
  }
  return FP8FLOW_OK;
}
}  // namespace

int fp8flow_ipc_get_handle(const void* dev_ptr, void* handle_out, int64_t* offset_out) {
  static_assert(sizeof(cudaIpcMemHandle_t) == FP8FLOW_IPC_HANDLE_BYTES, "IPC handle size");
  if (!dev_ptr || !handle_out || !offset_out) return FP8FLOW_ERR_NULL;
  static PFN_cuMemGetAddressRange get_range = nullptr;
  if (!get_range) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qres;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &qres);
    if (e != cudaSuccess || qres != cudaDriverEntryPointSuccess || !p) return fail_cuda(e != cudaSuccess ? e : cudaErrorNotSupported);
    get_range = reinterpret_cast<PFN_cuMemGetAddressRange>(p);
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<unsigned long long>(dev_ptr)) != 0) return fail_cuda(cudaErrorInvalidValue);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return fail_cuda(e);
  memcpy(handle_out, &h, sizeof(h));
  *offset_out = static_cast<int64_t>(reinterpret_cast<unsigned long long>(dev_ptr) - base);
  return FP8FLOW_OK;
}

int fp8flow_ipc_open(const void* handle, void** base_out) {
  if (!handle || !base_out) return FP8FLOW_ERR_NULL;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? FP8FLOW_OK : fail_cuda(e);
}

int fp8flow_ipc_close(void* base) {
  if (!base) return FP8FLOW_ERR_NULL;
  cudaError_t e = cudaIpcCloseMemHandle(base);
  return e == cudaSuccess ? FP8FLOW_OK : fail_cuda(e);
}

int fp8flow_peer_barrier(void* const* peer_signal, int32_t rank, int32_t n, int32_t* status, uint32_t timeout_ms,
                         void* stream) {
  if (n < 1 || n > FP8FLOW_MAX_RANKS || rank < 0 || rank >= n) return FP8FLOW_ERR_ARG;
  int st = peer_table_ok(peer_signal, n, false);
  if (st != FP8FLOW_OK) return st;
  int sms = 0;
  if ((st = device(&sms)) != FP8FLOW_OK) return st;
  return launched(launch_peer_barrier(peer_signal, rank, n, status, timeout_ms, static_cast<cudaStream_t>(stream)));
}

int fp8flow_peer_gather(const void* const* peer_src, int32_t n, int64_t bytes_per_rank, void* dst,
                        const int32_t* status, void* stream) {
  if (n < 1 || n > FP8FLOW_MAX_RANKS) return FP8FLOW_ERR_ARG;
  if (bytes_per_rank < 0 || bytes_per_rank % 4 != 0) return FP8FLOW_ERR_SHAPE;
  if (bytes_per_rank == 0) return FP8FLOW_OK;
  int st = peer_table_ok(peer_src, n, true);
  if (st != FP8FLOW_OK) return st;
  if (!dst) return FP8FLOW_ERR_NULL;
  if (!aligned16(dst)) return FP8FLOW_ERR_ALIGN;
  int sms = 0;
  if ((st = device(&sms)) != FP8FLOW_OK) return st;
  return launched(
      launch_peer_gather(peer_src, n, bytes_per_rank, dst, status, static_cast<cudaStream_t>(stream), sms));
}

int fp8flow_dispatch_permute_pad(const uint8_t* const* peer_q, const uint8_t* const* peer_s, int64_t ld_s_tok,
                                 int32_t n, int64_t tokens_per_rank, int64_t hidden, const int32_t* row_map,
                                 int32_t top_k, const int32_t* src_of_row, const int32_t* expert_offsets,
                                 int32_t num_local_experts, int64_t max_rows, uint8_t* q_out, uint8_t* s_out,
                                 int32_t kernel, const int32_t* status, void* stream) {
  if (n < 1 || n > FP8FLOW_MAX_RANKS) return FP8FLOW_ERR_ARG;
  if (kernel < FP8FLOW_DISPATCH_AUTO || kernel > FP8FLOW_DISPATCH_REGISTER) return FP8FLOW_ERR_ARG;
  if (top_k < 1 || top_k > 16 || num_local_experts < 1 || num_local_experts > 1024) return FP8FLOW_ERR_ARG;
  if (tokens_per_rank < 0 || hidden <= 0 || hidden % 128 != 0 || max_rows < 0) return FP8FLOW_ERR_SHAPE;
  if (ld_s_tok < tokens_per_rank) return FP8FLOW_ERR_SHAPE;
  if (tokens_per_rank * n > INT32_MAX) return FP8FLOW_ERR_SHAPE;
  if (tokens_per_rank == 0) return FP8FLOW_OK;  // no tokens: every expert is empty, no rows to write
  int st = peer_table_ok(reinterpret_cast<const void* const*>(peer_q), n, true);
  if (st != FP8FLOW_OK) return st;
  if ((st = peer_table_ok(reinterpret_cast<const void* const*>(peer_s), n, false)) != FP8FLOW_OK) return st;
  if (!row_map || !src_of_row || !expert_offsets || !q_out || !s_out) return FP8FLOW_ERR_NULL;
  if (!aligned16(q_out)) return FP8FLOW_ERR_ALIGN;
  int sms = 0;
  if ((st = device(&sms)) != FP8FLOW_OK) return st;
  return launched(launch_dispatch_permute_pad(peer_q, peer_s, ld_s_tok, n, tokens_per_rank, hidden, row_map, top_k,
                                              src_of_row, expert_offsets, num_local_experts, max_rows, q_out, s_out,
                                              kernel, status, static_cast<cudaStream_t>(stream), sms));
}

int fp8flow_combine_unpermute(const void* const* peer_x, const int32_t* const* peer_row_map, int32_t n,
                              int64_t hidden, const int32_t* topk_idx, int32_t experts_per_rank, const float* probs,
                              int64_t token_begin, int64_t num_tokens, int32_t top_k, void* y_bf16,
                              const int32_t* status, void* stream) {
  if (n < 1 || n > FP8FLOW_MAX_RANKS || experts_per_rank < 1) return FP8FLOW_ERR_ARG;
  if (top_k < 1 || top_k > 16) return FP8FLOW_ERR_ARG;
  if (num_tokens < 0 || token_begin < 0 || hidden <= 0 || hidden % 8 != 0) return FP8FLOW_ERR_SHAPE;
  if (num_tokens == 0) return FP8FLOW_OK;
  int st = peer_table_ok(peer_x, n, true);
  if (st != FP8FLOW_OK) return st;
  if ((st = peer_table_ok(reinterpret_cast<const void* const*>(peer_row_map), n, false)) != FP8FLOW_OK) return st;
  if (!topk_idx || !y_bf16) return FP8FLOW_ERR_NULL;
  if (!aligned16(y_bf16)) return FP8FLOW_ERR_ALIGN;
  int sms = 0;
  if ((st = device(&sms)) != FP8FLOW_OK) return st;
  return launched(launch_combine_unpermute(peer_x, peer_row_map, n, hidden, topk_idx, experts_per_rank, probs,
                                           token_begin, num_tokens, top_k, y_bf16, status,
                                           static_cast<cudaStream_t>(stream), sms));
}

}  // extern "C"
