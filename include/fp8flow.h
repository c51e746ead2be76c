/*
 * fp8flow.h -- C ABI of libfp8flow: the data-parallel hot path of FP8-Flow-MoE
 * ("FP8-Flow-MoE: A Casting-Free FP8 Recipe without Double Quantization Error", arXiv 2511.02302)
 * as hand-written CUDA kernels for NVIDIA B200 (sm_100a).
 *
 * Citations: P:n = line n of the paper's LaTeX source.  Readings of ambiguous passages are the
 * numbered readings R1..R28 of DESIGN.md §3.
 *
 * ------------------------------------------------------------------------------------------
 * Numeric contract (every entry point)
 *   E4M3 code   1 sign | 4 exponent (bias 7) | 3 mantissa bits, MSB first; max 448;
 *               Eq. 10.  Rounding: round-to-nearest, ties to even (R8);
 *               finite overflow saturates to +-448 (R9); the sign of zero is kept (R10).
 *   UE8M0 scale one byte b per 1x128 tile, value 2^(b-127).  b = T + 127 where
 *               T is the least integer with max|x| <= 448 * 2^T over the tile (Eq. 2, read
 *               with a power-of-two scale rounded up, R3), clamped to [-127, 127] (R13); an
 *               all-zero tile gets b = 0 (R11).
 *   Row-wise FP8 tensor: codes q[rows][cols] row-major (cols % 128 == 0) and scales
 *               s[cols/128][ld_s] "MN-major": one contiguous run of ld_s >= rows bytes per
 *               128-wide column tile; s[j][i] is the scale of row i, columns 128j..128j+127.
 *   Segments    an expert's rows [o_e, o_e + m_e) of a permuted buffer; device int32 offsets
 *               seg_offsets[0..num_segs], non-decreasing, every m_e % 16 == 0 and every
 *               o_e % 16 == 0.
 *
 * Memory and execution
 *   All tensor pointers are DEVICE pointers (cudaMalloc / torch CUDA storage) unless stated.
 *   The caller owns every buffer, including workspaces (size queries provided).  The library
 *   never allocates, frees, synchronises or keeps state between calls; it is reentrant.
 *   `stream` is a cudaStream_t (NULL = legacy default stream).  Every call is asynchronous on
 *   that stream; data-dependent sizes (padded rows, segment sizes) stay on the device, so every
 *   call is CUDA-graph capturable.
 *
 * Errors
 *   Arguments are validated synchronously; on error a status is returned and nothing is
 *   launched.  A failed launch returns FP8FLOW_ERR_CUDA and fp8flow_last_cuda_error() gives the
 *   cudaError_t.  Device faults surface at the caller's next synchronisation.  Non-finite
 *   inputs are a precondition violation (not checked on device).  There is no CPU fallback: on
 *   a device that is not sm_100 every compute entry point returns FP8FLOW_ERR_ARCH.
 * ------------------------------------------------------------------------------------------
 */
#ifndef FP8FLOW_H_
#define FP8FLOW_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FP8FLOW_API __attribute__((visibility("default")))
#else
#define FP8FLOW_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FP8FLOW_OK = 0,
  FP8FLOW_ERR_NULL = 1,      /* a required pointer is NULL                                        */
  FP8FLOW_ERR_SHAPE = 2,     /* negative size, cols % 128 != 0, rows % 16 != 0 where required     */
  FP8FLOW_ERR_ALIGN = 3,     /* a pointer or leading dimension is not 16-byte aligned              */
  FP8FLOW_ERR_ARG = 4,       /* top_k / expert range / align / num_segs out of range               */
  FP8FLOW_ERR_WORKSPACE = 5, /* workspace too small                                                */
  FP8FLOW_ERR_ARCH = 6,      /* current device is not sm_100 (B200); no fallback exists            */
  FP8FLOW_ERR_CUDA = 7       /* a CUDA runtime call or launch failed; see fp8flow_last_cuda_error() */
} fp8flow_status_t;

/* Human-readable name of a status code (static storage). */
FP8FLOW_API const char* fp8flow_status_string(int status);
/* cudaError_t of the last FP8FLOW_ERR_CUDA returned on the calling thread (0 if none). */
FP8FLOW_API int fp8flow_last_cuda_error(void);
/* Library version (major*10000 + minor*100 + patch) and the compiled target ("sm_100a"). */
FP8FLOW_API int fp8flow_version(void);
FP8FLOW_API const char* fp8flow_build_target(void);
/* sha256 prefix (16 hex digits) of the sources the library was compiled from (build.py); the Python
 * binding refuses a library whose hash differs from the sources next to it (a stale binary). */
FP8FLOW_API const char* fp8flow_source_hash(void);
/* FP8FLOW_OK if the current CUDA device is sm_100, else FP8FLOW_ERR_ARCH / FP8FLOW_ERR_CUDA. */
FP8FLOW_API int fp8flow_device_check(void);

/* ==========================================================================================
 * A1  Entry quantization, BF16 -> E4M3 with 1x128 power-of-two scales.
 *     Eq. 2, Eq. 3, s = 2^T; the single forward cast at the entry
 *     point and its backward twin on dY ("from 12 to 2" P:28; R27).
 *   x_bf16  [rows][cols] BF16, row-major, 16-byte aligned             (read)
 *   q       [rows][cols] E4M3 codes, 16-byte aligned                  (written)
 *   s       [cols/128][ld_s] UE8M0 scale bytes, MN-major, 16-byte aligned; ld_s >= rows,
 *           ld_s % 16 == 0 (written for rows [0, rows) of every tile column; bytes rows..ld_s-1
 *           untouched)
 *   rows >= 0 (0 = no-op), cols > 0 and cols % 128 == 0.  A misaligned pointer returns
 *   FP8FLOW_ERR_ALIGN before anything is launched.
 *   Result: q[i][j] = E4M3_RNE(x[i][j] * 2^-T[i][j/128]) (the product is exact; |.| <= 448).
 * ========================================================================================== */
FP8FLOW_API int fp8flow_quantize_rowwise(const void* x_bf16, int64_t rows, int64_t cols, uint8_t* q, uint8_t* s, int64_t ld_s,
                             void* stream);

/* ==========================================================================================
 * A2  Scaling-aware FP8 transpose (Algorithm 1; derivation P:173-200).
 *     Row-wise FP8 -> column-wise FP8 for the wgrad GEMM without dequantization:
 *     for each segment e and each block (ib, jb) of rows o_e+128ib.. (the last block of a
 *     segment may be partial, R14; blocks never straddle segments, R15) x columns 128jb..+127:
 *        T_max = max over the block's rows of T[i][jb]                 (R6)
 *        sT_e[ib][j] = T_max for all 128 columns j of the block
 *        qT_e[j][i - o_e] = E4M3_RNE(decode(q[i][j]) * 2^-(T_max - T[i][jb]))   (R5, R7)
 *     i.e. the exponent field is lowered by k = T_max - T_row; codes that leave the normal range
 *     are re-rounded into the subnormal grid (the only loss, "provided that no overflow or
 *     underflow occurs").
 *   q, s, ld_s   row-wise input [rows][cols] + MN-major scales (ld_s % 16 == 0, ld_s >= rows)
 *   rows % 16 == 0, cols % 128 == 0
 *   seg_offsets  device int32 [num_segs + 1], or NULL = one segment [0, rows); 1 <= num_segs <= 1024
 *   qT           output codes; segment e occupies bytes [cols*o_e, cols*(o_e + m_e)) as a
 *                row-major [cols][m_e] matrix (physically transposed, R23).  16-byte aligned.
 *   sT           output scales; segment e occupies rows [P_e, P_e + ceil(m_e/128)) of a
 *                [*][cols] byte matrix, P_e = sum_{e'<e} ceil(m_e'/128).  Capacity needed:
 *                cols * (rows/128 + num_segs) bytes.  16-byte aligned.
 * ========================================================================================== */
FP8FLOW_API int fp8flow_scaling_aware_transpose(const uint8_t* q, const uint8_t* s, int64_t ld_s, int64_t rows, int64_t cols,
                                    const int32_t* seg_offsets, int32_t num_segs, uint8_t* qT, uint8_t* sT,
                                    void* stream);

/* Naive comparator: dequantize to BF16 -> transpose -> column-wise requantize with
 * fresh pow2 scales per (column, 128-row block of a segment).  Same arguments and output layout as
 * A2 plus a device workspace of fp8flow_naive_workspace_bytes() bytes.  Benchmark comparator
 * only: it exhibits the second rounding the paper calls double quantization error (Eq. 9). */
FP8FLOW_API size_t fp8flow_naive_workspace_bytes(int64_t rows, int64_t cols, int32_t num_segs);
FP8FLOW_API int fp8flow_naive_transpose(const uint8_t* q, const uint8_t* s, int64_t ld_s, int64_t rows, int64_t cols,
                            const int32_t* seg_offsets, int32_t num_segs, uint8_t* qT, uint8_t* sT, void* ws,
                            size_t ws_bytes, void* stream);

/* ==========================================================================================
 * A3  Fused permute + padding: plan, then move.
 *
 * fp8flow_permute_plan -- routing plan for the local experts [expert_begin, expert_begin + E_loc):
 *   topk_idx        device int32 [num_tokens][top_k] global expert ids, distinct per token
 *   align           padding multiple, 16 in the paper; any value in [1, 1024]
 *   row_map         device int32 [num_tokens][top_k] (written): output row of pair (t, k), or -1
 *                   when topk_idx[t][k] is not a local expert
 *   src_of_row      device int32 [max_rows] (written for rows < expert_offsets[E_loc]): source
 *                   token of each output row, -1 for PAD rows
 *   expert_offsets  device int32 [E_loc + 1] (written): expert e's rows are
 *                   [offsets[e], offsets[e+1]), count_e real rows in ascending token order then
 *                   ceil(count_e/align)*align - count_e PAD rows (R16)
 *   max_rows        capacity; num_tokens*top_k + E_loc*(align-1) always suffices.  If the padded
 *                   total exceeds it, rows beyond are dropped (row_map = -1, src_of_row not
 *                   written past max_rows), expert_offsets still hold the true padded offsets
 *                   (so offsets[E_loc] > max_rows) and the workspace's first int32 is set to 1
 *                   (else 0) -- readable by the caller after sync.  Every consumer of the plan
 *                   (permute_pad, dispatch, SwiGLU via rows_dev) clamps the row count to its
 *                   max_rows / rows_max, so an overflowed plan never writes out of bounds.
 *   ws              device workspace of fp8flow_permute_workspace_bytes() bytes
 *   1 <= top_k <= 16, 1 <= E_loc <= 1024, num_tokens >= 0.  Deterministic: the plan depends only
 *   on topk_idx (no atomics decide an order).
 * ========================================================================================== */
FP8FLOW_API size_t fp8flow_permute_workspace_bytes(int64_t num_tokens, int32_t top_k, int32_t num_local_experts);
FP8FLOW_API int fp8flow_permute_plan(const int32_t* topk_idx, int64_t num_tokens, int32_t top_k, int32_t expert_begin,
                         int32_t num_local_experts, int32_t align, int32_t* row_map, int32_t* src_of_row,
                         int64_t max_rows, int32_t* expert_offsets, void* ws, size_t ws_bytes, void* stream);

/* fp8flow_permute_pad -- move row-wise FP8 tokens into the padded expert-major buffer in one pass:
 *   q_out[r] = q_tok[src_of_row[r]], s_out[j][r] = s_tok[j][src_of_row[r]] for r < R =
 *   min(expert_offsets[E_loc], max_rows); PAD rows get code 0x00 and scale byte 0x00 (R17, R11).
 *   Each token is read once and written to all of its local rows (row_map from the plan gives a
 *   token's rows), i.e. the one-rank case of fp8flow_dispatch_permute_pad.
 *   q_tok [num_tokens][hidden] + s_tok [hidden/128][ld_s_tok]  (row-wise FP8, as from A1)
 *   row_map [num_tokens][top_k], src_of_row [max_rows], expert_offsets [E_loc + 1]: the plan's
 *   q_out [max_rows][hidden], s_out [hidden/128][max_rows]       (rows >= R untouched)
 *   hidden % 128 == 0; q_tok, q_out 16-byte aligned; max_rows % 16 == 0; 1 <= top_k <= 16;
 *   num_tokens == 0 is a no-op (every expert is empty). */
FP8FLOW_API int fp8flow_permute_pad(const uint8_t* q_tok, const uint8_t* s_tok, int64_t ld_s_tok, int64_t num_tokens,
                        int64_t hidden, const int32_t* row_map, int32_t top_k, const int32_t* src_of_row,
                        const int32_t* expert_offsets, int32_t num_local_experts, int64_t max_rows, uint8_t* q_out,
                        uint8_t* s_out, void* stream);

/* ==========================================================================================
 * A4  Fused unpermute + unpadding, BF16 at the second boundary (R22):
 *     y[t][h] = BF16_RNE( sum over k = 0..top_k-1 with row_map[t][k] >= 0 of
 *                         probs[t][k] * x[row_map[t][k]][h] )
 *     accumulated in fp32 as acc = fmaf(p, x, acc) from +0 in k order (acc + x when probs is
 *     NULL); PAD rows are never read; tokens without a local expert get +0 (R21).
 *   x_bf16 [*][hidden] BF16 expert-major rows; row_map [num_tokens][top_k]; probs fp32
 *   [num_tokens][top_k] or NULL; y_bf16 [num_tokens][hidden].  hidden % 8 == 0, 16-byte aligned
 *   x and y, 1 <= top_k <= 16.
 * ========================================================================================== */
FP8FLOW_API int fp8flow_unpermute_unpad(const void* x_bf16, int64_t hidden, const int32_t* row_map, const float* probs,
                            int64_t num_tokens, int32_t top_k, void* y_bf16, void* stream);

/* ==========================================================================================
 * A5  Fused SwiGLU + quantization: from the BF16 fc1 output (R19)
 *     y = silu(a) * b = a*b / (1 + e^-a), a = h[:, :ffn] (gate), b = h[:, ffn:] (R18), then A1's
 *     1x128 quantization along ffn.  Reference value: fp64 evaluation rounded once to fp32 (R20);
 *     acceptance: codes within 1 E4M3 ULP on <= 1e-4 of elements, scale bytes identical.
 *   h_bf16  [rows_max][2*ffn] BF16, 16-byte aligned
 *   rows_dev device int32 holding the actual row count (e.g. &expert_offsets[E_loc]), or NULL
 *           for rows_max rows; a larger value (an overflowed plan's true total) is clamped to rows_max
 *   q       [rows_max][ffn] E4M3 codes; s [ffn/128][ld_s] MN-major, ld_s >= rows_max, % 16 == 0
 *   ffn % 128 == 0.
 * ========================================================================================== */
FP8FLOW_API int fp8flow_swiglu_quant(const void* h_bf16, int64_t rows_max, const int32_t* rows_dev, int64_t ffn, uint8_t* q,
                         uint8_t* s, int64_t ld_s, void* stream);

/* ==========================================================================================
 * NEXT-1  Fused SwiGLU backward + quantization: the activation's gradient at the BF16 boundary of
 *     the backward pass (R31), from the saved fc1 output h = [a | b] and the upstream
 *     gradient dA (fc2 dgrad output):
 *        da = dA * b * silu'(a),  silu'(a) = sig(a) (1 + a (1 - sig(a))),   db = dA * silu(a)
 *     dH = [da | db] quantized row-wise (A1's 1x128 tiles along 2*ffn) for the fc1 dgrad/wgrad
 *     GEMMs.  Reference: fp64 evaluation rounded once to fp32; acceptance as A5.
 *   h_bf16  [rows_max][2*ffn] BF16, dA_bf16 [rows_max][ffn] BF16 (16-byte aligned)
 *   rows_dev device int32 actual row count or NULL (rows_max)
 *   q       [rows_max][2*ffn] E4M3 codes; s [2*ffn/128][ld_s] MN-major, ld_s >= rows_max, % 16 == 0
 *   ffn % 128 == 0.
 * ========================================================================================== */
FP8FLOW_API int fp8flow_swiglu_bwd_quant(const void* h_bf16, const void* dA_bf16, int64_t rows_max,
                                         const int32_t* rows_dev, int64_t ffn, uint8_t* q, uint8_t* s,
                                         int64_t ld_s, void* stream);

/* ==========================================================================================
 * NEXT-1  Dual-output fusions (R32): one read of the BF16 input
 *     produces both the row-wise FP8 tensor (Fprop/Dgrad operand) and its column-wise
 *     scaling-aware transpose (Wgrad operand) per segment.  The result is by definition the
 *     composition: (q, s) = A1(x) [resp. A5(h)], (qT, sT) = A2(q, s, seg_offsets) -- bit-identical
 *     to calling the two entry points in sequence, with one fewer pass over q.
 *
 *   fp8flow_quantize_dual: x_bf16 [rows][cols] (A1's input); rows % 16 == 0, cols % 128 == 0.
 *   fp8flow_swiglu_quant_dual: h_bf16 [rows_max][2*ffn] (A5's input); the output columns are ffn.
 *     rows_dev: actual row count (device int32) or NULL, used only when seg_offsets is NULL.
 *   seg_offsets  device int32 [num_segs + 1] (segment lengths multiples of 16), or NULL = one
 *                segment [0, rows); 1 <= num_segs <= 1024.  For the SwiGLU variant the last
 *                offset is the actual row count.
 *   q, s, ld_s   row-wise output as A1 / A5 (s MN-major [cols/128][ld_s], ld_s >= rows, % 16 == 0)
 *   qT, sT       column-wise output as A2 (same capacities and per-segment placement).
 *   All pointers 16-byte aligned.
 * ========================================================================================== */
FP8FLOW_API int fp8flow_quantize_dual(const void* x_bf16, int64_t rows, int64_t cols, const int32_t* seg_offsets,
                                      int32_t num_segs, uint8_t* q, uint8_t* s, int64_t ld_s, uint8_t* qT,
                                      uint8_t* sT, void* stream);
FP8FLOW_API int fp8flow_swiglu_quant_dual(const void* h_bf16, int64_t rows_max, const int32_t* rows_dev,
                                          int64_t ffn, const int32_t* seg_offsets, int32_t num_segs, uint8_t* q,
                                          uint8_t* s, int64_t ld_s, uint8_t* qT, uint8_t* sT, void* stream);

/* fp8flow_permute_pad_dual -- the A3 move fused with A2 (NEXT-1 dual output, R37): one
 *     gather of each 128 x 128 block of the padded expert-major tensor produces both the row-wise
 *     output of fp8flow_permute_pad (X_perm, the Fprop operand) and its scaling-aware transpose per
 *     expert (A2 with segments = expert_offsets, the Wgrad operand).  By
 *     definition bit-identical to fp8flow_permute_pad followed by fp8flow_scaling_aware_transpose(
 *     q_out, s_out, ld_s = max_rows, rows = R, seg_offsets = expert_offsets, num_segs = E_loc),
 *     without the second pass over X_perm.
 *   q_tok, s_tok, ld_s_tok, num_tokens, hidden: as fp8flow_permute_pad (row-wise FP8 tokens)
 *   src_of_row, expert_offsets, num_local_experts, max_rows: the plan's (fp8flow_permute_plan), made
 *                with align % 16 == 0 (A2's segment lengths are multiples of 16); offsets past
 *                max_rows (an overflowed plan) are clamped to it
 *   q_out [max_rows][hidden], s_out [hidden/128][max_rows]: as fp8flow_permute_pad
 *   qT, sT: as fp8flow_scaling_aware_transpose (capacity hidden * max_rows and
 *           hidden * (max_rows/128 + E_loc) bytes)
 *   hidden % 128 == 0, max_rows % 16 == 0, ld_s_tok % 4 == 0 (scale bytes are fetched as the 4-byte
 *   words holding them); q_tok, s_tok, q_out, s_out, qT, sT, src_of_row 16-byte aligned;
 *   num_tokens == 0 is a no-op. */
FP8FLOW_API int fp8flow_permute_pad_dual(const uint8_t* q_tok, const uint8_t* s_tok, int64_t ld_s_tok,
                                         int64_t num_tokens, int64_t hidden, const int32_t* src_of_row,
                                         const int32_t* expert_offsets, int32_t num_local_experts, int64_t max_rows,
                                         uint8_t* q_out, uint8_t* s_out, uint8_t* qT, uint8_t* sT, void* stream);

/* ==========================================================================================
 * NEXT-2  Block-scaled FP8 GEMM, the consumer of the casting-free path (
 *     P:43): the row-wise (A1/A3/A5) or column-wise (A2) FP8 outputs with their
 *     1x128 UE8M0 scales feed the 5th-generation tensor cores directly (tcgen05.mma
 *     kind::mxf8f6f4.block_scale; a 1x128 power-of-two scale is replicated to the four 1x32 MX
 *     blocks, losslessly).  DESIGN.md R33.
 *        D[m][n] = sum_k dec(A[m][k]) 2^(sa[k/128][m] - 127) * dec(B_g[n][k]) 2^(sb_g[k/128][n] - 127)
 *     accumulated in fp32 by the tensor core; D stored as fp32 or BF16 (RNE).
 *   A       [M][K] E4M3, K-major (row-major with K contiguous); sa [K/128][ld_sa] MN-major
 *   B       [num_groups][N][K] E4M3, K-major; sb [num_groups][K/128][ld_sb] MN-major
 *   seg_offsets device int32 [num_groups + 1] splitting the rows of A into groups (experts;
 *           segment lengths multiples of 16), or NULL = one group of M rows; 1 <= num_groups <= 512
 *   D       [M][N] fp32 (d_f32 != 0) or BF16; rows outside every group are not written
 *   M % 16 == 0, N % 256 == 0, K % 128 == 0, ld_sa >= M, ld_sb >= N, both % 16 == 0;
 *   all pointers 16-byte aligned, A and B 1024-byte aligned recommended.
 * ========================================================================================== */
FP8FLOW_API int fp8flow_gemm_blockscaled(const uint8_t* A, const uint8_t* sa, int64_t ld_sa, const uint8_t* B,
                                         const uint8_t* sb, int64_t ld_sb, int64_t M, int64_t N, int64_t K,
                                         const int32_t* seg_offsets, int32_t num_groups, void* D, int32_t d_f32,
                                         void* stream);

/* NEXT-2 Wgrad: groups split K (each expert's tokens): D_e = AT_e * BT_e^T, i.e.
 *        D_e[m][n] = sum_{k < m_e} dec(AT_e[m][k]) 2^(saT[P_e + k/128][m] - 127) * dec(BT_e[n][k]) 2^(sbT[P_e + k/128][n] - 127)
 *     with both operands exactly as A2 (fp8flow_scaling_aware_transpose) leaves them for the same
 *     segments: AT_e = [Ma][m_e] at byte offset Ma*o_e, saT rows P_e .. P_e + ceil(m_e/128) - 1
 *     (P_e = sum_{e'<e} ceil(m_e'/128)), likewise BT/sbT with Nb.  Example: dW1_e = dH_e^T X_e with
 *     AT = A2(dH), BT = A2(X_perm).  Segment lengths multiples of 16 (a partial last K block is
 *     zero-padded); a group with no rows gets D_e = 0.
 *   D  [num_groups][Ma][Nb] fp32 (d_f32 != 0) or BF16.  Ma % 128 == 0, Nb % 256 == 0,
 *   1 <= num_groups <= 512, seg_offsets device int32 [num_groups + 1] (required).
 *   workspace: caller-owned device memory, 128-byte aligned, >= fp8flow_gemm_wgrad_workspace_bytes
 *     (num_groups) bytes (the per-group TMA descriptors, written by the call on `stream`; it must
 *     not be shared with a concurrent call).  Too small -> FP8FLOW_ERR_WORKSPACE.
 * ========================================================================================== */
FP8FLOW_API int64_t fp8flow_gemm_wgrad_workspace_bytes(int32_t num_groups);
FP8FLOW_API int fp8flow_gemm_wgrad(const uint8_t* AT, const uint8_t* saT, int64_t Ma, const uint8_t* BT,
                                   const uint8_t* sbT, int64_t Nb, const int32_t* seg_offsets, int32_t num_groups,
                                   void* D, int32_t d_f32, void* workspace, int64_t workspace_bytes, void* stream);

/* ==========================================================================================
 * NEXT-3  Expert-parallel FP8 dispatch / BF16 combine over peer memory (
 *     DESIGN.md R34).  The MoE layer's stages are routing -> dispatch -> permutation -> experts ->
 *     unpermutation -> combination; dispatch ships the row-wise FP8 format, codes
 *     and scales together, and the combine is BF16.  Rank r of n owns tokens
 *     [r*T_per_rank, (r+1)*T_per_rank) (global token id) and experts [r*E_per, (r+1)*E_per).
 *
 *   Peer tables: `peer_*` arguments are HOST arrays of n device pointers, entry r = rank r's
 *   buffer as mapped in the calling process (CUDA IPC via fp8flow_ipc_* on a multi-GPU node, or
 *   plain device pointers when several ranks share one device).  They are copied by value into
 *   the launch (CUDA-graph capturable); 1 <= n <= FP8FLOW_MAX_RANKS.  Every rank's buffers must
 *   be complete before a peer reads them: call fp8flow_peer_barrier on the same stream first.
 *   Buffers read by peers must not be overwritten until the peers are done (next barrier).
 * ========================================================================================== */
#define FP8FLOW_MAX_RANKS 64
#define FP8FLOW_IPC_HANDLE_BYTES 64

/* CUDA IPC plumbing (host calls, synchronous).  fp8flow_ipc_get_handle exports the allocation that
 * contains dev_ptr: handle_out receives FP8FLOW_IPC_HANDLE_BYTES opaque bytes and *offset_out the
 * byte offset of dev_ptr inside that allocation (caching allocators sub-allocate).
 * fp8flow_ipc_open maps a handle exported by ANOTHER process (peer access enabled lazily) and
 * returns the allocation's base in *base_out (add the exporter's offset); fp8flow_ipc_close unmaps
 * it.  Errors: FP8FLOW_ERR_NULL, FP8FLOW_ERR_CUDA. */
FP8FLOW_API int fp8flow_ipc_get_handle(const void* dev_ptr, void* handle_out, int64_t* offset_out);
FP8FLOW_API int fp8flow_ipc_open(const void* handle, void** base_out);
FP8FLOW_API int fp8flow_ipc_close(void* base);

/* fp8flow_peer_barrier -- device-side barrier of n ranks over peer flags (no host sync).
 *   peer_signal  host array [n] of device pointers; entry d = rank d's signal buffer of n + 1
 *                uint32, zero-initialised once by its owner before first use (slot s = the last
 *                epoch rank s announced; slot n = the owner's epoch counter, advanced on device)
 *   status       device int32 or NULL: 0 on success, 1 if the peers did not arrive within
 *                timeout_ms (the kernel then returns instead of hanging).
 * Every rank must call it the same number of times. */
FP8FLOW_API int fp8flow_peer_barrier(void* const* peer_signal, int32_t rank, int32_t n, int32_t* status,
                                     uint32_t timeout_ms, void* stream);

/* Gating on the barrier's status (gather, dispatch, combine): `status` is a device int32 or NULL.
 * When non-NULL and nonzero at the time the kernel runs (the preceding fp8flow_peer_barrier on the
 * stream timed out, so a peer's buffers may be incomplete), the kernel writes NOTHING and returns;
 * the caller must read status after the step and discard its outputs.  NULL = ungated. */

/* fp8flow_peer_gather -- all-gather by pulls: dst[r*bytes_per_rank ...] = peer_src[r][0 .. bytes_per_rank)
 * (e.g. every rank's topk_idx for the dispatch plan).  bytes_per_rank % 4 == 0 (16-byte copies
 * when bytes_per_rank % 16 == 0, else 4-byte words), all pointers 16-byte aligned, dst device
 * [n*bytes_per_rank].  status: the barrier gate above. */
FP8FLOW_API int fp8flow_peer_gather(const void* const* peer_src, int32_t n, int64_t bytes_per_rank, void* dst,
                                    const int32_t* status, void* stream);

/* fp8flow_dispatch_permute_pad -- the receive side of the FP8 dispatch fused with A3's move: every
 *   token routed to one of this rank's experts is read ONCE from its owner (codes + scale bytes)
 *   and written to all of its local expert rows; PAD rows get code 0x00 / scale 0x00.  The result
 *   is bit-identical to fp8flow_permute_pad on the rank-order concatenation of all ranks' tokens.
 *   peer_q    host array [n]: rank r's codes [tokens_per_rank][hidden] (as from A1)
 *   peer_s    host array [n]: rank r's scales [hidden/128][ld_s_tok] (MN-major, as from A1)
 *   row_map, src_of_row, expert_offsets: from fp8flow_permute_plan over the GATHERED topk_idx
 *             [n*tokens_per_rank][top_k] with this rank's expert range (global token ids)
 *   q_out [max_rows][hidden], s_out [hidden/128][max_rows] (rows >= expert_offsets[E_loc] untouched)
 *   hidden % 128 == 0, q pointers 16-byte aligned, 1 <= top_k <= 16, ld_s_tok >= tokens_per_rank.
 *   kernel    which kernel (identical results): FP8FLOW_DISPATCH_ENGINE = bulk-copy engine
 *             (cp.async.bulk token pulls into shared memory, bulk stores per row; verified for
 *             peers on the calling device; FP8FLOW_ERR_CUDA if its shared-memory ring cannot hold
 *             the shape, roughly hidden > 9K at DSv3 token counts), FP8FLOW_DISPATCH_REGISTER =
 *             register copies with plain 128-bit loads (valid on every peer mapping and shape),
 *             FP8FLOW_DISPATCH_AUTO = the engine when every peer_q lives on the calling device and
 *             the ring fits, else register copies.  Other values: FP8FLOW_ERR_ARG.
 *   status    the barrier gate above. */
#define FP8FLOW_DISPATCH_AUTO 0
#define FP8FLOW_DISPATCH_ENGINE 1
#define FP8FLOW_DISPATCH_REGISTER 2
FP8FLOW_API int fp8flow_dispatch_permute_pad(const uint8_t* const* peer_q, const uint8_t* const* peer_s,
                                             int64_t ld_s_tok, int32_t n, int64_t tokens_per_rank, int64_t hidden,
                                             const int32_t* row_map, int32_t top_k, const int32_t* src_of_row,
                                             const int32_t* expert_offsets, int32_t num_local_experts,
                                             int64_t max_rows, uint8_t* q_out, uint8_t* s_out, int32_t kernel,
                                             const int32_t* status, void* stream);

/* fp8flow_combine_unpermute -- the owner side of the BF16 combine fused with A4: for the caller's
 *   tokens t (global id token_begin + t),
 *     y[t][h] = BF16_RNE( sum_k p[t][k] * x_d[row_map_d[token_begin + t][k]][h] ),
 *     d = topk_idx[t][k] / experts_per_rank,
 *   fp32 fmaf in k order from +0 (p = 1 when probs is NULL) -- A4's arithmetic, so the result is
 *   bit-identical to fp8flow_unpermute_unpad over the concatenated expert outputs.  Terms whose
 *   expert id is outside [0, n*experts_per_rank) or whose row is -1 are skipped.
 *   peer_x       host array [n]: rank d's expert outputs, BF16 [rows_d][hidden], 16-byte aligned
 *   peer_row_map host array [n]: rank d's plan row_map [n*tokens_per_rank][top_k] (device int32)
 *   topk_idx [num_tokens][top_k], probs fp32 [num_tokens][top_k] or NULL, y BF16 [num_tokens][hidden].
 *   hidden % 8 == 0, 1 <= top_k <= 16.  status: the barrier gate above. */
FP8FLOW_API int fp8flow_combine_unpermute(const void* const* peer_x, const int32_t* const* peer_row_map, int32_t n,
                                          int64_t hidden, const int32_t* topk_idx, int32_t experts_per_rank,
                                          const float* probs, int64_t token_begin, int64_t num_tokens, int32_t top_k,
                                          void* y_bf16, const int32_t* status, void* stream);

/* Verification checksum (DESIGN.md §4 C11): *out_dev = sum_i buf[i] * (i * 0x9E3779B97F4A7C15 + 1)
 * mod 2^64 over nbytes bytes.  buf 16-byte aligned; out_dev a device uint64. */
FP8FLOW_API int fp8flow_checksum64(const void* buf, int64_t nbytes, uint64_t* out_dev, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FP8FLOW_H_ */
