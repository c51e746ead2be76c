// permute.cu -- A3 fused permute + padding (plan + move) and A4 fused unpermute + unpadding.
//
// Paper: P:319 ("each expert's input must contain a multiple of 16 entries"), P:322 ("a thread-
// block mapping scheme that dynamically computes the target offset in the padded layout while
// streaming reordered input elements from global memory"; the same fusion for unpermute +
// unpadding), P:245 (routing -> dispatch -> permutation -> experts -> unpermutation -> combine).
// Readings: R16 experts ascending, tokens ascending inside an expert, PAD rows at
// the end of each expert; R17 PAD = code 0x00 + scale byte 0x00; R21 gates applied at unpermute,
// fp32 fused multiply-add in k order, BF16 RNE output.
//
// Plan (deterministic, no CUB, no host sync):
//   K1 plan_count : per 256-token chunk, a shared-memory histogram over local experts
//   K2 plan_scan  : one CTA: per-expert exclusive scan over chunks (-> chunk bases) and counts;
//                   padded sizes; exclusive scan over experts -> expert_offsets; PAD rows of
//                   src_of_row = -1
//   K3 plan_rank  : per chunk, a (expert x token) bit matrix in shared memory; the rank of a
//                   token inside an expert is a popcount over the lower tokens' bits, so
//                   rows = offset[e] + chunk_base[e] + rank is stable in token order.
// Move: CTA item = 32 consecutive output rows; each warp streams 4 rows with 128-bit loads and
// stores (8 in flight per lane); the 32 rows' scale bytes are gathered per 1x128 tile and written
// as 32-byte MN-major runs.
#include "common.cuh"
#include "kernels.h"

namespace fp8flow {

constexpr int kChunk = 256;        // tokens per plan chunk (one thread per token)

size_t permute_workspace_bytes(int64_t num_tokens, int32_t num_local_experts) {
  const int64_t chunks = (num_tokens + kChunk - 1) / kChunk;
  return 256 + 4 * static_cast<size_t>(chunks) * num_local_experts + 4 * static_cast<size_t>(num_local_experts);
}

__global__ void __launch_bounds__(kChunk) plan_count_kernel(const int32_t* __restrict__ topk_idx, int64_t T, int K,
                                                            int e0, int E_loc, int32_t* __restrict__ chunk_counts) {
  extern __shared__ int32_t hist[];
  for (int i = threadIdx.x; i < E_loc; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kChunk + threadIdx.x;
  if (t < T) {
    for (int k = 0; k < K; ++k) {
      const int e = topk_idx[t * K + k] - e0;
      if (e >= 0 && e < E_loc) atomicAdd(&hist[e], 1);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < E_loc; i += blockDim.x)
    chunk_counts[static_cast<int64_t>(blockIdx.x) * E_loc + i] = hist[i];
}

__global__ void __launch_bounds__(1024) plan_scan_kernel(int32_t* __restrict__ chunk_counts, int64_t n_chunks,
                                                         int E_loc, int align, int32_t* __restrict__ expert_offsets,
                                                         int32_t* __restrict__ counts_out,
                                                         int32_t* __restrict__ src_of_row, int64_t max_rows,
                                                         int32_t* __restrict__ status) {
  __shared__ int32_t warp_tot[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // one expert per thread (E_loc <= 1024)
  int count = 0;
  if (tid < E_loc) {
    for (int64_t c = 0; c < n_chunks; ++c) {
      const int64_t idx = c * E_loc + tid;
      const int v = chunk_counts[idx];
      chunk_counts[idx] = count;  // exclusive base of this chunk inside the expert
      count += v;
    }
  }
  const int padded = (count + align - 1) / align * align;
  int incl = padded;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += n;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += warp_tot[w];
  const int excl = base + incl - padded;
  if (tid < E_loc) {
    expert_offsets[tid] = excl;
    counts_out[tid] = count;
    if (tid == E_loc - 1) {
      expert_offsets[E_loc] = excl + padded;
      *status = (excl + padded > max_rows) ? 1 : 0;
    }
    for (int r = excl + count; r < excl + padded; ++r)
      if (r < max_rows) src_of_row[r] = -1;  // PAD rows
  }
}

__global__ void __launch_bounds__(kChunk) plan_rank_kernel(const int32_t* __restrict__ topk_idx, int64_t T, int K,
                                                           int e0, int E_loc, const int32_t* __restrict__ chunk_base,
                                                           const int32_t* __restrict__ expert_offsets,
                                                           int32_t* __restrict__ row_map,
                                                           int32_t* __restrict__ src_of_row, int64_t max_rows) {
  extern __shared__ uint32_t bits[];  // [E_loc][kChunk / 32]
  constexpr int W = kChunk / 32;
  for (int i = threadIdx.x; i < E_loc * W; i += blockDim.x) bits[i] = 0;
  __syncthreads();
  const int tl = threadIdx.x;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kChunk + tl;
  if (t < T) {
    for (int k = 0; k < K; ++k) {
      const int e = topk_idx[t * K + k] - e0;
      if (e >= 0 && e < E_loc) atomicOr(&bits[e * W + (tl >> 5)], 1u << (tl & 31));
    }
  }
  __syncthreads();
  if (t < T) {
    for (int k = 0; k < K; ++k) {
      const int e = topk_idx[t * K + k] - e0;
      int32_t row = -1;
      if (e >= 0 && e < E_loc) {
        int rank = 0;
        for (int w = 0; w < (tl >> 5); ++w) rank += __popc(bits[e * W + w]);
        rank += __popc(bits[e * W + (tl >> 5)] & ((1u << (tl & 31)) - 1u));
        row = expert_offsets[e] + chunk_base[static_cast<int64_t>(blockIdx.x) * E_loc + e] + rank;
        if (row < max_rows) src_of_row[row] = static_cast<int32_t>(t);
        else row = -1;
      }
      row_map[t * K + k] = row;
    }
  }
}

cudaError_t launch_permute_plan(const int32_t* topk_idx, int64_t num_tokens, int32_t top_k, int32_t expert_begin,
                                int32_t num_local_experts, int32_t align, int32_t* row_map, int32_t* src_of_row,
                                int64_t max_rows, int32_t* expert_offsets, void* ws, cudaStream_t stream) {
  const int64_t chunks = (num_tokens + kChunk - 1) / kChunk;
  int32_t* status = static_cast<int32_t*>(ws);
  int32_t* chunk_counts = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws) + 256);
  int32_t* counts = chunk_counts + chunks * num_local_experts;
  if (chunks > 0) {
    plan_count_kernel<<<static_cast<unsigned>(chunks), kChunk, 4 * num_local_experts, stream>>>(
        topk_idx, num_tokens, top_k, expert_begin, num_local_experts, chunk_counts);
  }
  plan_scan_kernel<<<1, 1024, 0, stream>>>(chunk_counts, chunks, num_local_experts, align, expert_offsets, counts,
                                           src_of_row, max_rows, status);
  if (chunks > 0) {
    const size_t smem = 4 * static_cast<size_t>(num_local_experts) * (kChunk / 32);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(plan_rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    plan_rank_kernel<<<static_cast<unsigned>(chunks), kChunk, smem, stream>>>(
        topk_idx, num_tokens, top_k, expert_begin, num_local_experts, chunk_counts, expert_offsets, row_map,
        src_of_row, max_rows);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// A3 move
// ---------------------------------------------------------------------------------------------
constexpr int kMoveRows = 32;
constexpr int kMoveUnroll = 8;

__global__ void __launch_bounds__(256) permute_pad_kernel(const uint8_t* __restrict__ q_tok,
                                                          const uint8_t* __restrict__ s_tok, int64_t ld_s_tok,
                                                          int64_t H, const int32_t* __restrict__ src_of_row,
                                                          const int32_t* __restrict__ expert_offsets, int E_loc,
                                                          int64_t max_rows, uint8_t* __restrict__ q_out,
                                                          uint8_t* __restrict__ s_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t R = expert_offsets[E_loc];
  const int64_t n_items = (R + kMoveRows - 1) / kMoveRows;
  const int64_t n_vec = H / 16;  // 16-byte chunks per row
  const int n_tiles = static_cast<int>(H / kTile);
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int64_t r0 = item * kMoveRows;
    // --- codes: warp w moves rows r0 + 4w .. r0 + 4w + 3
#pragma unroll 1
    for (int rr = 0; rr < 4; ++rr) {
      const int64_t r = r0 + warp * 4 + rr;
      if (r >= R) break;
      const int32_t src = src_of_row[r];
      const uint4* sp = reinterpret_cast<const uint4*>(q_tok + static_cast<int64_t>(src) * H);
      uint4* dp = reinterpret_cast<uint4*>(q_out + r * H);
      for (int64_t v0 = 0; v0 < n_vec; v0 += 32 * kMoveUnroll) {
        uint4 buf[kMoveUnroll];
#pragma unroll
        for (int u = 0; u < kMoveUnroll; ++u) {
          const int64_t v = v0 + u * 32 + lane;
          buf[u] = make_uint4(0, 0, 0, 0);
          if (src >= 0 && v < n_vec) buf[u] = ld_nc_v4(sp + v);
        }
#pragma unroll
        for (int u = 0; u < kMoveUnroll; ++u) {
          const int64_t v = v0 + u * 32 + lane;
          if (v < n_vec) st_v4(dp + v, buf[u]);
        }
      }
    }
    // --- scales: lane = row within the item, warps stride over the 1x128 tiles
    const int64_t r = r0 + lane;
    const int32_t src = r < R ? src_of_row[r] : -1;
    for (int tl = warp; tl < n_tiles; tl += 8) {
      const uint8_t b = src >= 0 ? s_tok[static_cast<int64_t>(tl) * ld_s_tok + src] : static_cast<uint8_t>(0);
      if (r < R) s_out[static_cast<int64_t>(tl) * max_rows + r] = b;
    }
  }
}

cudaError_t launch_permute_pad(const uint8_t* q_tok, const uint8_t* s_tok, int64_t ld_s_tok, int64_t hidden,
                               const int32_t* src_of_row, const int32_t* expert_offsets, int32_t num_local_experts,
                               int64_t max_rows, uint8_t* q_out, uint8_t* s_out, cudaStream_t stream, int num_sms) {
  int64_t grid = (max_rows + kMoveRows - 1) / kMoveRows;
  const int64_t cap = static_cast<int64_t>(num_sms) * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  permute_pad_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(
      q_tok, s_tok, ld_s_tok, hidden, src_of_row, expert_offsets, num_local_experts, max_rows, q_out, s_out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// A4 unpermute + unpad: one warp per token; each lane owns 8 BF16 (16 B) per step and keeps up to
// K independent 128-bit loads in flight; fp32 fmaf in k order, BF16 RNE.
// ---------------------------------------------------------------------------------------------
constexpr int kMaxTopK = 16;

__global__ void __launch_bounds__(256) unpermute_unpad_kernel(const __nv_bfloat16* __restrict__ x, int64_t H,
                                                              const int32_t* __restrict__ row_map,
                                                              const float* __restrict__ probs, int64_t T, int K,
                                                              __nv_bfloat16* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t wstride = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t t = warp; t < T; t += wstride) {
    const int32_t my_row = lane < K ? row_map[t * K + lane] : -1;
    const float my_p = (lane < K && probs != nullptr) ? probs[t * K + lane] : 1.0f;
    int32_t rowk[kMaxTopK];
    float pk[kMaxTopK];
#pragma unroll
    for (int k = 0; k < kMaxTopK; ++k) {  // k order kept; non-local terms (row < 0) are skipped
      rowk[k] = __shfl_sync(0xffffffffu, my_row, k);
      pk[k] = __shfl_sync(0xffffffffu, my_p, k);
      if (k >= K) rowk[k] = -1;
    }
    for (int64_t h0 = lane * 8; h0 < H; h0 += 256) {
      float acc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.0f;
#pragma unroll
      for (int k = 0; k < kMaxTopK; ++k) {
        if (rowk[k] >= 0) {
          const uint4 v = ld_nc_v4(x + static_cast<int64_t>(rowk[k]) * H + h0);
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
          if (probs != nullptr) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              acc[2 * j] = __fmaf_rn(pk[k], bf16lo_to_f32(w[j]), acc[2 * j]);
              acc[2 * j + 1] = __fmaf_rn(pk[k], bf16hi_to_f32(w[j]), acc[2 * j + 1]);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              acc[2 * j] = __fadd_rn(acc[2 * j], bf16lo_to_f32(w[j]));
              acc[2 * j + 1] = __fadd_rn(acc[2 * j + 1], bf16hi_to_f32(w[j]));
            }
          }
        }
      }
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __nv_bfloat162 b = __floats2bfloat162_rn(acc[2 * j], acc[2 * j + 1]);
        o[j] = *reinterpret_cast<uint32_t*>(&b);
      }
      st_v4(y + t * H + h0, make_uint4(o[0], o[1], o[2], o[3]));
    }
  }
}

cudaError_t launch_unpermute_unpad(const void* x, int64_t hidden, const int32_t* row_map, const float* probs,
                                   int64_t num_tokens, int32_t top_k, void* y, cudaStream_t stream, int num_sms) {
  int64_t grid = (num_tokens + 7) / 8;
  const int64_t cap = static_cast<int64_t>(num_sms) * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  unpermute_unpad_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(x), hidden, row_map, probs, num_tokens, top_k,
      static_cast<__nv_bfloat16*>(y));
  return cudaGetLastError();
}

}  // namespace fp8flow
