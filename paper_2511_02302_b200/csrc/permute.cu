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
// Plan (deterministic, no CUB, no host sync), two kernels over 512-token chunks:
//   K1 plan_count : per chunk, a shared-memory histogram over the local experts
//   K2 plan_place : per chunk, the expert offsets (padded sizes, exclusive scan over experts) and
//                   the chunk's per-expert base are derived from the small count table; an
//                   (expert x token) bit matrix in shared memory gives each token's rank inside
//                   its experts as a prefix popcount, so row = offset[e] + base[e] + rank is
//                   stable in token order.  Chunk 0 also writes expert_offsets and the PAD rows.
// Move: warp item = 4 consecutive output rows (balanced contiguous item ranges per warp, one wave
// of CTAs); the 4 rows stream with 128-bit loads and stores (16 in flight per lane), their scale
// bytes are gathered per 1x128 tile (all gathers issued before the stores).
#include "common.cuh"
#include "kernels.h"

namespace fp8flow {

constexpr int kChunk = 512;         // tokens per plan chunk = threads per CTA (one thread per token)
constexpr int kWords = kChunk / 32;  // 32-bit words per expert row of the (expert x token) bit matrix

size_t permute_workspace_bytes(int64_t num_tokens, int32_t num_local_experts) {
  const int64_t chunks = (num_tokens + kChunk - 1) / kChunk;
  return 256 + 4 * static_cast<size_t>(chunks > 0 ? chunks : 1) * num_local_experts;
}

// K1: per-chunk expert histogram (shared-memory atomics; counts are order-independent)
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

// K2: every chunk CTA derives the expert offsets and its own per-expert base from the count table
// (tiny, L2 resident), then ranks its tokens inside each expert through a bit matrix:
//   rank(t, e) = #tokens t' < t of this chunk routed to e = prefix popcount of row e up to bit t.
__global__ void __launch_bounds__(kChunk) plan_place_kernel(const int32_t* __restrict__ topk_idx, int64_t T, int K,
                                                            int e0, int E_loc, int align, int64_t n_chunks,
                                                            const int32_t* __restrict__ chunk_counts,
                                                            int32_t* __restrict__ expert_offsets,
                                                            int32_t* __restrict__ row_map,
                                                            int32_t* __restrict__ src_of_row, int64_t max_rows,
                                                            int32_t* __restrict__ status) {
  extern __shared__ uint32_t smem[];
  uint32_t* bits = smem;                                   // [E_loc][kWords]
  int32_t* pre = reinterpret_cast<int32_t*>(bits + E_loc * kWords);  // [E_loc][kWords] exclusive popc
  int32_t* off = pre + E_loc * kWords;                     // [E_loc + 1]
  int32_t* base = off + E_loc + 1;                         // [E_loc]
  __shared__ int32_t warp_tot[kChunk / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t chunk = blockIdx.x;

  for (int i = tid; i < E_loc * kWords; i += kChunk) bits[i] = 0;
  // per-expert totals and this chunk's base (2 experts per thread: E_loc <= 1024)
  int cnt[2] = {0, 0}, pad[2] = {0, 0};
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int e = 2 * tid + j;
    if (e < E_loc) {
      int total = 0, mine = 0;
#pragma unroll 8
      for (int64_t c = 0; c < n_chunks; ++c) {  // independent L2 loads, kept in flight
        const int v = chunk_counts[c * E_loc + e];
        mine += (c < chunk) ? v : 0;
        total += v;
      }
      base[e] = mine;
      cnt[j] = total;
      pad[j] = (total + align - 1) / align * align;
    }
  }
  // block exclusive scan of the padded sizes in expert order
  const int tsum = pad[0] + pad[1];
  int incl = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += n;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  int wbase = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kChunk / 32; ++w) {
    wbase += (w < warp) ? warp_tot[w] : 0;
    all += warp_tot[w];
  }
  int run = wbase + incl - tsum;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int e = 2 * tid + j;
    if (e < E_loc) {
      off[e] = run;
      if (chunk == 0) {
        expert_offsets[e] = run;
        for (int r = run + cnt[j]; r < run + pad[j]; ++r)
          if (r < max_rows) src_of_row[r] = -1;  // PAD rows (R16: after the real rows)
      }
      run += pad[j];
    }
  }
  if (tid == 0) {
    off[E_loc] = all;
    if (chunk == 0) {
      expert_offsets[E_loc] = all;
      *status = all > max_rows ? 1 : 0;
    }
  }
  __syncthreads();
  // bit matrix of this chunk
  const int64_t t = chunk * kChunk + tid;
  if (t < T) {
    for (int k = 0; k < K; ++k) {
      const int e = topk_idx[t * K + k] - e0;
      if (e >= 0 && e < E_loc) atomicOr(&bits[e * kWords + (tid >> 5)], 1u << lane);
    }
  }
  __syncthreads();
  // exclusive popcount prefix along each expert row (kWords = 16 lanes per row, 2 rows per warp)
  for (int r0 = warp * 2; r0 < E_loc; r0 += (kChunk / 32) * 2) {  // warp-uniform trip count
    const int row = r0 + (lane >> 4), wi = lane & 15;
    const bool ok = row < E_loc;
    const int c = ok ? __popc(bits[row * kWords + wi]) : 0;
    int inc = c;
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, inc, d, 16);
      if (wi >= d) inc += n;
    }
    if (ok) pre[row * kWords + wi] = inc - c;
  }
  __syncthreads();
  if (t < T) {
    const uint32_t below = (1u << lane) - 1u;
    for (int k = 0; k < K; ++k) {
      const int e = topk_idx[t * K + k] - e0;
      int32_t row = -1;
      if (e >= 0 && e < E_loc) {
        const int w = tid >> 5;
        const int rank = pre[e * kWords + w] + __popc(bits[e * kWords + w] & below);
        row = off[e] + base[e] + rank;
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
  const int64_t grid = chunks > 0 ? chunks : 1;  // one CTA even without tokens: writes offsets
  int32_t* status = static_cast<int32_t*>(ws);
  int32_t* chunk_counts = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws) + 256);
  if (chunks == 0) {
    cudaError_t e = cudaMemsetAsync(chunk_counts, 0, 4 * static_cast<size_t>(num_local_experts), stream);
    if (e != cudaSuccess) return e;
  } else {
    plan_count_kernel<<<static_cast<unsigned>(chunks), kChunk, 4 * num_local_experts, stream>>>(
        topk_idx, num_tokens, top_k, expert_begin, num_local_experts, chunk_counts);
  }
  const size_t smem = static_cast<size_t>(num_local_experts) * kWords * 8 + 4 * (2 * num_local_experts + 1);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(plan_place_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  plan_place_kernel<<<static_cast<unsigned>(grid), kChunk, smem, stream>>>(
      topk_idx, num_tokens, top_k, expert_begin, num_local_experts, align, chunks > 0 ? chunks : 1, chunk_counts,
      expert_offsets, row_map, src_of_row, max_rows, status);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// A3 move
// ---------------------------------------------------------------------------------------------
constexpr int kMoveRows = 4;    // output rows per warp item
constexpr int kMoveBatch = 16;  // 16-byte loads in flight per lane

__global__ void __launch_bounds__(256) permute_pad_kernel(const uint8_t* __restrict__ q_tok,
                                                          const uint8_t* __restrict__ s_tok, int64_t ld_s_tok,
                                                          int64_t H, const int32_t* __restrict__ src_of_row,
                                                          const int32_t* __restrict__ expert_offsets, int E_loc,
                                                          int64_t max_rows, uint8_t* __restrict__ q_out,
                                                          uint8_t* __restrict__ s_out, int sched) {
  const int lane = threadIdx.x & 31;
  const int64_t R = expert_offsets[E_loc];
  const int n_vec = static_cast<int>(H / 16);  // 16-byte chunks per row
  const int n_tiles = static_cast<int>(H / kTile);
  for (ItemIter it = warp_item_iter((R + kMoveRows - 1) / kMoveRows, sched); it.cur < it.end; it.cur += it.step) {
    const int64_t item = it.cur;
    const int64_t r0 = item * kMoveRows;
    int32_t src[kMoveRows];
#pragma unroll
    for (int rr = 0; rr < kMoveRows; ++rr) src[rr] = (r0 + rr < R) ? __ldg(src_of_row + r0 + rr) : -2;
    // --- codes: the 4 rows flattened into 4 * n_vec 16-byte chunks, 16 loads in flight per lane
    const int total = kMoveRows * n_vec;
    for (int v0 = 0; v0 < total; v0 += 32 * kMoveBatch) {
      uint4 buf[kMoveBatch];
#pragma unroll
      for (int u = 0; u < kMoveBatch; ++u) {
        const int v = v0 + u * 32 + lane;
        const int rr = v / n_vec, cv = v - rr * n_vec;
        int32_t sr = -2;
#pragma unroll
        for (int q = 0; q < kMoveRows; ++q)
          if (q == rr) sr = src[q];
        buf[u] = make_uint4(0, 0, 0, 0);
        if (v < total && sr >= 0) buf[u] = ld_nc_v4(q_tok + static_cast<int64_t>(sr) * H + 16 * cv);
      }
#pragma unroll
      for (int u = 0; u < kMoveBatch; ++u) {
        const int v = v0 + u * 32 + lane;
        const int rr = v / n_vec, cv = v - rr * n_vec;
        if (v < total && r0 + rr < R) st_v4(q_out + (r0 + rr) * H + 16 * cv, buf[u]);
      }
    }
    // --- scales: (row, tile) pairs of the item spread over the lanes; gathers issued first
    constexpr int kMaxPairsPerLane = kMoveRows * 128 / 32;  // hidden <= 16384
    uint8_t b[kMaxPairsPerLane];
#pragma unroll
    for (int i = 0; i < kMaxPairsPerLane; ++i) {
      const int p = lane + 32 * i, rr = p & (kMoveRows - 1), tl = p / kMoveRows;
      int32_t sr = -2;
#pragma unroll
      for (int q = 0; q < kMoveRows; ++q)
        if (q == rr) sr = src[q];
      b[i] = (tl < n_tiles && sr >= 0) ? __ldg(s_tok + static_cast<int64_t>(tl) * ld_s_tok + sr) : static_cast<uint8_t>(0);
    }
#pragma unroll
    for (int i = 0; i < kMaxPairsPerLane; ++i) {
      const int p = lane + 32 * i, rr = p & (kMoveRows - 1), tl = p / kMoveRows;
      if (tl < n_tiles && r0 + rr < R) s_out[static_cast<int64_t>(tl) * max_rows + r0 + rr] = b[i];
    }
  }
}

cudaError_t launch_permute_pad(const uint8_t* q_tok, const uint8_t* s_tok, int64_t ld_s_tok, int64_t hidden,
                               const int32_t* src_of_row, const int32_t* expert_offsets, int32_t num_local_experts,
                               int64_t max_rows, uint8_t* q_out, uint8_t* s_out, cudaStream_t stream, int num_sms) {
  static const int occ = occupancy_of(permute_pad_kernel, 256, 0);
  const int sched = sched_for("A3", kSchedOnePerWarp);
  // the actual row count lives on the device: size the grid for max_rows (idle warps exit)
  const int64_t grid = sched_grid(sched, (max_rows + kMoveRows - 1) / kMoveRows, 8, occ, num_sms);
  permute_pad_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(
      q_tok, s_tok, ld_s_tok, hidden, src_of_row, expert_offsets, num_local_experts, max_rows, q_out, s_out, sched);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// A4 unpermute + unpad: warp item = (token, 1024-column chunk), balanced contiguous item ranges
// per warp over one wave of CTAs.  The token's local rows are compacted in k order across lanes
// (ballot + __fns, once per token); each lane owns 8 BF16 (16 B) per 256-column step and issues
// all loads of a row group before the fused multiply-adds, so several 128-bit loads per lane are
// in flight (4 steps x <= 2 rows on the common path, 2 steps x 4 rows otherwise).
// fp32 acc = fmaf(p_k, x_k, acc) in k order from +0 (p = 1 when probs is NULL: fmaf(1, x, acc) ==
// acc + x exactly), then BF16 RNE.
// ---------------------------------------------------------------------------------------------
template <int NROWS, int U>
__device__ __forceinline__ void unpermute_chunk(const __nv_bfloat16* __restrict__ x, int64_t H, int64_t h0, int nk,
                                                int32_t comp_row, float comp_p, float (&acc)[U][8]) {
  // local rows [0, nk) in k order, held one per lane (comp_row / comp_p of lane i = i-th term);
  // groups of NROWS rows: all loads of a group are issued before its FMAs
#pragma unroll 1
  for (int g = 0; g < nk; g += NROWS) {
    uint4 v[NROWS][U];
    float p[NROWS];
#pragma unroll
    for (int j = 0; j < NROWS; ++j) {
      const int32_t r = __shfl_sync(0xffffffffu, comp_row, (g + j) & 31);
      p[j] = __shfl_sync(0xffffffffu, comp_p, (g + j) & 31);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t h = h0 + u * 256;
        v[j][u] = (g + j < nk && h < H) ? ld_nc_v4(x + static_cast<int64_t>(r) * H + h) : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int j = 0; j < NROWS; ++j) {
      if (g + j < nk) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t w[4] = {v[j][u].x, v[j][u].y, v[j][u].z, v[j][u].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            acc[u][2 * i] = __fmaf_rn(p[j], bf16lo_to_f32(w[i]), acc[u][2 * i]);
            acc[u][2 * i + 1] = __fmaf_rn(p[j], bf16hi_to_f32(w[i]), acc[u][2 * i + 1]);
          }
        }
      }
    }
  }
}

template <int U>
__device__ __forceinline__ void unpermute_store(__nv_bfloat16* __restrict__ yrow, int64_t H, int64_t h0,
                                                const float (&acc)[U][8]) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t h = h0 + u * 256;
    if (h < H) {
      uint32_t o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 b = __floats2bfloat162_rn(acc[u][2 * i], acc[u][2 * i + 1]);
        o[i] = *reinterpret_cast<uint32_t*>(&b);
      }
      st_v4(yrow + h, make_uint4(o[0], o[1], o[2], o[3]));
    }
  }
}

constexpr int kUnpermChunk = 1024;  // BF16 columns per warp item (32 lanes x 8 x 4)

__global__ void __launch_bounds__(256, 2) unpermute_unpad_kernel(const __nv_bfloat16* __restrict__ x, int64_t H,
                                                              const int32_t* __restrict__ row_map,
                                                              const float* __restrict__ probs, int64_t T, int K,
                                                              __nv_bfloat16* __restrict__ y, int sched) {
  const int lane = threadIdx.x & 31;
  const int64_t n_chunks = (H + kUnpermChunk - 1) / kUnpermChunk;
  int64_t cur_t = -1;
  int nk = 0;
  int32_t comp_row = -1;
  float comp_p = 0.0f;
  for (ItemIter it = warp_item_iter(T * n_chunks, sched); it.cur < it.end; it.cur += it.step) {
    const int64_t item = it.cur;  // item = (token, 1024-column chunk)
    const int64_t t = item / n_chunks;
    const int64_t h0 = (item - t * n_chunks) * kUnpermChunk + lane * 8;
    if (t != cur_t) {  // consecutive items share the token: compact its local terms once
      cur_t = t;
      const int32_t my_row = lane < K ? row_map[t * K + lane] : -1;
      const float my_p = lane < K ? (probs != nullptr ? probs[t * K + lane] : 1.0f) : 0.0f;
      const uint32_t valid = __ballot_sync(0xffffffffu, my_row >= 0);
      nk = __popc(valid);
      const int src = static_cast<int>(__fns(valid, 0, lane + 1)) & 31;  // lane i <- i-th term (k order)
      comp_row = __shfl_sync(0xffffffffu, my_row, src);
      comp_p = __shfl_sync(0xffffffffu, my_p, src);
    }
    __nv_bfloat16* yrow = y + t * H;
    if (nk <= 2) {
      float acc[4][8];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[u][i] = 0.0f;
      unpermute_chunk<2, 4>(x, H, h0, nk, comp_row, comp_p, acc);
      unpermute_store<4>(yrow, H, h0, acc);
    } else {
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        float acc[2][8];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[u][i] = 0.0f;
        unpermute_chunk<4, 2>(x, H, h0 + hh * 512, nk, comp_row, comp_p, acc);
        unpermute_store<2>(yrow, H, h0 + hh * 512, acc);
      }
    }
  }
}

cudaError_t launch_unpermute_unpad(const void* x, int64_t hidden, const int32_t* row_map, const float* probs,
                                   int64_t num_tokens, int32_t top_k, void* y, cudaStream_t stream, int num_sms) {
  static const int occ = occupancy_of(unpermute_unpad_kernel, 256, 0);
  const int64_t items = num_tokens * ((hidden + kUnpermChunk - 1) / kUnpermChunk);
  const int sched = sched_for("A4", kSchedInterleaved);
  const int64_t grid = sched_grid(sched, items, 8, occ, num_sms);
  unpermute_unpad_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(x), hidden, row_map, probs, num_tokens, top_k,
      static_cast<__nv_bfloat16*>(y), sched);
  return cudaGetLastError();
}

}  // namespace fp8flow
