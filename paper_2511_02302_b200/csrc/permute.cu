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
// Plan (deterministic, no CUB, no host sync) over 512-token chunks, one thread per token:
//   plan_fused_kernel (one cooperative launch when every chunk CTA fits on the GPU at once, up to
//   ~150k tokens): each CTA builds its chunk's shared-memory histogram over the local experts, a
//   grid sync, then every CTA derives the expert offsets (padded sizes, exclusive scan over experts)
//   and its chunk's per-expert base from the count table; an (expert x token) bit matrix in shared
//   memory gives each token's rank inside its experts as a prefix popcount, so row = offset[e] +
//   base[e] + rank is stable in token order; chunk 0 also writes expert_offsets and the PAD rows.
//   Beyond that size the same two phases run as two kernels (plan_count_kernel, plan_place_kernel).
// Move: fp8flow_permute_pad is the one-rank case of the fused dispatch engine (ep.cu): each token
// read once by a 1D bulk copy and written to all of its local rows by bulk stores.
// Unpermute (A4, below): a bulk-copy engine -- one producer warp streams each token's local rows
// into a shared-memory ring, 7 consumer warps accumulate them in fp32 FMA in k order and store
// BF16 (RNE) with 128-bit stores.
#include <cooperative_groups.h>

#include "async.cuh"
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

// Single-launch plan (cooperative launch, all chunk CTAs co-resident): each CTA builds its chunk's
// (expert x token) bit matrix once, derives its per-expert counts from it by popcount and publishes
// them, then one grid-wide barrier, then the same placement as plan_place without re-reading the
// routing rows.  Used whenever the chunks fit on the GPU at once; otherwise the 2-kernel path.
__global__ void __launch_bounds__(kChunk) plan_fused_kernel(const int32_t* __restrict__ topk_idx, int64_t T, int K,
                                                            int e0, int E_loc, int align, int64_t n_chunks,
                                                            int32_t* __restrict__ chunk_counts,
                                                            int32_t* __restrict__ expert_offsets,
                                                            int32_t* __restrict__ row_map,
                                                            int32_t* __restrict__ src_of_row, int64_t max_rows,
                                                            int32_t* __restrict__ status) {
  extern __shared__ uint32_t smem_plan[];
  uint32_t* bits = smem_plan;                                            // [E_loc][kWords]
  int32_t* pre = reinterpret_cast<int32_t*>(bits + E_loc * kWords);      // [E_loc][kWords]
  int32_t* off = pre + E_loc * kWords;                                   // [E_loc + 1]
  int32_t* base = off + E_loc + 1;                                       // [E_loc]
  __shared__ int32_t warp_tot[kChunk / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t chunk = blockIdx.x;
  const int64_t t = chunk * kChunk + tid;

  for (int i = tid; i < E_loc * kWords; i += kChunk) bits[i] = 0;
  __syncthreads();
  int32_t le[16];  // this token's local expert ids (-1: not local), k order; K <= 16
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    le[k] = -1;
    if (k < K && t < T) {
      const int e = topk_idx[t * K + k] - e0;
      if (e >= 0 && e < E_loc) le[k] = e;
    }
    if (le[k] >= 0) atomicOr(&bits[le[k] * kWords + (tid >> 5)], 1u << lane);
  }
  __syncthreads();
  // prefix popcounts along each expert row; the row total is this chunk's count for the expert
  for (int r0 = warp * 2; r0 < E_loc; r0 += (kChunk / 32) * 2) {
    const int row = r0 + (lane >> 4), wi = lane & 15;
    const bool ok = row < E_loc;
    const int c = ok ? __popc(bits[row * kWords + wi]) : 0;
    int inc = c;
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, inc, d, 16);
      if (wi >= d) inc += n;
    }
    if (ok) {
      pre[row * kWords + wi] = inc - c;
      if (wi == 15) chunk_counts[chunk * E_loc + row] = inc;
    }
  }
  __threadfence();
  cooperative_groups::this_grid().sync();

  // per-expert totals and this chunk's base (2 experts per thread: E_loc <= 1024)
  int cnt[2] = {0, 0}, pad[2] = {0, 0};
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int e = 2 * tid + j;
    if (e < E_loc) {
      int total = 0, mine = 0;
      if (n_chunks <= 32) {  // all count loads in flight at once (one L2 round trip)
        int v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = c < n_chunks ? __ldcg(chunk_counts + c * E_loc + e) : 0;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          mine += (c < chunk) ? v[c] : 0;
          total += v[c];
        }
      } else {
#pragma unroll 8
        for (int64_t c = 0; c < n_chunks; ++c) {
          const int v = __ldcg(chunk_counts + c * E_loc + e);
          mine += (c < chunk) ? v : 0;
          total += v;
        }
      }
      base[e] = mine;
      cnt[j] = total;
      pad[j] = (total + align - 1) / align * align;
    }
  }
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
  if (t < T) {
    const uint32_t below = (1u << lane) - 1u;
    const int w = tid >> 5;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k < K) {
        int32_t row = -1;
        if (le[k] >= 0) {
          const int e = le[k];
          row = off[e] + base[e] + pre[e * kWords + w] + __popc(bits[e * kWords + w] & below);
          if (row < max_rows) src_of_row[row] = static_cast<int32_t>(t);
          else row = -1;
        }
        row_map[t * K + k] = row;
      }
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
  const size_t smem = static_cast<size_t>(num_local_experts) * kWords * 8 + 4 * (2 * num_local_experts + 1);
  // Single cooperative launch when every chunk CTA can be resident at once (up to ~150k tokens on
  // 148 SMs); beyond that, or for shared-memory needs above 64 KB (E_loc > ~450), the two-kernel
  // path (count, then place) -- same results, it re-reads the routing rows once more.
  int dev = 0, coop = 0, sms = 0;
  cudaError_t e0 = cudaGetDevice(&dev);
  if (e0 == cudaSuccess) e0 = cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (e0 == cudaSuccess) e0 = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e0 != cudaSuccess) return e0;
  static KernelSetup fused_setup;  // occupancy at 64 KB of shared memory (conservative)
  const int occ = coop ? prepare_kernel(fused_setup, plan_fused_kernel, kChunk, 64 * 1024, 64 * 1024) : 0;
  if (top_k <= 16 && smem <= 64 * 1024 && grid <= static_cast<int64_t>(occ) * sms) {
    int64_t n_chunks = grid;
    int K = top_k, e0i = expert_begin, E = num_local_experts, al = align;
    int64_t T = num_tokens, mr = max_rows;
    void* args[] = {const_cast<int32_t**>(&topk_idx), &T, &K, &e0i, &E, &al, &n_chunks, &chunk_counts,
                    &expert_offsets, &row_map, &src_of_row, &mr, &status};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(plan_fused_kernel), dim3(static_cast<unsigned>(grid)),
                                       dim3(kChunk), args, smem, stream);
  }
  if (chunks == 0) {
    cudaError_t e = cudaMemsetAsync(chunk_counts, 0, 4 * static_cast<size_t>(num_local_experts), stream);
    if (e != cudaSuccess) return e;
  } else {
    plan_count_kernel<<<static_cast<unsigned>(chunks), kChunk, 4 * num_local_experts, stream>>>(
        topk_idx, num_tokens, top_k, expert_begin, num_local_experts, chunk_counts);
  }
  static KernelSetup place_setup;  // opted in to the largest layout (E_loc = 1024)
  if (prepare_kernel(place_setup, plan_place_kernel, kChunk, 1024 * kWords * 8 + 4 * (2 * 1024 + 1), smem) == 0)
    return cudaErrorInvalidValue;
  plan_place_kernel<<<static_cast<unsigned>(grid), kChunk, smem, stream>>>(
      topk_idx, num_tokens, top_k, expert_begin, num_local_experts, align, chunks > 0 ? chunks : 1, chunk_counts,
      expert_offsets, row_map, src_of_row, max_rows, status);
  return cudaGetLastError();
}

// A3 move: fp8flow_permute_pad runs the one-rank case of the fused dispatch (ep.cu): every routed
// token is read ONCE and fanned out to all of its local expert rows (r01's per-row move read a
// token once per row -- 8x at top-8 with all experts local, 1.27x at EP8).

// ---------------------------------------------------------------------------------------------
// A4 unpermute + unpad on the bulk-copy engine.  One CTA per SM; tokens dealt round-robin.
//   warp 0 (producer): per token, compacts its local rows in k order (ballot + __fns) and streams
//     each row (2H bytes) global -> shared with a 1D bulk copy into a ring of row slots
//     (mbarrier `full[slot]` counts the bytes; `empty[slot]` is released by the consumers).
//   warps 1-7 (consumers, 224 threads): per token, in the same order, wait for each row, accumulate
//     acc = fmaf(p_k, x_k, acc) in fp32 in k order from +0 over their 16-byte chunks, round to BF16
//     (RNE) and store 128-bit.  Tokens without a local expert produce +0.
// Up to nslots rows (e.g. 15 x 14 KB) are in flight per SM without register staging.
// ---------------------------------------------------------------------------------------------
constexpr int kUnpermConsumerWarps = 7;
constexpr int kMaxUnpermSlots = 16;
constexpr int kUnpermChunksPerThread = 4;  // 224 threads x 4 x 8 BF16 = 7168 columns per pass
constexpr size_t kUnpermSmemBudget = 220 * 1024;

__global__ void __launch_bounds__(256, 1) unpermute_unpad_kernel(const __nv_bfloat16* __restrict__ x, int64_t H,
                                                                 const int32_t* __restrict__ row_map,
                                                                 const float* __restrict__ probs, int64_t T, int K,
                                                                 __nv_bfloat16* __restrict__ y, int nslots) {
  extern __shared__ __align__(128) uint8_t smem_unperm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_unperm);
  uint64_t* empty = full + kMaxUnpermSlots;
  uint8_t* slots = smem_unperm + 16 * kMaxUnpermSlots;  // 256 B in
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = gridDim.x;
  const int64_t row_bytes = 2 * H;

  if (tid == 0) {
    for (int i = 0; i < nslots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kUnpermConsumerWarps);
    }
    mbar_init_fence();
  }
  __syncthreads();

  if (warp == 0) {  // ---------------- producer
    int slot = 0;
    uint32_t parity = 0;   // parity of the current ring lap
    bool wrapped = false;  // the ring has been filled once: slots must be released before reuse
    // routing rows are read two tokens ahead so their latency never stalls the copy issue
    int64_t t = blockIdx.x;
    int32_t row_a = (t < T && lane < K) ? row_map[t * K + lane] : -1;
    int32_t row_b = (t + G < T && lane < K) ? row_map[(t + G) * K + lane] : -1;
    for (; t < T; t += G) {
      const int32_t my_row = row_a;
      row_a = row_b;
      row_b = (t + 2 * G < T && lane < K) ? row_map[(t + 2 * G) * K + lane] : -1;
      const uint32_t valid = __ballot_sync(0xffffffffu, my_row >= 0);
      const int nk = __popc(valid);
      const int32_t comp_row = __shfl_sync(0xffffffffu, my_row, static_cast<int>(__fns(valid, 0, lane + 1)) & 31);
      for (int i = 0; i < nk; ++i) {
        const int32_t r = __shfl_sync(0xffffffffu, comp_row, i);
        if (lane == 0) {
          if (wrapped) mbar_wait(&empty[slot], parity ^ 1u);  // released after the previous lap
          mbar_expect_tx(&full[slot], static_cast<uint32_t>(row_bytes));
          bulk_load_1d(slots + slot * row_bytes, x + static_cast<int64_t>(r) * H, static_cast<uint32_t>(row_bytes),
                       &full[slot]);
        }
        if (++slot == nslots) {
          slot = 0;
          parity ^= 1u;
          wrapped = true;
        }
      }
    }
  } else {  // ---------------- consumers
    const int ct = tid - 32;
    const int64_t n_chunks = H / 8;
    int slot0 = 0;           // ring slot of the token's first row
    uint32_t parity0 = 0;    // its lap parity
    int64_t t = blockIdx.x;
    // software-pipelined routing reads: the next token's row_map / probs are loaded one token ahead
    int32_t nxt_row = (t < T && lane < K) ? row_map[t * K + lane] : -1;
    float nxt_p = (t < T && lane < K) ? (probs != nullptr ? probs[t * K + lane] : 1.0f) : 0.0f;
    for (; t < T; t += G) {
      const int32_t my_row = nxt_row;
      const float my_p = nxt_p;
      const int64_t tn = t + G;
      nxt_row = (tn < T && lane < K) ? row_map[tn * K + lane] : -1;
      nxt_p = (tn < T && lane < K) ? (probs != nullptr ? probs[tn * K + lane] : 1.0f) : 0.0f;
      const uint32_t valid = __ballot_sync(0xffffffffu, my_row >= 0);
      const int nk = __popc(valid);
      const float comp_p = __shfl_sync(0xffffffffu, my_p, static_cast<int>(__fns(valid, 0, lane + 1)) & 31);
      for (int64_t c0 = 0; c0 < n_chunks; c0 += 224 * kUnpermChunksPerThread) {
        float acc[kUnpermChunksPerThread][8];
#pragma unroll
        for (int q = 0; q < kUnpermChunksPerThread; ++q)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[q][j] = 0.0f;
        int slot = slot0;
        uint32_t parity = parity0;
        for (int i = 0; i < nk; ++i) {
          const float pk = __shfl_sync(0xffffffffu, comp_p, i);
          mbar_wait(&full[slot], parity);
          const uint8_t* base = slots + slot * row_bytes;
#pragma unroll
          for (int q = 0; q < kUnpermChunksPerThread; ++q) {
            const int64_t c = c0 + ct + 224 * q;
            if (c < n_chunks) {
              const uint4 v = *reinterpret_cast<const uint4*>(base + c * 16);
              const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                acc[q][2 * j] = __fmaf_rn(pk, bf16lo_to_f32(w[j]), acc[q][2 * j]);
                acc[q][2 * j + 1] = __fmaf_rn(pk, bf16hi_to_f32(w[j]), acc[q][2 * j + 1]);
              }
            }
          }
          // the last pass over the columns releases the slot
          if (c0 + 224 * kUnpermChunksPerThread >= n_chunks) {
            // the warp's generic-proxy reads of the slot are ordered before the producer's next
            // async-proxy (bulk copy) write into it
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
          }
          if (++slot == nslots) {
            slot = 0;
            parity ^= 1u;
          }
        }
#pragma unroll
        for (int q = 0; q < kUnpermChunksPerThread; ++q) {
          const int64_t c = c0 + ct + 224 * q;
          if (c < n_chunks) {
            uint32_t o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              __nv_bfloat162 bb = __floats2bfloat162_rn(acc[q][2 * j], acc[q][2 * j + 1]);
              o[j] = *reinterpret_cast<uint32_t*>(&bb);
            }
            st_v4(y + t * H + c * 8, make_uint4(o[0], o[1], o[2], o[3]));
          }
        }
      }
      for (int i = 0; i < nk; ++i) {  // advance the token's first slot past its rows
        if (++slot0 == nslots) {
          slot0 = 0;
          parity0 ^= 1u;
        }
      }
    }
  }
}

cudaError_t launch_unpermute_unpad(const void* x, int64_t hidden, const int32_t* row_map, const float* probs,
                                   int64_t num_tokens, int32_t top_k, void* y, cudaStream_t stream, int num_sms) {
  const int64_t row_bytes = 2 * hidden;
  const int ctas = 2;  // co-resident CTAs per SM, sharing the shared-memory budget (r01_tune_ctas.txt)
  int nslots = static_cast<int>(kUnpermSmemBudget / ctas / row_bytes);
  if (nslots > kMaxUnpermSlots) nslots = kMaxUnpermSlots;
  // a token's rows must all fit the ring when the columns take more than one consumer pass
  const bool multi_pass = hidden / 8 > 224 * kUnpermChunksPerThread;
  if (nslots < 2 || (multi_pass && nslots < top_k)) return cudaErrorInvalidValue;
  const size_t smem = 16 * kMaxUnpermSlots + static_cast<size_t>(row_bytes) * nslots;
  static KernelSetup setup;
  if (prepare_kernel(setup, unpermute_unpad_kernel, 256, 16 * kMaxUnpermSlots + kUnpermSmemBudget, smem) == 0)
    return cudaErrorInvalidValue;
  const int64_t max_grid = static_cast<int64_t>(num_sms) * ctas;
  int64_t grid = num_tokens < max_grid ? num_tokens : max_grid;
  if (grid < 1) grid = 1;
  unpermute_unpad_kernel<<<static_cast<unsigned>(grid), 256, smem, stream>>>(
      static_cast<const __nv_bfloat16*>(x), hidden, row_map, probs, num_tokens, top_k,
      static_cast<__nv_bfloat16*>(y), nslots);
  return cudaGetLastError();
}

}  // namespace fp8flow
