// ep.cu -- NEXT-3: expert-parallel FP8 dispatch fused with A3's permute + pad on the receive side,
// and the BF16 combine fused with A4's unpermute, over peer memory (NVLink 5 / NVSwitch: CUDA IPC
// mappings of the other ranks' buffers; plain local pointers when several ranks share a device).
//
// Paper: P:245 (routing -> dispatch -> permutation -> experts -> unpermutation -> combination);
// P:128 (dispatch ships the row-wise FP8 format); P:347 ("the need to transmit both the FP8 tensor
// and its corresponding scaling factors doubles the number of data buffers and synchronizations");
// P:260 (BF16 at the combine boundary).  Reading R34: rank g's dispatched rows are
// A3 over all ranks' tokens gathered in rank order, restricted to g's experts; combine is A4 over the
// concatenated expert outputs (fp32 FMA in k order, BF16 RNE).
//
// B200 design (NEXT-3):
//  * PULL, not push: the receiver reads each routed token ONCE from its owner over NVLink and fans
//    it out to all of its local expert rows in HBM, so NVLink carries unique (token, rank) bytes
//    (~2x fewer than one message per (token, expert) pair at DSv3 routing) and no intermediate
//    receive buffer is written and re-read (the permute is fused into the receive).
//  * codes and scales in one kernel, one synchronisation (the barrier before it), no staging
//    buffer pair as in P:347.
//  * peer pointers travel by value in the kernel parameters (<= 64 ranks), so every launch is
//    CUDA-graph capturable; the barrier keeps its epoch on the device.
//  * the dispatch pulls whole tokens with 1D bulk copies (cp.async.bulk global -> shared, peer VA
//    through UVA) and writes rows with bulk stores; the combine and the LSU dispatch variant use
//    plain 128-bit non-coherent loads.
#include "async.cuh"
#include "common.cuh"
#include "kernels.h"

namespace fp8flow {

constexpr int kEpThreads = 256;
constexpr int kEpWarps = kEpThreads / 32;
constexpr int kCopyU = 16;  // uint4 per lane per pass of the token copy (8 KB per warp pass)
constexpr int kScaleChunk = 16;  // scale bytes per token with loads in flight together (LSU dispatch)

struct PeerPtrs {
  const void* p[kMaxRanks];
};
struct PeerPtrs2 {
  const void* a[kMaxRanks];
  const void* b[kMaxRanks];
};

// ---------------------------------------------------------------------------------------------
// all-gather by pulls: out[r * bytes + i] = peer[r][i]
// ---------------------------------------------------------------------------------------------
template <typename V>
__global__ void __launch_bounds__(kEpThreads) peer_gather_kernel(PeerPtrs src, int n, int64_t vec_per_rank,
                                                                 V* __restrict__ out,
                                                                 const int32_t* __restrict__ gate) {
  if (gate != nullptr && *gate != 0) return;  // the barrier before it timed out: peers not ready
  const int64_t total = vec_per_rank * n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / vec_per_rank);
    const int64_t j = i - r * vec_per_rank;
    if constexpr (sizeof(V) == 16) {
      out[i] = ld_nc_v4(static_cast<const uint4*>(src.p[r]) + j);
    } else {
      out[i] = __ldg(static_cast<const V*>(src.p[r]) + j);
    }
  }
}

cudaError_t launch_peer_gather(const void* const* peer_src, int32_t n, int64_t bytes_per_rank, void* dst,
                               const int32_t* gate, cudaStream_t stream, int num_sms) {
  PeerPtrs pp{};
  for (int r = 0; r < n; ++r) pp.p[r] = peer_src[r];
  const bool v16 = bytes_per_rank % 16 == 0;  // else 4-byte words (the ABI requires bytes % 4 == 0)
  const int64_t vec = bytes_per_rank / (v16 ? 16 : 4);
  int64_t grid = (vec * n + kEpThreads - 1) / kEpThreads;
  if (grid > 4LL * num_sms) grid = 4LL * num_sms;
  if (grid < 1) grid = 1;
  if (v16)
    peer_gather_kernel<uint4><<<static_cast<unsigned>(grid), kEpThreads, 0, stream>>>(pp, n, vec, static_cast<uint4*>(dst),
                                                                                     gate);
  else
    peer_gather_kernel<uint32_t><<<static_cast<unsigned>(grid), kEpThreads, 0, stream>>>(pp, n, vec,
                                                                                        static_cast<uint32_t*>(dst), gate);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// device barrier over peer flags.  Rank r's signal buffer holds n + 1 uint32: slot s = the last
// epoch rank s announced to r, slot n = r's own epoch counter (advanced only by r).  Every call
// advances the epoch, stores it (release, system scope) into slot r of every peer, then waits
// (acquire) until every slot of its own buffer has reached it.  Bounded: after ~timeout_ms the
// kernel gives up and writes 1 to *status (0 on success).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kMaxRanks) peer_barrier_kernel(PeerPtrs sig, int rank, int n, int32_t* status,
                                                                 uint64_t timeout_ns) {
  __shared__ uint32_t epoch_s;
  __shared__ int failed;
  uint32_t* mine = static_cast<uint32_t*>(const_cast<void*>(sig.p[rank]));
  if (threadIdx.x == 0) {
    epoch_s = mine[n] + 1;
    mine[n] = epoch_s;
    failed = 0;
  }
  __syncthreads();
  const uint32_t epoch = epoch_s;
  const int d = threadIdx.x;
  if (d < n) {
    __threadfence_system();  // everything this stream wrote before the barrier, visible system-wide
    st_release_sys(static_cast<uint32_t*>(const_cast<void*>(sig.p[d])) + rank, epoch);
    const uint64_t t0 = globaltimer_ns();
    while (static_cast<int32_t>(ld_acquire_sys(mine + d) - epoch) < 0) {
      if (globaltimer_ns() - t0 > timeout_ns) {
        failed = 1;
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && status != nullptr) *status = failed;
}

cudaError_t launch_peer_barrier(void* const* peer_signal, int32_t rank, int32_t n, int32_t* status,
                                uint32_t timeout_ms, cudaStream_t stream) {
  PeerPtrs pp{};
  for (int r = 0; r < n; ++r) pp.p[r] = peer_signal[r];
  peer_barrier_kernel<<<1, kMaxRanks, 0, stream>>>(pp, rank, n, status,
                                                   static_cast<uint64_t>(timeout_ms) * 1000000ull);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// dispatch + permute + pad (receive side), register-copy kernel (the path across GPUs).  Three
// kinds of work in one launch, each spread over the whole grid:
//   codes : per global token with >= 1 local row: the warp pulls its H code bytes once (128-bit
//           non-coherent loads, up to 8 KB in flight per warp) and stores them to every local row;
//   scales: per batch of 32 consecutive tokens, one 32-byte sector per tile from the owner for
//           the whole batch (the link-efficient gather), scattered to each token's local rows;
//   PAD   : per 32 output rows, the PAD rows' codes and scale bytes 0x00.
// (Measured on the way: PAD rows handled per expert by 32 warps, or scales per 32-token chunk
// before the codes, each cost ~15 us of serial latency at DSv3 sizes.)
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kEpThreads) dispatch_permute_lsu_kernel(
    PeerPtrs2 peer, int64_t ld_s_tok, int64_t Tpr, int n, int64_t H, const int32_t* __restrict__ row_map, int K,
    const int32_t* __restrict__ src_of_row, const int32_t* __restrict__ offsets, int E_loc, int64_t max_rows,
    uint8_t* __restrict__ q_out, uint8_t* __restrict__ s_out, const int32_t* __restrict__ gate) {
  if (gate != nullptr && *gate != 0) return;  // the barrier before it timed out: peers not ready
  const int lane = threadIdx.x & 31;
  const int64_t W = static_cast<int64_t>(gridDim.x) * kEpWarps;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kEpWarps + (threadIdx.x >> 5);
  const int64_t T = Tpr * n;
  const int64_t n_tiles = H / 128;
  const int64_t R = min64(offsets[E_loc], max_rows);  // an overflowed plan: only max_rows rows exist

  // warp roles: the first S warps gather the scale bytes (by 32-token batches, below), the other
  // Wc warps copy the codes -- so the scale batches' few serial link round trips overlap the
  // code copies instead of adding to them
  const int64_t n_batches = (T + 31) / 32;
  const int64_t S = W >= 8 ? min64(n_batches, W / 4) : 0;
  const int64_t Wc = W - S;
  const int64_t gc = gw - S;  // code-warp index (< 0: a scale warp)

  // ---- codes: code warp gc owns tokens gc, gc+Wc, ...; their row_map rows are read 32 tokens at a
  // time (lane l: token gc + (i0+l)Wc), a ballot marks the routed ones; per routed token the warp
  // pulls its H code bytes once (16-byte non-coherent loads, up to 8 KB in flight per warp) and
  // stores them to every local row.
  const int64_t nvec = H / 16;
  for (int64_t i0 = 0; gc >= 0 && gc + i0 * Wc < T; i0 += 32) {
    const int64_t my_gt = gc + (i0 + lane) * Wc;
    int32_t rows[16];
    bool any = false;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      rows[k] = (my_gt < T && k < K) ? __ldg(row_map + my_gt * K + k) : -1;
      any |= rows[k] >= 0;
    }
    for (uint32_t mask = __ballot_sync(0xffffffffu, any); mask != 0; mask &= mask - 1) {
      const int j = __ffs(mask) - 1;
      const int64_t gt = gc + (i0 + j) * Wc;
      const int src_rank = static_cast<int>(gt / Tpr);
      const uint4* src = reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(peer.a[src_rank]) +
                                                        (gt - src_rank * Tpr) * H);
      for (int64_t v0 = 0; v0 < nvec; v0 += 32 * kCopyU) {
        uint4 buf[kCopyU];
#pragma unroll
        for (int u = 0; u < kCopyU; ++u) {
          const int64_t v = v0 + lane + 32 * u;
          if (v < nvec) buf[u] = ld_nc_v4(src + v);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int32_t r = __shfl_sync(0xffffffffu, rows[k], j);
          if (r >= 0) {
            uint4* dst = reinterpret_cast<uint4*>(q_out + static_cast<int64_t>(r) * H);
#pragma unroll
            for (int u = 0; u < kCopyU; ++u) {
              const int64_t v = v0 + lane + 32 * u;
              if (v < nvec) st_v4(dst + v, buf[u]);
            }
          }
        }
      }
    }
  }

  // ---- scales, by batches of 32 consecutive global tokens (scale warp gw: batches gw, gw+S, ...; all
  // warps when the grid is tiny): lane l
  // owns token 32c+l, so for every 1x128 tile the warp's 32 scale-byte reads from the owner fall in
  // ONE 32-byte sector -- 56 link transactions per 32 tokens, where a row-by-row gather costs one
  // per (row, tile) (~30x more transactions over NVLink for DSv3 routing); each lane then writes
  // its token's bytes to the token's local rows (local HBM).  kScaleChunk loads in flight per lane.
  const int64_t scale_stride = S > 0 ? S : W;
  for (int64_t c = gw; (S == 0 || gw < S) && c * 32 < T; c += scale_stride) {
    const int64_t gt = c * 32 + lane;
    int32_t rows[16];
    bool any = false;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      rows[k] = (gt < T && k < K) ? __ldg(row_map + gt * K + k) : -1;
      any |= rows[k] >= 0;
    }
    if (!__any_sync(0xffffffffu, any)) continue;
    const int src_rank = any ? static_cast<int>(gt / Tpr) : 0;
    const uint8_t* sp = static_cast<const uint8_t*>(peer.b[src_rank]) + (any ? gt - src_rank * Tpr : 0);
    for (int64_t j0 = 0; j0 < n_tiles; j0 += kScaleChunk) {
      uint32_t v[kScaleChunk];
#pragma unroll
      for (int j = 0; j < kScaleChunk; ++j) v[j] = (any && j0 + j < n_tiles) ? __ldg(sp + (j0 + j) * ld_s_tok) : 0u;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (rows[k] >= 0) {
#pragma unroll
          for (int j = 0; j < kScaleChunk; ++j)
            if (j0 + j < n_tiles) s_out[(j0 + j) * max_rows + rows[k]] = static_cast<uint8_t>(v[j]);
        }
      }
    }
  }

  // ---- PAD rows (codes 0x00, scale bytes 0x00): 32-row chunks from the last warp down
  for (int64_t c = W - 1 - gw; c * 32 < R; c += W) {
    const int64_t r0 = c * 32;
    const bool pad = r0 + lane < R && src_of_row[r0 + lane] < 0;
    for (uint32_t m = __ballot_sync(0xffffffffu, pad); m != 0; m &= m - 1) {
      const int64_t r = r0 + __ffs(m) - 1;
      for (int64_t i = lane * 16; i < H; i += 32 * 16) st_v4(q_out + r * H + i, make_uint4(0, 0, 0, 0));
      for (int64_t j = lane; j < n_tiles; j += 32) s_out[j * max_rows + r] = 0;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// dispatch + permute + pad on the bulk-copy engine (same-device peers).  Four CTAs per SM (one producer
// thread each: 1 CTA/SM 54 us, 2: 34.7, 3: 33.6, 4: 32.8 at DSv3 sizes; store slack 2/4/8 made no
// difference -- the single issuing thread per CTA is what bounds it); CTA c owns global
// tokens c, c+G, c+2G, ...
//   1. all warps compact the CTA's routed tokens (row_map read 32 tokens at a time, ballot, one
//      shared atomic per batch) into a shared list {token, its top_k rows};
//   2. warp 0 / lane 0 streams the list through a ring of token slots: a 1D bulk copy pulls a
//      token's H code bytes from its owner into a slot (mbarrier-completed, `lead` tokens ahead),
//      then one 1D bulk store per local row writes it out (one bulk group per token; a slot is
//      refilled once its stores have read it) -- up to ~25 tokens (180 KB) in flight per SM with
//      no register staging and no per-16-byte LSU instructions;
//   3. warps 1-7 meanwhile gather the scale bytes row by row over the CTA's share of the output
//      rows (coalesced stores; PAD rows 0x00), then zero the PAD rows' codes (32-row chunks).
// ---------------------------------------------------------------------------------------------
constexpr int kDispMaxSlots = 32;
constexpr int kDispStoreSlack = 4;
constexpr size_t kDispSmemBudget = 220 * 1024;
constexpr int kDispListStride = 17;  // token id + up to 16 rows

template <int SLACK>
__global__ void __launch_bounds__(256) dispatch_engine_kernel(
    PeerPtrs2 peer, int64_t ld_s_tok, int64_t Tpr, int n, int64_t H, const int32_t* __restrict__ row_map, int K,
    const int32_t* __restrict__ src_of_row, const int32_t* __restrict__ offsets, int E_loc, int64_t max_rows,
    uint8_t* __restrict__ q_out, uint8_t* __restrict__ s_out, int nslots, int list_cap,
    const int32_t* __restrict__ gate) {
  if (gate != nullptr && *gate != 0) return;  // the barrier before it timed out: peers not ready
  extern __shared__ __align__(128) uint8_t smem_disp[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_disp);
  int32_t* list_n = reinterpret_cast<int32_t*>(full + kDispMaxSlots);
  int32_t* list = list_n + 4;
  uint8_t* slots = smem_disp + ((8 * kDispMaxSlots + 16 + 4 * static_cast<int64_t>(list_cap) * kDispListStride + 127) / 128) * 128;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = gridDim.x, cta = blockIdx.x;
  const int64_t T = Tpr * n;
  const int64_t n_tiles = H / 128;

  if (tid == 0) {
    for (int i = 0; i < nslots; ++i) mbar_init(&full[i], 1);
    mbar_init_fence();
    *list_n = 0;
  }
  __syncthreads();
  // every warp compacts 32-token batches (warp w: batches w, w+8, ...); list order is irrelevant
  // to the result (each row's content is fixed by row_map), so slots are taken with one shared
  // atomic per batch
  for (int64_t i0 = static_cast<int64_t>(warp) * 32; cta + i0 * G < T; i0 += 32 * 8) {
    const int64_t gt = cta + (i0 + lane) * G;
    int32_t rows[16];
    bool any = false;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      rows[k] = (gt < T && k < K) ? __ldg(row_map + gt * K + k) : -1;
      any |= rows[k] >= 0;
    }
    const uint32_t mask = __ballot_sync(0xffffffffu, any);
    int base = 0;
    if (lane == 0 && mask != 0) base = atomicAdd(list_n, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (any) {
      int32_t* e = list + (base + __popc(mask & ((1u << lane) - 1u))) * kDispListStride;
      e[0] = static_cast<int32_t>(gt);
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k < K) e[1 + k] = rows[k];
    }
  }
  __syncthreads();
  const int N = *list_n;

  if (warp == 0) {
    if (lane == 0) {
      const int lead = nslots - SLACK;
      uint32_t phase_bits = 0;
      for (int nn = 0; nn < N + lead; ++nn) {
        const int m = nn - lead;
        if (m >= 0) {  // store stage: token m is in slot m % nslots
          const int slot = m % nslots;
          mbar_wait(&full[slot], (phase_bits >> slot) & 1u);
          phase_bits ^= 1u << slot;
          const int32_t* e = list + m * kDispListStride;
          for (int k = 0; k < K; ++k)
            if (e[1 + k] >= 0)
              bulk_store_1d(q_out + static_cast<int64_t>(e[1 + k]) * H, slots + static_cast<int64_t>(slot) * H,
                            static_cast<uint32_t>(H));
          bulk_commit();
        }
        if (nn < N) {  // load stage
          const int slot = nn % nslots;
          if (nn >= nslots) bulk_wait_read<SLACK>();  // token nn - nslots's stores have read it
          const int64_t gt = list[nn * kDispListStride];
          const int src_rank = static_cast<int>(gt / Tpr);
          mbar_expect_tx(&full[slot], static_cast<uint32_t>(H));
          bulk_load_1d(slots + static_cast<int64_t>(slot) * H,
                       static_cast<const uint8_t*>(peer.a[src_rank]) + (gt - src_rank * Tpr) * H,
                       static_cast<uint32_t>(H), &full[slot]);
        }
      }
      bulk_wait_all();
    }
  } else {
    // scales, row-major like A3's move: the CTA's contiguous share of the output rows, (row, tile)
    // pairs with consecutive threads on consecutive rows (coalesced stores); a row's byte comes
    // from its source token's owner (src_of_row holds the global token id), PAD rows get 0x00
    const int64_t R_all = min64(offsets[E_loc], max_rows);
    const int64_t rb = cta * R_all / G;
    const int nr = static_cast<int>((cta + 1) * R_all / G - rb);
    // 8 (row, tile) pairs per thread in flight: the source-row loads, then the byte gathers, then
    // the stores (a dependent load -> load -> store chain per pair otherwise bounds the kernel's tail)
    const int tpr = static_cast<int>(Tpr);
    constexpr int kSU = 8;
    const int total = nr * static_cast<int>(n_tiles);
    for (int p0 = tid - 32; p0 < total; p0 += 224 * kSU) {
      int32_t src[kSU];
      int64_t r[kSU];
      int tl[kSU];
#pragma unroll
      for (int u = 0; u < kSU; ++u) {
        const int p = p0 + 224 * u;
        tl[u] = p < total ? p / nr : 0;
        r[u] = rb + (p - tl[u] * nr);
        src[u] = p < total ? __ldg(src_of_row + r[u]) : -2;
      }
      uint8_t v[kSU];
#pragma unroll
      for (int u = 0; u < kSU; ++u) {
        v[u] = 0;
        if (src[u] >= 0) {
          const int src_rank = src[u] / tpr;
          v[u] = __ldg(static_cast<const uint8_t*>(peer.b[src_rank]) + static_cast<int64_t>(tl[u]) * ld_s_tok +
                       (src[u] - src_rank * tpr));
        }
      }
#pragma unroll
      for (int u = 0; u < kSU; ++u)
        if (src[u] != -2) s_out[static_cast<int64_t>(tl[u]) * max_rows + r[u]] = v[u];
    }
    // PAD rows: 32-row chunks over the grid's warps 1..7
    const int64_t R = min64(offsets[E_loc], max_rows);  // an overflowed plan: only max_rows rows exist
    for (int64_t c = cta * 7 + (warp - 1); c * 32 < R; c += G * 7) {
      const int64_t r0 = c * 32;
      const bool pad = r0 + lane < R && src_of_row[r0 + lane] < 0;
      for (uint32_t msk = __ballot_sync(0xffffffffu, pad); msk != 0; msk &= msk - 1) {
        const int64_t r = r0 + __ffs(msk) - 1;
        for (int64_t i = lane * 16; i < H; i += 32 * 16) st_v4(q_out + r * H + i, make_uint4(0, 0, 0, 0));
      }
    }
  }
}

cudaError_t launch_dispatch_permute_pad(const uint8_t* const* peer_q, const uint8_t* const* peer_s, int64_t ld_s_tok,
                                        int32_t n, int64_t tokens_per_rank, int64_t hidden, const int32_t* row_map,
                                        int32_t top_k, const int32_t* src_of_row, const int32_t* expert_offsets,
                                        int32_t num_local_experts, int64_t max_rows, uint8_t* q_out, uint8_t* s_out,
                                        int32_t kernel, const int32_t* gate, cudaStream_t stream, int num_sms) {
  PeerPtrs2 pp{};
  for (int r = 0; r < n; ++r) {
    pp.a[r] = peer_q[r];
    pp.b[r] = peer_s[r];
  }
  const int64_t T = tokens_per_rank * n;
  // The bulk-copy engine reads peers with cp.async.bulk; that is verified only for buffers on the
  // calling device (virtual ranks, processes sharing a GPU).  AUTO takes the register-copy kernel
  // -- plain 128-bit loads, valid on every peer mapping -- when any peer's codes live on another
  // device (NVLink), or when the engine's shared-memory ring does not fit the shape.
  bool use_engine = kernel != 2;  // 0 auto, 1 engine, 2 register copies (fp8flow.h)
  if (kernel == 0) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    for (int r = 0; r < n && use_engine; ++r) {
      cudaPointerAttributes a;
      if (cudaPointerGetAttributes(&a, peer_q[r]) != cudaSuccess) {
        cudaGetLastError();
        use_engine = false;  // unknown mapping: take the path that is valid everywhere
      } else if (a.device != dev) {
        use_engine = false;
      }
    }
  }
  // engine geometry: 4 co-resident CTAs per SM share the shared-memory budget (1 CTA/SM 54 us,
  // 2 34.7, 4 32.8 at DSv3 sizes); more CTAs (queued) when a CTA would own more than 256 tokens
  constexpr int kCtasPerSm = 4;
  const size_t budget = kDispSmemBudget / kCtasPerSm;
  int64_t grid = static_cast<int64_t>(num_sms) * kCtasPerSm;
  if ((T + grid - 1) / grid > 256) grid = (T + 255) / 256;
  const int list_cap = static_cast<int>((T + grid - 1) / grid);
  const size_t head = ((8 * kDispMaxSlots + 16 + 4 * static_cast<size_t>(list_cap) * kDispListStride + 127) / 128) * 128;
  int nslots = head + static_cast<size_t>(hidden) * (kDispStoreSlack + 2) <= budget
                   ? static_cast<int>((budget - head) / hidden) : 0;
  if (nslots > kDispMaxSlots) nslots = kDispMaxSlots;
  if (use_engine && nslots < kDispStoreSlack + 2) {
    if (kernel == 1) return cudaErrorInvalidValue;  // explicitly requested, cannot run this shape
    use_engine = false;
  }
  if (!use_engine) {
    static KernelSetup lsu_setup;
    const int occ = prepare_kernel(lsu_setup, dispatch_permute_lsu_kernel, kEpThreads, 0, 0);
    if (occ == 0) return cudaErrorInvalidValue;
    const int64_t need = (T + kEpWarps - 1) / kEpWarps;
    const int64_t lgrid = one_wave_grid(occ, num_sms, need > num_local_experts ? need : num_local_experts);
    dispatch_permute_lsu_kernel<<<static_cast<unsigned>(lgrid), kEpThreads, 0, stream>>>(
        pp, ld_s_tok, tokens_per_rank, n, hidden, row_map, top_k, src_of_row, expert_offsets, num_local_experts,
        max_rows, q_out, s_out, gate);
    return cudaGetLastError();
  }
  const size_t smem = head + static_cast<size_t>(hidden) * nslots;
  static KernelSetup engine_setup;
  if (prepare_kernel(engine_setup, dispatch_engine_kernel<kDispStoreSlack>, 256, kDispSmemBudget, smem) == 0)
    return cudaErrorInvalidValue;
  dispatch_engine_kernel<kDispStoreSlack><<<static_cast<unsigned>(grid), 256, smem, stream>>>(
      pp, ld_s_tok, tokens_per_rank, n, hidden, row_map, top_k, src_of_row, expert_offsets, num_local_experts,
      max_rows, q_out, s_out, nslots, list_cap, gate);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// combine + unpermute (owner side): warp per owned token; lane k resolves (rank, row, gate) of its
// expert; column passes of 2 x 8 BF16 per lane, rows taken four at a time so 8 x 16 B loads per
// lane are in flight, then acc = fmaf(p_k, x_k, acc) strictly in k order; BF16 RNE 128-bit stores.
// ---------------------------------------------------------------------------------------------
constexpr int kCombU = 2;   // 16-byte chunks per lane per pass
constexpr int kCombKB = 8;  // rows loaded together

__global__ void __launch_bounds__(kEpThreads) combine_kernel(PeerPtrs2 peer, int n, int64_t H,
                                                             const int32_t* __restrict__ topk_idx, int E_per,
                                                             const float* __restrict__ probs, int64_t token_begin,
                                                             int64_t T, int K, __nv_bfloat16* __restrict__ y,
                                                             const int32_t* __restrict__ gate) {
  if (gate != nullptr && *gate != 0) return;  // the barrier before it timed out: peers not ready
  const int lane = threadIdx.x & 31;
  const int64_t W = static_cast<int64_t>(gridDim.x) * kEpWarps;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kEpWarps + (threadIdx.x >> 5);
  const int64_t nchunk = H / 8;
  for (int64_t t = gw; t < T; t += W) {
    // lane k: the expert's rank and row on that rank (a 4-byte load from the rank's plan)
    const uint8_t* my_base = nullptr;
    float my_p = 0.0f;
    if (lane < K) {
      const int e = __ldg(topk_idx + t * K + lane);
      const int d = e / E_per;
      if (e >= 0 && d < n) {
        const int32_t r = static_cast<const int32_t*>(peer.b[d])[(token_begin + t) * K + lane];
        if (r >= 0) {
          my_base = static_cast<const uint8_t*>(peer.a[d]) + static_cast<int64_t>(r) * H * 2;
          my_p = probs != nullptr ? __ldg(probs + t * K + lane) : 1.0f;
        }
      }
    }
    const uint32_t valid = __ballot_sync(0xffffffffu, my_base != nullptr);
    const int nk = __popc(valid);
    // compact the valid terms to lanes 0..nk-1, k order preserved
    const int from = static_cast<int>(__fns(valid, 0, lane + 1)) & 31;
    const uint64_t cb = __shfl_sync(0xffffffffu, reinterpret_cast<uint64_t>(my_base), from);
    const float cp = __shfl_sync(0xffffffffu, my_p, from);
    for (int64_t c0 = 0; c0 < nchunk; c0 += 32 * kCombU) {
      float acc[kCombU][8];
#pragma unroll
      for (int u = 0; u < kCombU; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[u][j] = 0.0f;
      for (int i0 = 0; i0 < nk; i0 += kCombKB) {
        uint4 v[kCombKB][kCombU];
        float p[kCombKB];
#pragma unroll
        for (int b = 0; b < kCombKB; ++b) {
          const uint64_t base = __shfl_sync(0xffffffffu, cb, (i0 + b) & 31);
          p[b] = __shfl_sync(0xffffffffu, cp, (i0 + b) & 31);
#pragma unroll
          for (int u = 0; u < kCombU; ++u) {
            const int64_t c = c0 + lane + 32 * u;
            if (i0 + b < nk && c < nchunk) v[b][u] = ld_nc_v4(reinterpret_cast<const uint8_t*>(base) + c * 16);
          }
        }
#pragma unroll
        for (int b = 0; b < kCombKB; ++b) {
          if (i0 + b < nk) {
#pragma unroll
            for (int u = 0; u < kCombU; ++u) {
              const uint32_t w[4] = {v[b][u].x, v[b][u].y, v[b][u].z, v[b][u].w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                acc[u][2 * j] = __fmaf_rn(p[b], bf16lo_to_f32(w[j]), acc[u][2 * j]);
                acc[u][2 * j + 1] = __fmaf_rn(p[b], bf16hi_to_f32(w[j]), acc[u][2 * j + 1]);
              }
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kCombU; ++u) {
        const int64_t c = c0 + lane + 32 * u;
        if (c < nchunk) {
          uint32_t o[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            __nv_bfloat162 bb = __floats2bfloat162_rn(acc[u][2 * j], acc[u][2 * j + 1]);
            o[j] = *reinterpret_cast<uint32_t*>(&bb);
          }
          st_v4(y + t * H + c * 8, make_uint4(o[0], o[1], o[2], o[3]));
        }
      }
    }
  }
}

cudaError_t launch_combine_unpermute(const void* const* peer_x, const int32_t* const* peer_row_map, int32_t n,
                                     int64_t hidden, const int32_t* topk_idx, int32_t experts_per_rank,
                                     const float* probs, int64_t token_begin, int64_t num_tokens, int32_t top_k,
                                     void* y, const int32_t* gate, cudaStream_t stream, int num_sms) {
  PeerPtrs2 pp{};
  for (int r = 0; r < n; ++r) {
    pp.a[r] = peer_x[r];
    pp.b[r] = peer_row_map[r];
  }
  static KernelSetup setup;
  const int occ = prepare_kernel(setup, combine_kernel, kEpThreads, 0, 0);
  if (occ == 0) return cudaErrorInvalidValue;
  const int64_t grid = one_wave_grid(occ, num_sms, (num_tokens + kEpWarps - 1) / kEpWarps);
  combine_kernel<<<static_cast<unsigned>(grid), kEpThreads, 0, stream>>>(
      pp, n, hidden, topk_idx, experts_per_rank, probs, token_begin, num_tokens, top_k,
      static_cast<__nv_bfloat16*>(y), gate);
  return cudaGetLastError();
}

}  // namespace fp8flow
