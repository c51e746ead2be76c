// permute_dual.cu -- NEXT-1 dual-output fusion of the A3 move with A2 (R37): the permute
// + pad move emitting, from ONE gathered copy of each 128 x 128 block in shared memory,
// both the padded expert-major row-wise FP8 tensor X_perm (the Fprop operand) and its scaling-aware
// transpose per expert (Algorithm 1; the Wgrad operand).  Unfused, the same
// result is fp8flow_permute_pad (write X_perm) followed by fp8flow_scaling_aware_transpose with the
// plan's expert offsets as segments (read X_perm back, write X_perm^T): the fusion removes the
// re-read of X_perm -- 7168 bytes per padded row, ~0.95 GB per DeepSeek-V3 layer.
//
// Semantics = composition: (q_out, s_out) are exactly permute_pad's (q_out[r] = q_tok[src_of_row[r]],
// PAD rows code 0x00 / scale 0x00), (qT, sT) exactly A2 of them with segments = expert_offsets:
//     T_max = max_i T[i][jb];  sT_e[ib][j] = T_max;  qT_e[j][i-o] = shift(q_out[i][j], T_max - T[i][jb]).
//
// Kernel: A2's persistent, warp-specialised structure (transpose.cu) with gathering producers, units
// of W column blocks (W = 2 for launches with >= 32 blocks per SM: 256-byte pieces of every token
// and X_perm row, as A2's two-block units) in A2's segment-major order but unit column by unit
// column (all experts' units of one column before the next: the token pieces gathered meanwhile
// stay in L2 for the ~8 expert rows that read each):
//   * 4 producer warps: warp p gathers block rows 32p..32p+31 with 16-byte cp.async (each warp
//     instruction = 4 rows x 128 bytes; PAD rows by zero-fill) and writes their scale bytes; a
//     tile's two dependent global reads (src_of_row, then s_tok) are issued 4 and 2 tiles ahead as
//     4-byte cp.async into a shared-memory ring; tile coordinates are computed 32 at a time, one
//     per lane, and shuffled out; the stage's mbarrier counts each lane's cp.async completion and
//     its arrival after the scale writes;
//   * 8 consumer warps: thread (g, c) copies block rows 4g..4g+3 x bytes 16c..16c+15 to registers,
//     stores them unchanged to q_out (each warp store = 4 full 128-byte row segments), warp 0
//     stores the scale run to s_out, then A2's shift + 4x4 byte transposes into a staging buffer;
//   * 4 store warps: drain the staging buffers to qT (A2's coalesced 128-bit stores) and write sT.
// Outputs are stored with an L2 evict-first policy, the gathered tokens loaded evict-last.
#include <cuda.h>

#include "async.cuh"
#include "common.cuh"
#include "kernels.h"
#include "segments.cuh"

namespace fp8flow {

namespace {

constexpr int kPdCons = 256;  // 8 consumer warps
constexpr int kPdMaxSegs = 1024;
constexpr int kPdProducers = 4;  // producer warps: 32 block rows each
// tiles walked in column chunks of one block: all experts' tiles of column block jb before jb + 1,
// so the token bytes gathered meanwhile (num_tokens x 128) stay in L2 for their ~8 expert rows
constexpr int kPdChunk = 1;

#ifndef PDDEPTH
#define PDDEPTH 4
#endif
constexpr int kPdDepth = PDDEPTH;  // tiles whose sources are in flight (scales: kPdDepth - 2)
static_assert(kPdDepth >= 4, "a tile's scales must be two cp.async groups old when it is issued");
template <int WS>
__host__ __device__ constexpr int pd_threads() { return kPdCons + 32 * WS + 32 * kPdProducers; }  // + store warps + producers
constexpr int kPdMaxThreads = pd_threads<4>();

template <int STAGES, int W>
struct PermDualSmem {
  uint8_t in[STAGES][W * kTile * kTile];  // gathered unit: row i = token src_of_row[r0 + i], W*128 bytes
  uint32_t sc[STAGES][W][kTile / 4];      // the 128 row-scale bytes of each of the W blocks
  uint32_t out[2][kTile * kTile / 4]; // transposed staging (A2's swizzle)
  TileCoord tc[STAGES];
  TileCoord out_tc[2];                // pad[0] = T_max
  uint64_t full_bar[STAGES];          // 32 producer-lane arrivals + the bulk-copied bytes
  uint64_t empty_bar[STAGES];
  uint64_t out_full[2];
  uint64_t out_empty[2];
  int32_t psrc[kPdProducers][kPdDepth * 32];  // per producer warp: ring of source tokens
  uint32_t psc[kPdProducers][kPdDepth * W * 32];  // ... and of the words holding their scale bytes
  uint32_t mult[33];
  uint32_t red[kPdMaxThreads / 32];
  int32_t total_rb;
  // followed in dynamic shared memory by seg_off[num_segs + 1] and blk_prefix[num_segs + 1]
};
template <typename Smem>
__host__ __device__ constexpr size_t pd_smem_bytes(int nsegs) {
  return (sizeof(Smem) + 15) / 16 * 16 + 8 * static_cast<size_t>(nsegs + 1);
}

// 16-byte cp.async (LDGSTS, L2 only); src_bytes 0 fills the 16 destination bytes with zeros;
// `policy` an L2 cache policy (createpolicy)
__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, uint32_t src_bytes, uint64_t policy) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes), "l"(policy)
               : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_v4_hint(void* p, uint4 v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w), "l"(policy)
               : "memory");
}
// 4-byte cp.async (L1-allocating .ca: sizes below 16), in the current group
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// arrive on `bar` once every cp.async this thread issued so far has completed (counts as one of
// the barrier's expected arrivals)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int STAGES, int MINB, int WS, int W>
__global__ void __launch_bounds__(pd_threads<WS>(), MINB)
    permute_dual_kernel(const uint8_t* __restrict__ q_tok, const uint8_t* __restrict__ s_tok, int64_t ld_s_tok,
                        int64_t hidden, const int32_t* __restrict__ src_of_row,
                        const int32_t* __restrict__ expert_offsets, int32_t num_segs, int64_t max_rows,
                        uint8_t* __restrict__ q_out, uint8_t* __restrict__ s_out, uint8_t* __restrict__ qT,
                        uint8_t* __restrict__ sT) {
  extern __shared__ __align__(1024) uint8_t smem_pd[];
  using Smem = PermDualSmem<STAGES, W>;
  Smem& sm = *reinterpret_cast<Smem*>(smem_pd);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int32_t* seg_off = reinterpret_cast<int32_t*>(smem_pd + (sizeof(Smem) + 15) / 16 * 16);
  int32_t* blk_prefix = seg_off + num_segs + 1;
  const SegTables segt{seg_off, blk_prefix};
  constexpr int kThreads = pd_threads<WS>();
  constexpr int kProducerWarp = kPdCons / 32 + WS;

  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&sm.full_bar[i], 2 * 32 * kPdProducers);  // per producer lane: copies landed + writes
      mbar_init(&sm.empty_bar[i], kPdCons);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.out_full[i], kPdCons);
      mbar_init(&sm.out_empty[i], 32 * WS);
    }
    mbar_init_fence();
  }
  if (tid <= 32) sm.mult[tid] = shift_multiplier(static_cast<uint32_t>(tid));
  // the plan's offsets, clamped to the buffer (an overflowed plan reports its true total)
  load_segments<kThreads>(seg_off, blk_prefix, sm.red, &sm.total_rb, expert_offsets, num_segs, max_rows,
                          static_cast<int32_t>(max_rows));  // (+ barrier)

  const int n_jb = static_cast<int>(hidden / (W * kTile));  // units of W column blocks
  const int total_tiles = sm.total_rb * n_jb;
  const int first = blockIdx.x;
  const int stride = gridDim.x;
  const int n_local = first < total_tiles ? (total_tiles - first + stride - 1) / stride : 0;

  if (warp >= kPdCons / 32 && warp < kProducerWarp) {
    // ---- store warps: A2's drain of staging buffer b (transposed tile) + its sT run
    const int st_tid = tid - kPdCons;
    const int c8 = st_tid & 7;
    const uint64_t pol_out = l2_policy_evict_first();  // streamed outputs
    for (int i = 0; i < n_local * W; ++i) {  // one staged output per column block
      const int b = i & 1;
      mbar_wait(&sm.out_full[b], (i >> 1) & 1);
      const TileCoord tc = sm.out_tc[b];
      const uint32_t* out = sm.out[b];
      uint8_t* qTe = qT + hidden * static_cast<int64_t>(tc.o);
      if (16 * c8 < tc.rows_valid) {
#pragma unroll 4
        for (int j = st_tid >> 3; j < kTile; j += 4 * WS) {
          const int phys = c8 ^ ((j >> 4) & 7);
          const uint4 o4 = *reinterpret_cast<const uint4*>(&out[j * 32 + 4 * phys]);
          st_v4_hint(qTe + (static_cast<int64_t>(tc.jb) * kTile + j) * tc.m + tc.ib * kTile + 16 * c8, o4, pol_out);
        }
      }
      if (st_tid < 8) {
        const uint32_t b4 = static_cast<uint32_t>(tc.pad[0]) * 0x01010101u;
        st_v4(sT + static_cast<int64_t>(tc.rb) * hidden + tc.jb * kTile + 16 * st_tid, make_uint4(b4, b4, b4, b4));
      }
      mbar_arrive(&sm.out_empty[b]);
    }
    return;
  }
  if (warp >= kProducerWarp) {
    // ---- producer warps: gather tile i = first + i * stride into stage st.  Warp p copies block
    // rows [32p, 32p + 32): lane l owns row 32p + l's source token and scale byte, and the warp's
    // 16-byte cp.async (LDGSTS) instructions move 4 rows x 128 bytes each (PAD rows by zero-fill).
    // A tile's two dependent global reads -- its sources, then their scale bytes -- are issued
    // kPdDepth and kPdDepth - 2 tiles ahead as 4-byte cp.async into a shared-memory ring (no
    // register waits on the loads), one cp.async group per tile.
    const int pw = warp - kProducerWarp;
    const int row = pw * 32 + lane;  // this lane's block row
    int32_t* rsrc = sm.psrc[pw];     // [kPdDepth][32] source tokens of tiles i .. i + kPdDepth - 1
    uint32_t* rsc = sm.psc[pw];      // [kPdDepth][32] the 4-byte words holding their scale bytes
    const uint64_t pol_in = l2_policy_evict_last();
    auto coord = [&](int i) {
      TileCoord c = i < n_local ? tile_coord_chunked(segt, num_segs, n_jb, sm.total_rb, kPdChunk, first + i * stride)
                                : TileCoord{};
      c.jb *= W;  // the unit's first column block
      return c;
    };
    // tile coordinates, 32 at a time: lane k computes those of tiles base + k (cur) and
    // base + 32 + k (nxt); using one costs a shuffle per field
    TileCoord cur = coord(lane), nxt = coord(32 + lane);
    int base = 0;
    auto get = [&](int i) {  // i in [base, base + 64), warp-uniform
      const int k = i & 31;
      const bool in_cur = i < base + 32;
      TileCoord c;
      c.o = __shfl_sync(0xffffffffu, in_cur ? cur.o : nxt.o, k);
      c.m = __shfl_sync(0xffffffffu, in_cur ? cur.m : nxt.m, k);
      c.ib = __shfl_sync(0xffffffffu, in_cur ? cur.ib : nxt.ib, k);
      c.jb = __shfl_sync(0xffffffffu, in_cur ? cur.jb : nxt.jb, k);
      c.rb = __shfl_sync(0xffffffffu, in_cur ? cur.rb : nxt.rb, k);
      c.rows_valid = __shfl_sync(0xffffffffu, in_cur ? cur.rows_valid : nxt.rows_valid, k);
      return c;
    };
    auto issue_src = [&](int i) {  // src_of_row of this lane's row of tile i -> rsrc slot
      int32_t* d = &rsrc[(i % kPdDepth) * 32 + lane];
      if (i >= n_local) return;
      const TileCoord c = get(i);
      if (row < c.rows_valid) cp_async4(d, src_of_row + static_cast<int64_t>(c.o) + c.ib * kTile + row);
      else *d = -1;
    };
    auto issue_scale = [&](int i) {  // the words of s_tok[jb + h] holding this row's scale bytes -> rsc
      if (i >= n_local) return;
      const int sl = (i % kPdDepth) * 32 + lane;
      const int src = rsrc[sl];
      const int jb = get(i).jb;  // (shuffles: every lane)
#pragma unroll
      for (int h = 0; h < W; ++h)
        if (src >= 0)
          cp_async4(&rsc[((i % kPdDepth) * W + h) * 32 + lane],
                    s_tok + static_cast<int64_t>(jb + h) * ld_s_tok + (src & ~3));
    };
#pragma unroll 1
    for (int d = 0; d < kPdDepth; ++d) issue_src(d);
    cp_async_commit();
    cp_async_wait<0>();
#pragma unroll 1
    for (int d = 0; d < kPdDepth - 2; ++d) issue_scale(d);
    cp_async_commit();
    cp_async_wait<0>();
    int st = 0;
    uint32_t phase = 0;
    for (int i = 0; i < n_local; ++i) {
      if (i + kPdDepth >= base + 64) {  // the lookahead leaves the two coordinate batches
        cur = nxt;
        base += 32;
        nxt = coord(base + 32 + lane);
      }
      cp_async_wait<1>();  // every group but the last: sources of tile i + kPdDepth - 2, scales of tile i
      issue_scale(i + kPdDepth - 2);
      const TileCoord c0 = get(i);
      const int sl0 = (i % kPdDepth) * 32;
      if (i >= STAGES) mbar_wait_sleep(&sm.empty_bar[st], phase ^ 1u, 32);
      if (lane == 0 && pw == 0) sm.tc[st] = c0;
      // a warp instruction copies 32 / (8 W) rows of W * 128 bytes (8 W lanes per row)
      constexpr int kLpr = 8 * W, kRpi = 32 / kLpr;
      const int col = c0.jb * kTile + 16 * (lane % kLpr);
      const int my_src = rsrc[sl0 + lane];  // this lane's own cp.async result (complete, visible to it)
#pragma unroll
      for (int k = 0; k < 32 / kRpi; ++k) {
        const int r = pw * 32 + kRpi * k + lane / kLpr;
        const int src = __shfl_sync(0xffffffffu, my_src, kRpi * k + lane / kLpr);
        if (r < c0.rows_valid) {
          cp_async16_zfill(sm.in[st] + r * (W * kTile) + 16 * (lane % kLpr),
                           q_tok + static_cast<int64_t>(src >= 0 ? src : 0) * hidden + col, src >= 0 ? 16u : 0u,
                           pol_in);
        }
      }
      cp_async_mbar_arrive(&sm.full_bar[st]);  // arrives once this lane's copies have landed
      if (row < c0.rows_valid) {
#pragma unroll
        for (int h = 0; h < W; ++h)
          reinterpret_cast<uint8_t*>(sm.sc[st][h])[row] =
              my_src >= 0 ? static_cast<uint8_t>(rsc[((i % kPdDepth) * W + h) * 32 + lane] >> (8 * (my_src & 3)))
                          : uint8_t{0};
      }
      mbar_arrive(&sm.full_bar[st]);  // releases this lane's scale / coordinate writes
      issue_src(i + kPdDepth);  // into slot i % kPdDepth (read above by this lane only)
      cp_async_commit();
      if (++st == STAGES) {
        st = 0;
        phase ^= 1u;
      }
    }
    cp_async_wait<0>();
    return;
  }

  // ---- consumer warps (256 threads): thread (g, c) = block rows 4g..4g+3 x bytes 16c..16c+15
  const int g = tid >> 3;
  const int c = tid & 7;
  const uint64_t pol_out = l2_policy_evict_first();  // streamed outputs
  int st = 0;
  uint32_t phase = 0;
  for (int i = 0; i < n_local; ++i) {
    mbar_wait(&sm.full_bar[st], phase);
    const TileCoord tc = sm.tc[st];
    const int64_t r0 = static_cast<int64_t>(tc.o) + tc.ib * kTile;
#pragma unroll 1
    for (int h = 0; h < W; ++h) {
      const int o = i * W + h;  // staged output index
      const int jb = tc.jb + h;
      // block scale max (Algorithm 1), per warp; rows beyond the segment count as 0
      const uint32_t sw_l = (4 * lane < tc.rows_valid) ? sm.sc[st][h][lane] : 0u;
      const uint32_t mx = max(max(sw_l & 0xFFu, (sw_l >> 8) & 0xFFu), max((sw_l >> 16) & 0xFFu, sw_l >> 24));
      const uint32_t tmax = __reduce_max_sync(0xffffffffu, mx);
      const uint32_t sw = __shfl_sync(0xffffffffu, sw_l, g);
      if (warp == 0 && 4 * lane < tc.rows_valid)  // row-wise scales: s_out[jb][r0 + 4l .. + 3]
        *reinterpret_cast<uint32_t*>(s_out + static_cast<int64_t>(jb) * max_rows + r0 + 4 * lane) = sw_l;
      uint4 v[4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
        v[r] = *reinterpret_cast<const uint4*>(&sm.in[st][(4 * g + r) * (W * kTile) + h * kTile + 16 * c]);
      if (h == W - 1) mbar_arrive(&sm.empty_bar[st]);
      // row-wise output: the gathered codes unchanged (a warp store = 4 rows x 128 bytes; the W
      // blocks of a unit give each row W * 128 contiguous bytes)
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (4 * g + r < tc.rows_valid)
          st_v4_hint(q_out + (r0 + 4 * g + r) * hidden + jb * kTile + 16 * c, v[r], pol_out);
      // A2's exponent shift (rows past rows_valid hold stale bytes: shifted, never stored)
      uint32_t R[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint32_t k = tmax - ((sw >> (8 * r)) & 0xFFu);
        const uint32_t m2 = sm.mult[k < 32u ? k : 32u];
        R[r][0] = shift4(v[r].x, m2);
        R[r][1] = shift4(v[r].y, m2);
        R[r][2] = shift4(v[r].z, m2);
        R[r][3] = shift4(v[r].w, m2);
      }
      const int wpos = 4 * ((g >> 2) ^ c) + (g & 3);
      uint32_t* out = sm.out[o & 1];
      if (o >= 2) mbar_wait(&sm.out_empty[o & 1], ((o >> 1) - 1) & 1);
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint32_t t0 = __byte_perm(R[0][w], R[1][w], 0x5140);
        const uint32_t t1 = __byte_perm(R[0][w], R[1][w], 0x7362);
        const uint32_t t2 = __byte_perm(R[2][w], R[3][w], 0x5140);
        const uint32_t t3 = __byte_perm(R[2][w], R[3][w], 0x7362);
        const int j0 = 16 * c + 4 * w;
        out[(j0 + 0) * 32 + wpos] = __byte_perm(t0, t2, 0x5410);
        out[(j0 + 1) * 32 + wpos] = __byte_perm(t0, t2, 0x7632);
        out[(j0 + 2) * 32 + wpos] = __byte_perm(t1, t3, 0x5410);
        out[(j0 + 3) * 32 + wpos] = __byte_perm(t1, t3, 0x7632);
      }
      if (tid == 0) {
        TileCoord ob = tc;
        ob.jb = jb;
        ob.pad[0] = static_cast<int32_t>(tmax);
        sm.out_tc[o & 1] = ob;
      }
      __syncwarp();
      mbar_arrive(&sm.out_full[o & 1]);
    }
    if (++st == STAGES) {
      st = 0;
      phase ^= 1u;
    }
  }
}

template <int S, int B, int WS, int W>
cudaError_t launch_pd(const uint8_t* q_tok, const uint8_t* s_tok, int64_t ld_s_tok, int64_t hidden,
                      const int32_t* src_of_row, const int32_t* expert_offsets, int32_t num_segs, int64_t max_rows,
                      uint8_t* q_out, uint8_t* s_out, uint8_t* qT, uint8_t* sT, cudaStream_t stream, int num_sms,
                      int64_t ub_tiles) {
  static KernelSetup setup;
  auto kernel = permute_dual_kernel<S, B, WS, W>;
  constexpr int kThreads = pd_threads<WS>();
  const size_t smem = pd_smem_bytes<PermDualSmem<S, W>>(num_segs);
  if (prepare_kernel(setup, kernel, kThreads, pd_smem_bytes<PermDualSmem<S, W>>(kPdMaxSegs), smem) == 0)
    return cudaErrorInvalidValue;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem) != cudaSuccess || occ < 1) occ = 1;
  const int64_t grid = one_wave_grid(occ, num_sms, (ub_tiles + W - 1) / W);
  kernel<<<static_cast<unsigned>(grid), kThreads, smem, stream>>>(q_tok, s_tok, ld_s_tok, hidden, src_of_row,
                                                                  expert_offsets, num_segs, max_rows, q_out, s_out,
                                                                  qT, sT);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_permute_pad_dual(const uint8_t* q_tok, const uint8_t* s_tok, int64_t ld_s_tok, int64_t hidden,
                                    const int32_t* src_of_row, const int32_t* expert_offsets,
                                    int32_t num_local_experts, int64_t max_rows, uint8_t* q_out, uint8_t* s_out,
                                    uint8_t* qT, uint8_t* sT, cudaStream_t stream, int num_sms) {
  const int64_t ub_tiles = (max_rows / kTile + num_local_experts) * (hidden / kTile);
  // as A2: launches with >= 32 blocks per SM gather units of 2 column blocks (256 contiguous bytes
  // of every token row and of every X_perm row per unit); 1 CTA per SM with 3 stages from 64 blocks
  // per SM (whole layer 599 -> 561-564 us; 2 CTAs/SM there: 620), 2 CTAs per SM with 2 stages below
  // (EP8 shard 61.4 -> 60.2 us)
  const bool wide = hidden % (2 * kTile) == 0 && ub_tiles >= 32LL * num_sms;
  if (wide && ub_tiles >= 64LL * num_sms)
    return launch_pd<3, 1, 4, 2>(q_tok, s_tok, ld_s_tok, hidden, src_of_row, expert_offsets, num_local_experts,
                                 max_rows, q_out, s_out, qT, sT, stream, num_sms, ub_tiles);
  if (wide)
    return launch_pd<2, 2, 4, 2>(q_tok, s_tok, ld_s_tok, hidden, src_of_row, expert_offsets, num_local_experts,
                                 max_rows, q_out, s_out, qT, sT, stream, num_sms, ub_tiles);
  // 2 CTAs per SM (448-thread CTAs: 3 per SM would spill), 3 stages, 4 store warps
  return launch_pd<3, 2, 4, 1>(q_tok, s_tok, ld_s_tok, hidden, src_of_row, expert_offsets, num_local_experts,
                               max_rows, q_out, s_out, qT, sT, stream, num_sms, ub_tiles);
}

}  // namespace fp8flow
