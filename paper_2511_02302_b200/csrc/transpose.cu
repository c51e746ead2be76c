// transpose.cu -- A2: scaling-aware FP8 transpose (Algorithm 1), plus the naive
// dequantize -> transpose -> requantize comparator used only for benchmarking.
//
// A2 semantics (R5-R7, R14, R15, R23): per segment e = [o, o+m) (an expert's rows,
// m a multiple of 16) and per block (ib, jb) = rows o+128ib.. (partial last block) x columns
// 128jb..128jb+127:
//     T_max = max_i T[i][jb];  sT_e[ib][j] = T_max;  qT_e[j][i-o] = shift(q[i][j], T_max - T[i][jb])
//
// Kernel design (sm_100a, HBM-bound, 2.016 B/element):
//   * persistent CTAs, warp-specialised: 8 consumer warps (shift + transpose), 2-4 store warps
//     (read-out + global stores) and one producer warp; below 64 tiles per SM 3 CTAs per SM with
//     2 TMA stages and 2 store warps; above, W = 2 column blocks per staged unit (one 256-byte x
//     128-row box: input rows read 256 contiguous bytes at a time), 1 CTA per SM with 3-4 stages
//     and 4 store warps -- the consumers transpose the unit's two 128x128 blocks one after the other
//     (each with its own T_max) into the staging buffers.  Units are walked in segment-major order
//     (segments.cuh tile_coord); the segment tables are built in shared memory from the DEVICE
//     segment offsets (no host sync: CUDA-graph capturable).
//   * producer (one lane): per tile its coordinates, the 16 KB code tile by TMA (one 128x128 box,
//     or 16-row boxes for a segment's partial last block, so no bytes of the next segment are
//     read) and the block's run of row scales by a 1D bulk copy, all on one mbarrier of the stage
//     ring; it refills a stage as soon as every consumer warp has copied it to registers.
//   * T_max per block: each warp max-reduces the staged scale run itself (redux.sync), no barrier.
//   * thread (g, c) owns rows 4g..4g+3 x bytes 16c..16c+15: 4 conflict-free LDS.128 (8 threads of
//     a quarter-warp read one full 128-byte row); the per-row exponent shift (common.cuh shift4:
//     hardware e4m3x2 -> f16x2 decode, one HMUL2 by 2^-k, one RNE back, 8 instructions per 4
//     codes) is applied to whole 32-bit words (4 codes of one row share k), then 4x4 byte blocks
//     are transposed with PRMT.
//   * the transposed words go to one of two 16 KB staging buffers with a 16-byte-chunk XOR swizzle
//     (chunk ^= j/16) that makes both the 32-bit writes and the 128-bit read-out conflict-free; the
//     store warps drain a buffer (coalesced 128-bit stores, each output row's 128 bytes one full
//     line) while the consumers fill the other -- handed over on mbarriers, no CTA-wide barrier.
#include <cuda.h>

#include "async.cuh"
#include "common.cuh"
#include "kernels.h"
#include "segments.cuh"


namespace fp8flow {

// <STAGES, OUTBUF>: TMA stages of the input ring and staging buffers for the transposed tile
constexpr int kTConsumers = 256;              // 8 consumer (shift + transpose) warps
constexpr int kMaxThreadsA2 = kTConsumers + 32 * 8 + 32;
constexpr int kPrefixThreads = 288;             // 4 segments per thread: covers offsets[0..1024]
template <int WS>
__host__ __device__ constexpr int a2_threads() { return kTConsumers + 32 * WS + 32; }  // + WS store warps + 1 producer
constexpr int kMaxSegs = 1024;
constexpr int kTileBytes = kTile * kTile;

template <int STAGES, int OUTBUF, int W = 1>
struct TransposeSmem {
  uint8_t in[STAGES][W * kTileBytes];  // W column blocks of 128 rows (rows W*128 bytes apart)
  uint32_t sc[STAGES][W][kTile / 4];   // the 128 row-scale bytes of each of the W blocks
  uint32_t out[OUTBUF][kTile * kTile / 4];
  TileCoord tc[STAGES];            // coordinates of the staged tile (written by the producer)
  TileCoord out_tc[OUTBUF];        // coordinates (pad[0] = T_max) of the tile in each staging buffer
  uint64_t full_bar[STAGES];
  uint64_t empty_bar[STAGES];
  uint64_t out_full[OUTBUF];       // store-warp mode: staging buffer written / drained
  uint64_t out_empty[OUTBUF];
  uint32_t mult[33];               // f16x2 multiplier 2^-k for k = 0..32
  uint32_t red[kMaxThreadsA2 / 32];
  int32_t total_rb;
  // followed in dynamic shared memory by seg_off[num_segs + 1] and blk_prefix[num_segs + 1]
};
template <typename Smem>
__host__ __device__ constexpr size_t a2_smem_bytes(int nsegs) {
  return (sizeof(Smem) + 15) / 16 * 16 + 8 * static_cast<size_t>(nsegs + 1);
}
// WS > 0 (store-warp mode, OUTBUF == 2): WS extra warps drain the staging buffers (read-out and
// global stores) while the 8 consumer warps shift and transpose the next tile; buffers are handed
// over on out_full / out_empty mbarriers instead of consumer-wide barriers.
template <int STAGES, int OUTBUF, int MINB, int WS, int W>
__global__ void __launch_bounds__(a2_threads<WS>(), MINB)
    scaling_aware_transpose_kernel(const __grid_constant__ CUtensorMap tmap_q,
                                   const __grid_constant__ CUtensorMap tmap_q16, const uint8_t* __restrict__ s,
                                   int64_t ld_s, int64_t rows, int64_t cols, const int32_t* __restrict__ seg_offsets,
                                   int32_t num_segs, uint8_t* __restrict__ qT, uint8_t* __restrict__ sT) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  using Smem = TransposeSmem<STAGES, OUTBUF, W>;
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nsegs = seg_offsets == nullptr ? 1 : num_segs;
  int32_t* seg_off = reinterpret_cast<int32_t*>(smem_raw + (sizeof(Smem) + 15) / 16 * 16);
  int32_t* blk_prefix = seg_off + nsegs + 1;
  const SegTables segt{seg_off, blk_prefix};

  static_assert(WS > 0 && OUTBUF == 2, "store warps drain a double staging buffer");
  constexpr int kThreads = a2_threads<WS>();
  constexpr int kProducerWarp = kTConsumers / 32 + WS;
  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&sm.full_bar[i], 1);
      mbar_init(&sm.empty_bar[i], kTConsumers);
    }
    for (int i = 0; i < OUTBUF; ++i) {  // every thread arrives: each releases its own accesses
      mbar_init(&sm.out_full[i], kTConsumers);
      mbar_init(&sm.out_empty[i], 32 * WS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_q)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_q16)) : "memory");
  }
  if (tid <= 32) sm.mult[tid] = shift_multiplier(static_cast<uint32_t>(tid));
  load_segments<kThreads>(seg_off, blk_prefix, sm.red, &sm.total_rb, seg_offsets, nsegs, rows);  // (+ barrier)

  const int n_jb = static_cast<int>(cols / (kTile * W));  // staged units: W column blocks each
  const int total_tiles = sm.total_rb * n_jb;  // < 2^31 (rows < 2^31, checked by the ABI)
  const int first = blockIdx.x;
  const int stride = gridDim.x;
  const int n_local = first < total_tiles ? (total_tiles - first + stride - 1) / stride : 0;

  if (warp >= kTConsumers / 32 && warp < kProducerWarp) {
    // ---- store warps: drain staging buffer b of tile i (coalesced 128-bit stores, 16 bytes per
    // thread per output-row chunk), then hand it back
    const int st_tid = tid - kTConsumers;
    const int c8 = st_tid & 7;
    for (int i = 0; i < n_local * W; ++i) {  // one staged output per column block
      const int b = i & 1;
      mbar_wait(&sm.out_full[b], (i >> 1) & 1);
      const TileCoord tc = sm.out_tc[b];
      const uint32_t* out = sm.out[b];
      uint8_t* qTe = qT + cols * static_cast<int64_t>(tc.o);
      if (16 * c8 < tc.rows_valid) {
#pragma unroll 4
        for (int j = st_tid >> 3; j < kTile; j += 4 * WS) {
          const int phys = c8 ^ ((j >> 4) & 7);
          const uint4 o4 = *reinterpret_cast<const uint4*>(&out[j * 32 + 4 * phys]);
          st_v4(qTe + (static_cast<int64_t>(tc.jb) * kTile + j) * tc.m + tc.ib * kTile + 16 * c8, o4);
        }
      }
      if (st_tid < 8) {
        const uint32_t b4 = static_cast<uint32_t>(tc.pad[0]) * 0x01010101u;
        st_v4(sT + static_cast<int64_t>(tc.rb) * cols + tc.jb * kTile + 16 * st_tid, make_uint4(b4, b4, b4, b4));
      }
      mbar_arrive(&sm.out_empty[b]);
    }
    return;
  }
  if (warp == kProducerWarp) {
    // ---- producer warp (lane 0): tile i of this CTA is t = first + i * stride.  The code tile
    // arrives by TMA -- one 128x128 box, or rows_valid/16 boxes of 16 rows for the partial last
    // block of a segment (no bytes of the next segment are read) -- and its run of row scales by
    // a 1D bulk copy, all on the stage's full barrier; the coordinates go with it.
    if (lane == 0) {
      int st = 0;
      uint32_t phase = 0;
      for (int i = 0; i < n_local; ++i) {
        if (i >= STAGES) mbar_wait_sleep(&sm.empty_bar[st], phase ^ 1u, 32);
        TileCoord c = tile_coord(segt, nsegs, n_jb, first + i * stride);
        c.jb *= W;  // the first of the unit's W column blocks
        sm.tc[st] = c;
        const int r0 = c.o + c.ib * kTile;
        mbar_expect_tx(&sm.full_bar[st], static_cast<uint32_t>(c.rows_valid * W * (kTile + 1)));
        if (c.rows_valid == kTile) {
          tma_load_2d(sm.in[st], &tmap_q, &sm.full_bar[st], c.jb * kTile, r0);
        } else {
          for (int r = 0; r < c.rows_valid; r += 16)
            tma_load_2d(sm.in[st] + r * W * kTile, &tmap_q16, &sm.full_bar[st], c.jb * kTile, r0 + r);
        }
#pragma unroll
        for (int h = 0; h < W; ++h)
          bulk_load_1d(sm.sc[st][h], s + static_cast<int64_t>(c.jb + h) * ld_s + r0, c.rows_valid, &sm.full_bar[st]);
        if (++st == STAGES) {
          st = 0;
          phase ^= 1u;
        }
      }
    }
    return;
  }

  // ---- consumer warps (256 threads) ----------------------------------------------------------
  const int g = tid >> 3;  // row quad 0..31
  const int c = tid & 7;   // 16-byte column chunk 0..7
  int st = 0;
  uint32_t phase = 0;
  for (int i = 0; i < n_local; ++i) {
    mbar_wait(&sm.full_bar[st], phase);
    const TileCoord tc = sm.tc[st];
#pragma unroll 1
    for (int h = 0; h < W; ++h) {
      const int o = i * W + h;  // staged output index
      // ---- block scale max (Algorithm 1: S_max = max_i S_i^row), per warp, no CTA barrier:
      // lane l reads the staged scale bytes of rows 4l..4l+3; rows beyond the segment count as 0
      const uint32_t sw_l = (4 * lane < tc.rows_valid) ? sm.sc[st][h][lane] : 0u;
      const uint32_t mx = max(max(sw_l & 0xFFu, (sw_l >> 8) & 0xFFu), max((sw_l >> 16) & 0xFFu, sw_l >> 24));
      const uint32_t tmax = __reduce_max_sync(0xffffffffu, mx);
      const uint32_t sw = __shfl_sync(0xffffffffu, sw_l, g);  // this thread's rows 4g..4g+3

      // ---- shift rows (rows past rows_valid hold stale bytes: shifted, never stored) ---------
      uint4 v[4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
        v[r] = *reinterpret_cast<const uint4*>(&sm.in[st][(4 * g + r) * (W * kTile) + h * kTile + 16 * c]);
      if (h == W - 1) mbar_arrive(&sm.empty_bar[st]);  // done with the stage (scales, coordinates, codes)
      uint32_t R[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint32_t k = tmax - ((sw >> (8 * r)) & 0xFFu);  // k = T_max - T_row >= 0
        const uint32_t m2 = sm.mult[k < 32u ? k : 32u];
        R[r][0] = shift4(v[r].x, m2);
        R[r][1] = shift4(v[r].y, m2);
        R[r][2] = shift4(v[r].z, m2);
        R[r][3] = shift4(v[r].w, m2);
      }
      // ---- 4x4 byte transposes into the swizzled staging buffer --------------------------------
      const int wpos = 4 * ((g >> 2) ^ c) + (g & 3);  // swizzled word position within an out row
      uint32_t* out = sm.out[o & 1];
      if (o >= 2) mbar_wait(&sm.out_empty[o & 1], ((o >> 1) - 1) & 1);  // drained by the store warps
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
      // hand the buffer (and the block's coordinates) to the store warps
      if (tid == 0) {
        TileCoord ob = tc;
        ob.jb = tc.jb + h;
        ob.pad[0] = static_cast<int32_t>(tmax);
        sm.out_tc[o & 1] = ob;
      }
      __syncwarp();  // (tid 0's out_tc write above, before warp 0's arrivals)
      mbar_arrive(&sm.out_full[o & 1]);
    }
    if (++st == STAGES) {
      st = 0;
      phase ^= 1u;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// host side: tensor map + launch
// ---------------------------------------------------------------------------------------------
template <int S, int O, int B, int WS, int W>
static cudaError_t launch_a2v(const CUtensorMap& map, const CUtensorMap& map16, const uint8_t* s, int64_t ld_s, int64_t rows, int64_t cols,
                              const int32_t* seg_offsets, int32_t num_segs, uint8_t* qT, uint8_t* sT,
                              cudaStream_t stream, int num_sms, int64_t ub_tiles) {
  static KernelSetup setup;
  auto kernel = scaling_aware_transpose_kernel<S, O, B, WS, W>;
  constexpr int kThreads = a2_threads<WS>();
  const size_t smem = a2_smem_bytes<TransposeSmem<S, O, W>>(seg_offsets ? num_segs : 1);
  if (prepare_kernel(setup, kernel, kThreads, a2_smem_bytes<TransposeSmem<S, O, W>>(kMaxSegs), smem) == 0)
    return cudaErrorInvalidValue;
  int occ = 0;  // occupancy at this launch's shared memory (the segment tables vary with num_segs)
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem) != cudaSuccess || occ < 1) occ = 1;
  const int64_t grid = one_wave_grid(occ, num_sms, (ub_tiles + W - 1) / W);
  kernel<<<static_cast<unsigned>(grid), kThreads, smem, stream>>>(
      map, map16, s, ld_s, rows, cols, seg_offsets, num_segs, qT, sT);
  return cudaGetLastError();
}

cudaError_t launch_scaling_aware_transpose(const uint8_t* q, const uint8_t* s, int64_t ld_s, int64_t rows,
                                           int64_t cols, const int32_t* seg_offsets, int32_t num_segs,
                                           uint8_t* qT, uint8_t* sT, cudaStream_t stream, int num_sms) {
  const int64_t ub_tiles = (rows / kTile + (seg_offsets ? num_segs : 1)) * (cols / kTile);
  // Launches with >= 32 blocks per SM (the whole-layer X_perm and A, an EP8 shard's X_perm) stage 2
  // column blocks per unit:
  // one 256-byte x 128-row TMA box, so every input row is read 256 contiguous bytes at a time (half
  // the DRAM page openings of 128-byte tile rows): X_perm 133056x7168 358 -> 313 us, A 99 -> 89 us
  // (profiles/r02_a2_midsize.txt); >= 64 blocks per SM: 1 CTA per SM with 3 units in flight (4 for
  // <= 2048 columns); 32..64: 2 CTAs per SM with 2 (EP8 X_perm 40.8 -> 39.0 us).
  const bool wide = cols % (2 * kTile) == 0 && ub_tiles >= 32LL * num_sms;
  const uint32_t bw = wide ? 2 * kTile : kTile;
  CUtensorMap map, map16;  // (W x 128)-byte x 128-row boxes; 16-row boxes for the partial last block
  if (!encode_2d(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, q, static_cast<uint64_t>(cols), static_cast<uint64_t>(rows),
                 static_cast<uint64_t>(cols), bw, kTile) ||
      !encode_2d(&map16, CU_TENSOR_MAP_DATA_TYPE_UINT8, q, static_cast<uint64_t>(cols), static_cast<uint64_t>(rows),
                 static_cast<uint64_t>(cols), bw, 16))
    return cudaErrorInvalidValue;
  if (wide && ub_tiles < 64LL * num_sms)  // 32..64 blocks per SM (an EP8 shard's X_perm): 2 CTAs/SM
    return launch_a2v<2, 2, 2, 2, 2>(map, map16, s, ld_s, rows, cols, seg_offsets, num_segs, qT, sT, stream, num_sms,
                                     ub_tiles);
  if (wide && cols >= 4096)
    return launch_a2v<3, 2, 1, 4, 2>(map, map16, s, ld_s, rows, cols, seg_offsets, num_segs, qT, sT, stream, num_sms,
                                     ub_tiles);
  if (wide)
    return launch_a2v<4, 2, 1, 4, 2>(map, map16, s, ld_s, rows, cols, seg_offsets, num_segs, qT, sT, stream, num_sms,
                                     ub_tiles);
  // Below that, 128-column units.  Tiles held at once = SMs x CTAs x stages: mid-size launches
  // (~12 tiles per SM) need 3 CTAs per SM to ramp up (profiles/r02_a2_order_window.txt).
  if (ub_tiles >= 64LL * num_sms)
    return launch_a2v<3, 2, 2, 4, 1>(map, map16, s, ld_s, rows, cols, seg_offsets, num_segs, qT, sT, stream, num_sms,
                                     ub_tiles);
  return launch_a2v<2, 2, 3, 2, 1>(map, map16, s, ld_s, rows, cols, seg_offsets, num_segs, qT, sT, stream, num_sms,
                                   ub_tiles);
}

// =============================================================================================
// Naive comparator: dequantize (E4M3 x 2^T -> BF16) -> BF16 transpose per segment ->
// column-wise 1x128 requantization with fresh scales.  Three plain kernels + a segment prefix.
// =============================================================================================
__global__ void seg_prefix_kernel(const int32_t* __restrict__ seg_offsets, int32_t num_segs, int64_t rows,
                                  int32_t* __restrict__ seg_out, int32_t* __restrict__ blk_prefix) {
  __shared__ int32_t so[kMaxSegs + 1];
  __shared__ uint32_t red[kPrefixThreads / 32];
  __shared__ int total;
  const int tid = threadIdx.x;
  const int nsegs = seg_offsets == nullptr ? 1 : num_segs;
  if (seg_offsets == nullptr) {
    if (tid == 0) {
      so[0] = 0;
      so[1] = static_cast<int32_t>(rows);
    }
  } else {
    for (int i = tid; i <= nsegs; i += kPrefixThreads) so[i] = seg_offsets[i];
  }
  __syncthreads();
  int nb[4], tsum = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int e = tid * 4 + i;
    nb[i] = e < nsegs ? (so[e + 1] - so[e] + kTile - 1) / kTile : 0;
    tsum += nb[i];
  }
  int run = block_exclusive_scan<kPrefixThreads>(tsum, red, &total);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int e = tid * 4 + i;
    if (e <= nsegs) {
      blk_prefix[e] = run;
      seg_out[e] = so[e];
    }
    run += nb[i];
  }
}

// K1 dequantize: thread per 2 x 16 codes (two 128-bit loads in flight), the row's 1x128 scale
// byte from the MN-major run; decode exactly (e4m3x2 -> f16x2 -> f32), x 2^T in fp32 (exact), one
// RNE to BF16 (R29); two 128-bit stores per 16 codes.
constexpr int kNaiveU = 2;
__global__ void __launch_bounds__(256) naive_dequant_kernel(const uint8_t* __restrict__ q, const uint8_t* __restrict__ s,
                                                            int64_t ld_s, int64_t rows, int64_t cols,
                                                            __nv_bfloat16* __restrict__ xd) {
  const int64_t cpr = cols / 16;                   // 16-code chunks per row
  const int64_t n16 = rows * cpr;
  const int64_t k0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x) * kNaiveU + threadIdx.x;
  uint4 w[kNaiveU];
  float sc[kNaiveU];
#pragma unroll
  for (int u = 0; u < kNaiveU; ++u) {
    const int64_t k = k0 + u * blockDim.x;
    if (k < n16) {
      const int64_t r = k / cpr, cc = k - r * cpr;
      w[u] = ld_nc_v4(q + k * 16);
      sc[u] = scale_from_byte(__ldg(s + (cc >> 3) * ld_s + r));
    }
  }
#pragma unroll
  for (int u = 0; u < kNaiveU; ++u) {
    const int64_t k = k0 + u * blockDim.x;
    if (k >= n16) continue;
    const uint32_t ws[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
    uint32_t o[8];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      uint32_t lo = cvt_f16x2_from_e4m3x2(ws[t] & 0xFFFFu), hi = cvt_f16x2_from_e4m3x2(ws[t] >> 16);
      const float2 a = __half22float2(*reinterpret_cast<__half2*>(&lo));
      const float2 b = __half22float2(*reinterpret_cast<__half2*>(&hi));
      __nv_bfloat162 pa = __floats2bfloat162_rn(a.x * sc[u], a.y * sc[u]);
      __nv_bfloat162 pb = __floats2bfloat162_rn(b.x * sc[u], b.y * sc[u]);
      o[2 * t] = *reinterpret_cast<uint32_t*>(&pa);
      o[2 * t + 1] = *reinterpret_cast<uint32_t*>(&pb);
    }
    st_v4(xd + k * 16, make_uint4(o[0], o[1], o[2], o[3]));
    st_v4(xd + k * 16 + 8, make_uint4(o[4], o[5], o[6], o[7]));
  }
}

// K2 BF16 transpose per segment, xT_e[j][i] = xd[o + i][j]: CTA tile = one 128-row block of a
// segment x 64 columns (16 KB).  Loads: 128-bit, 8 threads per 128-byte row piece, into shared
// memory with the 16-byte chunks XOR-swizzled by (row / 8) & 7.  Read-out: a thread takes 8 rows x
// one 32-bit word (2 columns), i.e. 8 i-elements of output rows j and j + 1, packs them with PRMT
// and stores one 16-byte chunk to each row.  Lane l of a warp: i-chunk l & 7 (+ 8 * half), word
// 4 * chunk + (l >> 3): the 32 lanes read 32 distinct banks, and 8 lanes write 128 contiguous
// bytes of each of the warp's 8 output rows.
__global__ void __launch_bounds__(256) naive_transpose_bf16_kernel(const __nv_bfloat16* __restrict__ xd, int64_t cols,
                                                                   const int32_t* __restrict__ seg_off,
                                                                   const int32_t* __restrict__ blk_prefix,
                                                                   int32_t nsegs, __nv_bfloat16* __restrict__ xT) {
  __shared__ __align__(16) uint32_t tile[128][32];
  __shared__ int32_t seg_s[3];
  const int tid = threadIdx.x;
  const int n_jt = static_cast<int>(cols / 64);
  const int rb = blockIdx.x / n_jt;
  const int jt = blockIdx.x - rb * n_jt;
  if (rb >= __ldg(blk_prefix + nsegs)) return;  // (the grid is an upper bound)
  if (tid == 0) {
    const int e = find_segment(blk_prefix, nsegs, rb);
    seg_s[0] = seg_off[e];
    seg_s[1] = seg_off[e + 1] - seg_off[e];
    seg_s[2] = rb - blk_prefix[e];
  }
  __syncthreads();
  const int o = seg_s[0], m = seg_s[1], ib = seg_s[2];
  const int valid = min(kTile, m - ib * kTile);
  const uint16_t* src = reinterpret_cast<const uint16_t*>(xd) + (static_cast<int64_t>(o) + ib * kTile) * cols + jt * 64;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int id = tid + 256 * k, i = id >> 3, c = id & 7;
    if (i < valid) {
      const uint4 v = ld_nc_v4(src + static_cast<int64_t>(i) * cols + c * 8);
      *reinterpret_cast<uint4*>(&tile[i][4 * (c ^ ((i >> 3) & 7))]) = v;
    }
  }
  __syncthreads();
  uint16_t* dst = reinterpret_cast<uint16_t*>(xT) + static_cast<int64_t>(cols) * o;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int p = tid + 256 * k, l = p & 31, w = p >> 5;   // w: 0..15
    const int ic = (l & 7) + 8 * (w >> 3);                  // 8-row chunk of the block
    const int jp = 4 * (w & 7) + (l >> 3);                  // 32-bit word = column pair 2jp, 2jp+1
    if (ic * 8 >= valid) continue;
    uint32_t wv[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int i = ic * 8 + r;
      wv[r] = tile[i][4 * ((jp >> 2) ^ ((i >> 3) & 7)) + (jp & 3)];
    }
    uint32_t a[4], b[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      a[t] = __byte_perm(wv[2 * t], wv[2 * t + 1], 0x5410);  // column 2 jp, rows i, i + 1
      b[t] = __byte_perm(wv[2 * t], wv[2 * t + 1], 0x7632);  // column 2 jp + 1
    }
    const int64_t j = static_cast<int64_t>(jt) * 64 + 2 * jp;
    st_v4(dst + j * m + ib * kTile + ic * 8, make_uint4(a[0], a[1], a[2], a[3]));
    st_v4(dst + (j + 1) * m + ib * kTile + ic * 8, make_uint4(b[0], b[1], b[2], b[3]));
  }
}

// K3 column-wise requantization: rows j of xT_e (length m_e), 1x128 tiles along i with a fresh
// scale each (ragged last tile).  A1's structure: 8 lanes per tile row, 16 BF16 per lane; a warp
// takes 8 output rows (lanes 8r..8r+7: rows 8w + r and 8w + r + 4) of one 128-column tile.
__device__ __forceinline__ uint32_t absmax2_bf16(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("max.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__global__ void __launch_bounds__(256) naive_colquant_kernel(const __nv_bfloat16* __restrict__ xT, int64_t cols,
                                                             const int32_t* __restrict__ seg_off,
                                                             const int32_t* __restrict__ blk_prefix, int32_t nsegs,
                                                             uint8_t* __restrict__ qT, uint8_t* __restrict__ sT) {
  const int lane = threadIdx.x & 31;
  const int64_t jg8 = cols / 8;                                  // 8-row groups per block
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t total = static_cast<int64_t>(__ldg(blk_prefix + nsegs)) * jg8;
  if (warp >= total) return;
  const int rb = static_cast<int>(warp / jg8);
  const int64_t j0 = (warp - static_cast<int64_t>(rb) * jg8) * 8 + (lane >> 3);
  const int e = find_segment(blk_prefix, nsegs, rb);
  const int64_t o = __ldg(seg_off + e), m = __ldg(seg_off + e + 1) - o;
  const int ib = rb - __ldg(blk_prefix + e);
  const int valid = static_cast<int>(min64(kTile, m - ib * kTile));
  const int c16 = (lane & 7) * 16;
  const bool ok = c16 < valid;
  uint4 v[2][2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const __nv_bfloat16* p = xT + cols * o + (j0 + 4 * h) * m + ib * kTile + c16;
    v[h][0] = ok ? ld_nc_v4(p) : make_uint4(0, 0, 0, 0);
    v[h][1] = ok ? ld_nc_v4(p + 8) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t w[8] = {v[h][0].x, v[h][0].y, v[h][0].z, v[h][0].w, v[h][1].x, v[h][1].y, v[h][1].z, v[h][1].w};
    const uint32_t mm = absmax2_bf16(absmax2_bf16(absmax2_bf16(w[0], w[1]), absmax2_bf16(w[2], w[3])),
                                     absmax2_bf16(absmax2_bf16(w[4], w[5]), absmax2_bf16(w[6], w[7])));
    uint32_t mag = max(mm & 0x7FFFu, (mm >> 16) & 0x7FFFu);
    mag = max(mag, __shfl_xor_sync(0xffffffffu, mag, 1));
    mag = max(mag, __shfl_xor_sync(0xffffffffu, mag, 2));
    mag = max(mag, __shfl_xor_sync(0xffffffffu, mag, 4));
    const int sb = max(static_cast<int>((mag + 0x1Fu) >> 7) - 8, 0);  // the A1 scale rule (R3)
    const float inv = __uint_as_float(static_cast<uint32_t>(254 - sb) << 23);
    uint32_t c[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t] = cvt_e4m3x2_f32(bf16lo_to_f32(w[t]) * inv, bf16hi_to_f32(w[t]) * inv);
    const int64_t j = j0 + 4 * h;
    if (ok)
      st_v4(qT + cols * o + j * m + ib * kTile + c16,
            make_uint4(c[0] | (c[1] << 16), c[2] | (c[3] << 16), c[4] | (c[5] << 16), c[6] | (c[7] << 16)));
    if ((lane & 7) == 0) sT[static_cast<int64_t>(rb) * cols + j] = static_cast<uint8_t>(sb);
  }
}

size_t naive_workspace_bytes(int64_t rows, int64_t cols, int32_t num_segs) {
  return 256 + 2 * 4 * static_cast<size_t>(num_segs + 1) + 256 + 4 * static_cast<size_t>(rows) * cols;
}

cudaError_t launch_naive_transpose(const uint8_t* q, const uint8_t* s, int64_t ld_s, int64_t rows, int64_t cols,
                                   const int32_t* seg_offsets, int32_t num_segs, uint8_t* qT, uint8_t* sT,
                                   void* ws, cudaStream_t stream, int num_sms) {
  const int nsegs = seg_offsets == nullptr ? 1 : num_segs;
  uint8_t* base = static_cast<uint8_t*>(ws);
  int32_t* seg_out = reinterpret_cast<int32_t*>(base);
  int32_t* blk_prefix = seg_out + (nsegs + 1);
  size_t off = (2 * 4 * static_cast<size_t>(nsegs + 1) + 255) / 256 * 256;
  __nv_bfloat16* xd = reinterpret_cast<__nv_bfloat16*>(base + off);
  __nv_bfloat16* xT = xd + rows * cols;
  seg_prefix_kernel<<<1, kPrefixThreads, 0, stream>>>(seg_offsets, num_segs, rows, seg_out, blk_prefix);
  const int64_t n16 = rows * cols / 16;
  const int64_t g1 = (n16 + 256 * kNaiveU - 1) / (256 * kNaiveU);
  if (g1 > 0)
    naive_dequant_kernel<<<static_cast<unsigned>(g1), 256, 0, stream>>>(q, s, ld_s, rows, cols, xd);
  const int64_t blocks_ub = rows / kTile + nsegs;  // 128-row blocks (upper bound; extra CTAs exit)
  naive_transpose_bf16_kernel<<<static_cast<unsigned>(blocks_ub * (cols / 64)), 256, 0, stream>>>(
      xd, cols, seg_out, blk_prefix, nsegs, xT);
  const int64_t warps = blocks_ub * (cols / 8);
  naive_colquant_kernel<<<static_cast<unsigned>((warps + 7) / 8), 256, 0, stream>>>(xT, cols, seg_out, blk_prefix,
                                                                                      nsegs, qT, sT);
  return cudaGetLastError();
}

}  // namespace fp8flow
