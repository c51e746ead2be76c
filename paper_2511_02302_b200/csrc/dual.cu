// dual.cu -- NEXT-1 dual-output fusions: A1 (quantize) or A5 (SwiGLU +
// quantize) emitting, from ONE read of the BF16 input, both the row-wise FP8 tensor (Fprop/Dgrad
// operand) and its scaling-aware transpose (Algorithm 1; the Wgrad operand) per
// segment.  Unfused, the same result costs A1/A5 (write q) followed by A2 (read q back, write qT):
// the fusion removes the re-read of q and one launch per layer.
//
// Semantics = composition (R32): q, s are exactly what the row-wise kernel (A1 / A5)
// produces, and qT, sT are exactly A2 applied to that q, s with the same segments:
//     T_max = max_i T[i][jb];  sT_e[ib][j] = T_max;  qT_e[j][i-o] = shift(q[i][j], T_max - T[i][jb]).
//
// Kernel: one 128-row x 128-column block (inside one segment, partial last block) per tile,
// persistent CTAs walking the flat tile index of A2 (row blocks of all segments x column tiles).
// Three warp roles, pipelined so that the row math of tile i+1 overlaps the transpose of tile i:
//   * warp 24 (one elected lane), TMA producer: each tile's BF16 input (A1: one box; A5: the a- and
//     b-part boxes) arrives as two 64-row half stages in a STAGES-deep mbarrier ring;
//   * warps 0-15, row warps: warp w owns block rows 8w..8w+7, a full warp per 1x128 tile row
//     (lane l: columns 4l..4l+3), redux.sync for the tile amax (A5: the row math of
//     swiglu_math.cuh, identical to the A5 kernel's).  Codes go to global memory (row-wise output)
//     and to a double-buffered 16 KB row-major code tile in shared memory, scale bytes to global
//     and shared memory; the tile's buffer is handed over on an mbarrier (cfull);
//   * warps 16-23, transpose warps (A2's arithmetic): warp w owns 16 complete output rows of the
//     block (block columns 16w..16w+15); lane a reads block rows 4a..4a+3 of that column chunk
//     (the code tile's chunks are XOR-swizzled by row/4 so these reads are conflict-free), shifts
//     them by k = T_max - T_row, transposes 4x4 byte blocks in registers and stores one 32-bit
//     word per output row -- a full 128-byte line per warp store; no staging buffer, no barrier.
#include <cuda.h>

#include "async.cuh"
#include "common.cuh"
#include "kernels.h"
#include "segments.cuh"
#include "swiglu_math.cuh"

namespace fp8flow {

namespace {

constexpr int kDT = 128;              // block edge (rows and columns)
constexpr int kDRowWarps = 16;        // row warps: 8 rows each
constexpr int kDRpw = kDT / kDRowWarps;
constexpr int kDTrWarps = 8;          // transpose warps: 256 threads, A2's (g, c) mapping
constexpr int kDThreads = (kDRowWarps + kDTrWarps + 1) * 32;
constexpr int kDMaxSegs = 1024;
constexpr int kDHalf = kDT / 2;       // rows per input stage: a tile arrives as two half stages
constexpr int kDBox = kDHalf * kDT * 2;  // one BF16 box (64 rows x 128 columns), 16 KB

// OP 0: A1 (x, one box), OP 1: A5 (h, a- and b-part boxes)
template <int OP, int STAGES>
struct DualSmem {
  static constexpr int kParts = OP == 0 ? 1 : 2;
  uint8_t in[STAGES][kParts][kDBox];  // ring of half-tile stages
  uint32_t ctile[2][kDT * kDT / 4];   // codes of the block, row-major with 16-byte chunks XOR-swizzled
                                      // by (row / 4) % 8 (double buffer)
  uint32_t sc[2][kDT / 4];            // row scale bytes of the block
  uint32_t wmax[2][kDRowWarps];       // per row warp: max scale byte of its valid rows
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t cfull[2];                  // code tile b written (16 row-warp arrivals)
  uint64_t cempty[2];                 // code tile b consumed (8 transpose-warp arrivals)
  uint32_t mult[33];                  // f16x2 multiplier 2^-k for k = 0..32
  uint32_t red[kDThreads / 32];       // scan scratch (load_segments)
  int32_t seg_off[kDMaxSegs + 1];
  int32_t blk_prefix[kDMaxSegs + 1];
  int32_t total_rb;
};


template <int OP, int STAGES>
__global__ void __launch_bounds__(kDThreads, 1)
    dual_kernel(const __grid_constant__ CUtensorMap tmap, int64_t rows_max, const int32_t* __restrict__ rows_dev,
                int64_t cols, const int32_t* __restrict__ seg_offsets, int32_t num_segs, uint8_t* __restrict__ q,
                uint8_t* __restrict__ s, int64_t ld_s, uint8_t* __restrict__ qT, uint8_t* __restrict__ sT) {
  // cols = output columns (A1: x's columns; A5: F, h has 2F)
  extern __shared__ __align__(1024) uint8_t smem_dual[];
  using Smem = DualSmem<OP, STAGES>;
  Smem& sm = *reinterpret_cast<Smem*>(smem_dual);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nsegs = seg_offsets == nullptr ? 1 : num_segs;
  const int64_t rows = rows_dev != nullptr ? min64(static_cast<int64_t>(*rows_dev), rows_max) : rows_max;  // clamped: an overflowed plan reports its true total

  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], kDRowWarps / 2);  // the row warps of one half tile
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.cfull[b], kDRowWarps * 32);  // every lane of every row warp
      mbar_init(&sm.cempty[b], kDTrWarps * 32);  // every transpose thread
    }
    mbar_init_fence();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  if (tid <= 32) sm.mult[tid] = shift_multiplier(static_cast<uint32_t>(tid));
  load_segments<kDThreads>(sm, seg_offsets, nsegs, rows);  // ends with a CTA barrier

  const int n_jb = static_cast<int>(cols / kDT);
  const int total_tiles = sm.total_rb * n_jb;
  const int first = blockIdx.x, stride = gridDim.x;

  if (warp == kDRowWarps + kDTrWarps) {  // ------------------------------------- TMA producer
    if (lane == 0) {
      int st = 0, n = 0;
      uint32_t parity = 0;
      for (int t = first; t < total_tiles; t += stride) {
        const int rb = t / n_jb, jb = t - rb * n_jb;
        const int e = find_segment(sm.blk_prefix, nsegs, rb);
        const int r0 = sm.seg_off[e] + (rb - sm.blk_prefix[e]) * kDT;
        for (int hh = 0; hh < 2; ++hh, ++n) {
          if (n >= STAGES) mbar_wait_sleep(&sm.empty[st], parity ^ 1u, 64);
          mbar_expect_tx(&sm.full[st], Smem::kParts * kDBox);
          tma_load_2d(sm.in[st][0], &tmap, &sm.full[st], jb * kDT, r0 + kDHalf * hh);
          if (OP == 1)
            tma_load_2d(sm.in[st][Smem::kParts - 1], &tmap, &sm.full[st], static_cast<int32_t>(cols) + jb * kDT,
                        r0 + kDHalf * hh);
          if (++st == STAGES) {
            st = 0;
            parity ^= 1u;
          }
        }
      }
    }
    return;
  }

  // tile walk shared by the row and transpose roles: (rb, jb) advance incrementally
  const int stride_rb = stride / n_jb, stride_jb = stride % n_jb;
  int rb = first / n_jb, jb = first % n_jb;

  if (warp < kDRowWarps) {  // ------------------------------------------------------ row warps
    const int wr0 = kDRpw * warp;
    const int hr0 = wr0 % kDHalf;  // first row inside the half stage
    int st = 0;
    uint32_t parity = 0;
    for (int t = first, i = 0; t < total_tiles; t += stride, ++i) {
      if (i > 0) {
        jb += stride_jb;
        rb += stride_rb;
        if (jb >= n_jb) {
          jb -= n_jb;
          ++rb;
        }
      }
      const int e = find_segment_warp(sm.blk_prefix, nsegs, rb);
      const int m = sm.seg_off[e + 1] - sm.seg_off[e];
      const int ib = rb - sm.blk_prefix[e];
      const int r0 = sm.seg_off[e] + ib * kDT;
      const int rows_valid = min(kDT, m - ib * kDT);  // multiple of 16: whole warps in or out
      const bool active = wr0 < rows_valid;
      const int b = i & 1;
      int hs = st + wr0 / kDHalf;  // this warp's half-tile stage
      uint32_t hp = parity;
      if (hs >= STAGES) {
        hs -= STAGES;
        hp ^= 1u;
      }
      st += 2;  // a tile = two half stages
      if (st >= STAGES) {
        st -= STAGES;
        parity ^= 1u;
      }
      mbar_wait(&sm.full[hs], hp);
      if (OP == 0) {
        // A1's lane layout (common.cuh a1_quant16): lanes 8k..8k+7 hold rows k and k + 4 of the
        // warp's 8, lane chunk c8 = columns 8c8..8c8+7 and 64+8c8..+7 (conflict-free smem reads)
        const int r_in = lane >> 3, c8 = lane & 7;
        uint4 v[2][2];
        if (active) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint8_t* rp = &sm.in[hs][0][(hr0 + r_in + 4 * h) * kDT * 2];
            v[h][0] = *reinterpret_cast<const uint4*>(rp + 16 * c8);
            v[h][1] = *reinterpret_cast<const uint4*>(rp + 128 + 16 * c8);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[hs]);
        uint32_t cw[2][4], sb[2] = {0u, 0u};
        if (active) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t w8[8] = {v[h][0].x, v[h][0].y, v[h][0].z, v[h][0].w,
                                    v[h][1].x, v[h][1].y, v[h][1].z, v[h][1].w};
            uint32_t c[8];
            sb[h] = a1_quant16(w8, c);
            cw[h][0] = c[0] | (c[1] << 16);
            cw[h][1] = c[2] | (c[3] << 16);
            cw[h][2] = c[4] | (c[5] << 16);
            cw[h][3] = c[6] | (c[7] << 16);
            const int64_t row = r0 + wr0 + r_in + 4 * h;
            uint8_t* qrow = q + row * cols + jb * kDT + 8 * c8;
            st_v2(qrow, cw[h][0], cw[h][1]);
            st_v2(qrow + 64, cw[h][2], cw[h][3]);
            if (c8 == 0) s[static_cast<int64_t>(jb) * ld_s + row] = static_cast<uint8_t>(sb[h]);
          }
        }
        const uint32_t wm = __reduce_max_sync(0xffffffffu, max(sb[0], sb[1]));  // 0 when inactive
        if (i >= 2) mbar_wait(&sm.cempty[b], ((i >> 1) - 1) & 1);  // tile i-2's transpose is done with b
        if (active) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = wr0 + r_in + 4 * h;
            const int swz = (row >> 2) & 7;
            uint32_t* crow = &sm.ctile[b][row * (kDT / 4) + (c8 & 1) * 2];
            *reinterpret_cast<uint2*>(crow + (((c8 >> 1) ^ swz) << 2)) = make_uint2(cw[h][0], cw[h][1]);
            *reinterpret_cast<uint2*>(crow + (((4 + (c8 >> 1)) ^ swz) << 2)) = make_uint2(cw[h][2], cw[h][3]);
            if (c8 == 0) reinterpret_cast<uint8_t*>(sm.sc[b])[row] = static_cast<uint8_t>(sb[h]);
          }
        }
        if (lane == 0) sm.wmax[b][warp] = wm;
        __syncwarp();
        mbar_arrive(&sm.cfull[b]);  // release (per lane): this lane's code-tile writes are visible
        continue;
      }
      uint32_t cw[kDRpw], sbyte = 0;
      if (active) {
        uint2 wa[kDRpw];
#pragma unroll
        for (int r = 0; r < kDRpw; ++r)
          wa[r] = *reinterpret_cast<const uint2*>(&sm.in[hs][0][((hr0 + r) * kDT + 4 * lane) * 2]);
        {
          uint2 wb[kDRpw];
#pragma unroll
          for (int r = 0; r < kDRpw; ++r)
            wb[r] = *reinterpret_cast<const uint2*>(&sm.in[hs][Smem::kParts - 1][((hr0 + r) * kDT + 4 * lane) * 2]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.empty[hs]);
          // two groups of 4 rows (register budget of 800 threads); decisions are per row, so the
          // grouping does not change any result
          uint2 a4[4], b4[4];
          uint32_t c4[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            a4[r] = wa[r];
            b4[r] = wb[r];
          }
          const uint32_t s_lo = swiglu_quant_rows<4>(a4, b4, c4);
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            cw[r] = c4[r];
            a4[r] = wa[4 + r];
            b4[r] = wb[4 + r];
          }
          const uint32_t s_hi = swiglu_quant_rows<4>(a4, b4, c4);
#pragma unroll
          for (int r = 0; r < 4; ++r) cw[4 + r] = c4[r];
          sbyte = (lane & 4) ? s_hi : s_lo;
        }
      } else if (lane == 0) {
        mbar_arrive(&sm.empty[hs]);
      }
      if (active) {
        uint8_t* qrow = q + static_cast<int64_t>(r0 + wr0) * cols + jb * kDT + 4 * lane;
#pragma unroll
        for (int r = 0; r < kDRpw; ++r) *reinterpret_cast<uint32_t*>(qrow + r * cols) = cw[r];
        if (lane < kDRpw) s[static_cast<int64_t>(jb) * ld_s + r0 + wr0 + lane] = static_cast<uint8_t>(sbyte);
      }
      const uint32_t wm = __reduce_max_sync(0xffffffffu, active && lane < kDRpw ? sbyte : 0u);
      if (i >= 2) mbar_wait(&sm.cempty[b], ((i >> 1) - 1) & 1);  // tile i-2's transpose is done with b
      if (active) {
#pragma unroll
        for (int r = 0; r < kDRpw; ++r) {  // word `lane` of row wr0+r: chunk lane/4 lands at (lane/4) ^ ((row/4) % 8)
          const int row = wr0 + r;
          sm.ctile[b][row * (kDT / 4) + ((((lane >> 2) ^ (row >> 2)) & 7) << 2) + (lane & 3)] = cw[r];
        }
        if (lane < kDRpw) reinterpret_cast<uint8_t*>(sm.sc[b])[wr0 + lane] = static_cast<uint8_t>(sbyte);
      }
      if (lane == 0) sm.wmax[b][warp] = wm;
      __syncwarp();
      mbar_arrive(&sm.cfull[b]);  // release (per lane): this lane's code-tile writes are visible
    }
    return;
  }

  // ----------------------------------------------------------------------- transpose warps
  // warp w owns output rows 16w .. 16w+15 of the block (= block columns, chunk w of every code
  // row); lane a holds block rows 4a..4a+3 (conflict-free: the chunk swizzle depends on row / 4),
  // so every output row leaves as one 128-byte line per warp store -- no staging buffer, no barrier
  const int w = warp - kDRowWarps;  // 0..7
  for (int t = first, i = 0; t < total_tiles; t += stride, ++i) {
    if (i > 0) {
      jb += stride_jb;
      rb += stride_rb;
      if (jb >= n_jb) {
        jb -= n_jb;
        ++rb;
      }
    }
    const int e = find_segment_warp(sm.blk_prefix, nsegs, rb);
    const int o = sm.seg_off[e];
    const int m = sm.seg_off[e + 1] - o;
    const int ib = rb - sm.blk_prefix[e];
    const int rows_valid = min(kDT, m - ib * kDT);
    const int b = i & 1;
    mbar_wait(&sm.cfull[b], (i >> 1) & 1);
    uint32_t tmax = 0;
#pragma unroll
    for (int x = 0; x < kDRowWarps; ++x) tmax = max(tmax, sm.wmax[b][x]);
    const uint32_t sw = sm.sc[b][lane];  // scale bytes of rows 4a..4a+3
    const int pchunk = ((w ^ lane) & 7) << 2;  // physical word offset of chunk w in rows 4a..4a+3
    uint32_t R[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint4 v = *reinterpret_cast<const uint4*>(&sm.ctile[b][(4 * lane + r) * (kDT / 4) + pchunk]);
      const uint32_t k = tmax - ((sw >> (8 * r)) & 0xFFu);  // rows outside the segment: never stored
      const uint32_t m2 = sm.mult[k < 32u ? k : 32u];
      R[r][0] = shift4(v.x, m2);
      R[r][1] = shift4(v.y, m2);
      R[r][2] = shift4(v.z, m2);
      R[r][3] = shift4(v.w, m2);
    }
    mbar_arrive(&sm.cempty[b]);  // (per thread) its reads of code tile b, scales and maxima are done
    if (4 * lane < rows_valid) {
      uint8_t* out = qT + cols * static_cast<int64_t>(o) + (static_cast<int64_t>(jb) * kDT + 16 * w) * m + ib * kDT +
                     4 * lane;
#pragma unroll
      for (int qd = 0; qd < 4; ++qd) {
        const uint32_t t0 = __byte_perm(R[0][qd], R[1][qd], 0x5140);
        const uint32_t t1 = __byte_perm(R[0][qd], R[1][qd], 0x7362);
        const uint32_t t2 = __byte_perm(R[2][qd], R[3][qd], 0x5140);
        const uint32_t t3 = __byte_perm(R[2][qd], R[3][qd], 0x7362);
        uint8_t* o4 = out + static_cast<int64_t>(4 * qd) * m;
        *reinterpret_cast<uint32_t*>(o4) = __byte_perm(t0, t2, 0x5410);
        *reinterpret_cast<uint32_t*>(o4 + m) = __byte_perm(t0, t2, 0x7632);
        *reinterpret_cast<uint32_t*>(o4 + 2 * m) = __byte_perm(t1, t3, 0x5410);
        *reinterpret_cast<uint32_t*>(o4 + 3 * m) = __byte_perm(t1, t3, 0x7632);
      }
    }
    if (w == 0 && lane < 8) {
      const uint32_t b4 = tmax * 0x01010101u;
      st_v4(sT + static_cast<int64_t>(rb) * cols + jb * kDT + 16 * lane, make_uint4(b4, b4, b4, b4));
    }
  }
}

template <int OP, int STAGES>
cudaError_t launch_dual(const void* in, int64_t in_cols, int64_t rows_max, const int32_t* rows_dev, int64_t cols,
                        const int32_t* seg_offsets, int32_t num_segs, uint8_t* q, uint8_t* s, int64_t ld_s,
                        uint8_t* qT, uint8_t* sT, cudaStream_t stream, int num_sms) {
  using Smem = DualSmem<OP, STAGES>;
  static KernelSetup setup;
  if (prepare_kernel(setup, dual_kernel<OP, STAGES>, kDThreads, sizeof(Smem), sizeof(Smem)) == 0)
    return cudaErrorInvalidValue;
  CUtensorMap map;
  if (!encode_2d(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, in, static_cast<uint64_t>(in_cols),
                 static_cast<uint64_t>(rows_max), static_cast<uint64_t>(2 * in_cols), kDT, kDHalf))
    return cudaErrorInvalidValue;
  const int64_t ub_tiles = (rows_max / kDT + (seg_offsets ? num_segs : 1)) * (cols / kDT);
  int64_t grid = ub_tiles < num_sms ? ub_tiles : num_sms;
  if (grid < 1) grid = 1;
  dual_kernel<OP, STAGES><<<static_cast<unsigned>(grid), kDThreads, sizeof(Smem), stream>>>(
      map, rows_max, rows_dev, cols, seg_offsets, num_segs, q, s, ld_s, qT, sT);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_quantize_dual(const void* x, int64_t rows, int64_t cols, const int32_t* seg_offsets,
                                 int32_t num_segs, uint8_t* q, uint8_t* s, int64_t ld_s, uint8_t* qT, uint8_t* sT,
                                 cudaStream_t stream, int num_sms) {
  return launch_dual<0, 10>(x, cols, rows, nullptr, cols, seg_offsets, num_segs, q, s, ld_s, qT, sT, stream, num_sms);
}

cudaError_t launch_swiglu_quant_dual(const void* h, int64_t rows_max, const int32_t* rows_dev, int64_t ffn,
                                     const int32_t* seg_offsets, int32_t num_segs, uint8_t* q, uint8_t* s,
                                     int64_t ld_s, uint8_t* qT, uint8_t* sT, cudaStream_t stream, int num_sms) {
  return launch_dual<1, 5>(h, 2 * ffn, rows_max, rows_dev, ffn, seg_offsets, num_segs, q, s, ld_s, qT, sT, stream,
                           num_sms);
}

}  // namespace fp8flow
