// segments.cuh -- device-side segment bookkeeping shared by the transposing kernels (A2 and the
// dual-output kernels): the segment offsets (expert row ranges, device memory) are loaded into
// shared memory and the number of 128-row blocks per segment is prefix-summed, so that a flat
// tile index maps to (segment, row block) without any host synchronisation.
#pragma once

#include <climits>
#include <cstdint>

namespace fp8flow {

// block-wide exclusive scan of one value per thread (blockDim.x == NT); returns the
// exclusive prefix and writes the block total to *total (visible after the trailing sync).
template <int NT>
__device__ __forceinline__ int block_exclusive_scan(int v, uint32_t* warp_tmp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int n = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += n;
  }
  if (lane == 31) warp_tmp[warp] = static_cast<uint32_t>(incl);
  __syncthreads();
  int base = 0, all = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) {
    int t = static_cast<int>(warp_tmp[w]);
    base += (w < warp) ? t : 0;
    all += t;
  }
  if (threadIdx.x == 0) *total = all;
  __syncthreads();
  return base + incl - v;
}

// Loads the segment offsets into seg_off[0..num_segs] and builds blk_prefix[e] = sum_{e'<e}
// ceil(m_e'/128) in shared memory; *total_rb = blk_prefix[num_segs].  NT * 4 > num_segs.
// clamp: every offset is first clamped to it (an overflowed permute plan reports its true padded
// total past the buffer's capacity; its consumers see the rows that exist).
template <int NT>
__device__ __forceinline__ void load_segments(int32_t* seg_off, int32_t* blk_prefix, uint32_t* red, int32_t* total_rb,
                                              const int32_t* seg_offsets, int32_t num_segs, int64_t rows,
                                              int32_t clamp = INT32_MAX) {
  const int tid = threadIdx.x;
  if (seg_offsets == nullptr) {  // one segment: no scan, one barrier
    if (tid == 0) {
      const int32_t nb = static_cast<int32_t>((rows + kTile - 1) / kTile);
      seg_off[0] = 0;
      seg_off[1] = static_cast<int32_t>(rows);
      blk_prefix[0] = 0;
      blk_prefix[1] = nb;
      *total_rb = nb;
    }
    __syncthreads();
    return;
  }
  for (int i = tid; i <= num_segs; i += NT) seg_off[i] = min(seg_offsets[i], clamp);
  __syncthreads();
  // 4 consecutive segments per thread (num_segs <= 1024)
  int nb[4], tsum = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int e = tid * 4 + i;
    nb[i] = e < num_segs ? (seg_off[e + 1] - seg_off[e] + kTile - 1) / kTile : 0;
    tsum += nb[i];
  }
  int run = block_exclusive_scan<NT>(tsum, red, total_rb);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int e = tid * 4 + i;
    if (e <= num_segs) blk_prefix[e] = run;
    run += nb[i];
  }
  __syncthreads();
}
template <int NT, typename Smem>
__device__ __forceinline__ void load_segments(Smem& sm, const int32_t* seg_offsets, int32_t num_segs,
                                              int64_t rows) {
  load_segments<NT>(sm.seg_off, sm.blk_prefix, sm.red, &sm.total_rb, seg_offsets, num_segs, rows);
}

// warp-cooperative: the segment owning row block rb = #{e in [1, num_segs) : blk_prefix[e] <= rb}
// (blk_prefix is non-decreasing, blk_prefix[0] = 0; empty segments are skipped automatically)
__device__ __forceinline__ int find_segment_warp(const int32_t* blk_prefix, int num_segs, int rb) {
  const int lane = threadIdx.x & 31;
  int cnt = 0;
  for (int base = 1; base < num_segs; base += 32) {
    const int e = base + lane;
    cnt += __popc(__ballot_sync(0xffffffffu, e < num_segs && blk_prefix[e] <= rb));
  }
  return cnt;
}

// largest e in [0, num_segs) with blk_prefix[e] <= rb  (the segment that owns row block rb)
__device__ __forceinline__ int find_segment(const int32_t* blk_prefix, int num_segs, int rb) {
  int lo = 0, hi = num_segs;  // invariant: blk_prefix[lo] <= rb < blk_prefix[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (blk_prefix[mid] <= rb) lo = mid;
    else hi = mid;
  }
  return lo;
}


// ------------------------------------------------------------------------------------------
// A2's tile walk over 128x128 blocks of segmented rows (used by A2 and the permute dual kernel)
// ------------------------------------------------------------------------------------------
constexpr int kRowGroup = 8;  // row blocks of a segment walked together (tile order)

struct TileCoord {
  int32_t o, m;     // segment row offset and length
  int32_t ib, jb;   // row block inside the segment, column block
  int32_t rb;       // global row-block index of the output scales
  int32_t rows_valid;
  int32_t pad[2];
};


struct SegTables {
  const int32_t* seg_off;
  const int32_t* blk_prefix;
};

// Tile order (segment-major): for each segment e, its row blocks in groups of kRowGroup, and inside
// a group column block jb, then row block ib fastest.  Consecutive tiles -- the ones the persistent
// CTAs hold at the same time -- therefore read whole input rows of up to 1024 rows (contiguous) and
// write, for each output row j, up to 1024 contiguous bytes: at the whole-layer size (256 experts,
// output rows of ~520 bytes spread over 1 GB) a row-block-major order left the L2 evicting 128-byte
// pieces of ~60 MB of scattered output (r02: 0.54 of peak).  Tile t -> (e, ib, jb):
//   e = segment of virtual row block t / n_jb (segment tiles = n_jb * blocks, contiguous in t),
//   t' = t - n_jb * blk_prefix[e], group g = t' / (n_jb * RG), gsz = min(RG, nblk - g * RG),
//   u = t' - g * n_jb * RG, jb = u / gsz, ib = g * RG + u % gsz.
__device__ __forceinline__ TileCoord tile_coord(const SegTables& sm, int nsegs, int n_jb, int t) {
  const int rbv = t / n_jb;
  const int e = find_segment(sm.blk_prefix, nsegs, rbv);
  const int b0 = sm.blk_prefix[e];
  const int nblk = sm.blk_prefix[e + 1] - b0;
  const int tp = t - b0 * n_jb;
  const int g = tp / (n_jb * kRowGroup);
  const int gsz = min(kRowGroup, nblk - g * kRowGroup);
  const int u = tp - g * n_jb * kRowGroup;
  const int jb = u / gsz;
  const int ib = g * kRowGroup + (u - jb * gsz);
  TileCoord c;
  c.o = sm.seg_off[e];
  c.m = sm.seg_off[e + 1] - c.o;
  c.ib = ib;
  c.jb = jb;
  c.rb = b0 + ib;
  c.rows_valid = min(kTile, c.m - ib * kTile);
  return c;
}

// The same walk split into column chunks of `ch` blocks: all segments' tiles of column blocks
// [q*ch, q*ch + ch) before those of the next chunk (the last chunk may be narrower); inside a chunk
// tile_coord's segment-major order over the chunk's columns.  A kernel that gathers its input rows
// (the permute dual kernel) then reads only ch * 128 bytes of each source row per chunk.
__device__ __forceinline__ TileCoord tile_coord_chunked(const SegTables& sm, int nsegs, int n_jb, int total_rb, int ch,
                                                        int t) {
  const int nq = (n_jb + ch - 1) / ch;
  const int per_chunk = total_rb * ch;
  const int q = min(t / per_chunk, nq - 1);
  const int w = min(ch, n_jb - q * ch);
  const int tc = t - q * per_chunk;
  TileCoord c = tile_coord(sm, nsegs, w, tc);
  c.jb += q * ch;
  return c;
}

}  // namespace fp8flow
