// segments.cuh -- device-side segment bookkeeping shared by the transposing kernels (A2 and the
// dual-output kernels): the segment offsets (expert row ranges, device memory) are loaded into
// shared memory and the number of 128-row blocks per segment is prefix-summed, so that a flat
// tile index maps to (segment, row block) without any host synchronisation.
#pragma once

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
template <int NT>
__device__ __forceinline__ void load_segments(int32_t* seg_off, int32_t* blk_prefix, uint32_t* red, int32_t* total_rb,
                                              const int32_t* seg_offsets, int32_t num_segs, int64_t rows) {
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
  for (int i = tid; i <= num_segs; i += NT) seg_off[i] = seg_offsets[i];
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

}  // namespace fp8flow
