// gemm.cu -- NEXT-2: the consumer of the casting-free FP8 path: an sm_100a
// block-scaled FP8 GEMM on the 5th-generation tensor cores, fed directly by the row-wise (A1, A3,
// A5) and column-wise (A2) outputs with their 1x128 UE8M0 scales -- no dequantization, no cast.
//
//     D[m][n] = sum_k  dec(A[m][k]) 2^(TA[k/128][m])  *  dec(B[n][k]) 2^(TB[k/128][n])
//
// A [M][K] and B [N][K] are K-major E4M3 (Fprop: A = X_perm, B = W_e; Wgrad: A, B = the transposed
// operands of A2), scales MN-major like every other op of the library.  Groups (experts) split M:
// rows [o_g, o_g+1) use B_g = B + g*N*K and its scales (one GEMM per local expert).
//
// Why this maps onto tcgen05 without any rescaling: a 1x128 power-of-two scale is a UE8M0 byte, and
// kind::mxf8f6f4.block_scale consumes one UE8M0 byte per 32-element K block -- replicating the
// byte x4 is lossless.  Accumulation is the tensor core's fp32.
//
// Kernel: persistent, one CTA per SM walking 128 x 256 output tiles (row blocks of all groups x
// column tiles), K in steps of 128 through a 4-stage mbarrier ring.  Warp roles:
//   * warp 0: TMEM allocation (512 columns: the 256-column fp32 accumulator + scale factors) and
//     the TMA producer -- per K step the A tile (128 x 128 B) and B tile (256 x 128 B) with
//     128-byte swizzle; every four K steps the scale runs of those steps (TMA boxes of the
//     MN-major scale tensors: 4 x 128 and 4 x 256 bytes) into a 2-slot scale ring.  CTA pairs
//     (clusters of 2) working on the two column tiles of one row block load half of the shared A
//     tile each and multicast it to both;
//   * warp 1: MMA issuer -- one elected lane issues, once per four K steps, tcgen05.cp of the
//     scale-factor chunks (SFA, SFB) into a double-buffered set of TMEM columns, and per K step
//     4 x tcgen05.mma (M128 N256 K32) with sf_id = the step's position in its group; commits each
//     stage (multicast to the pair), each scale slot, and each finished tile;
//   * warp 2: expands each scale slot into the tensor-memory scale-factor layout: byte j of the
//     word of row r is row r's 1x128 scale of K step kb0 + j (32-row x 16-byte chunks that
//     tcgen05.cp.32x128b.warpx4 broadcasts to the four lane quadrants) -- one copy set per four
//     steps instead of one per step (12 % of the tensor pipe's time at one set per step);
//   * warps 3-10: epilogue -- two warps per TMEM lane quadrant (128 columns each) load the whole
//     accumulator with tcgen05.ld, hand the tensor memory back at once (so the next tile's MMAs
//     overlap these stores), convert fp32 -> BF16 (RNE) or keep fp32, and store the group's rows.
#include <cuda.h>
#include <cuda_bf16.h>

#include "async.cuh"
#include "common.cuh"
#include "kernels.h"
#include "segments.cuh"

namespace fp8flow {

namespace {

constexpr int kGM = 128, kGN = 256, kGK = 128;  // CTA tile
constexpr int kGStages = 4;
constexpr int kGThreads = 352;                  // 11 warps
constexpr int kGMaxGroups = 512;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kSfCol = 256;                // scale-factor columns start after the accumulator

struct __align__(1024) GemmStage {
  uint8_t a[kGM * kGK];     // 16 KB, 128B-swizzled by TMA
  uint8_t b[kGN * kGK];     // 32 KB
  uint8_t sa[kGM];          // raw scale bytes of the 128 A rows
  uint8_t sb[kGN];          // raw scale bytes of the 256 B rows
  uint8_t sfa[512];         // tcgen05.cp source: 32 rows x 16 B
  uint8_t sfb[2][512];
};

// Fprop: operand stages carry only A and B; the scales travel on their own ring, four K steps per
// slot: byte j of a scale-factor word is the scale of K step kb0 + j, so one set of tcgen05.cp
// serves four K steps (sf_id = j selects it for all four 32-wide MMAs of step kb0 + j).
struct __align__(1024) FpStage {
  uint8_t a[kGM * kGK];  // 16 KB, 128B-swizzled by TMA
  uint8_t b[kGN * kGK];  // 32 KB
};
constexpr int kSfGroup = 4;  // K steps per scale slot
struct __align__(128) FpSf {
  uint8_t sa[kSfGroup][kGM];  // raw scale runs of 4 K steps (TMA box of the MN-major scale tensor)
  uint8_t sb[kSfGroup][kGN];
  uint8_t sfa[512];           // tcgen05.cp sources: 32 rows x 16 B
  uint8_t sfb[2][512];
};

struct GemmSmem {
  FpStage st[kGStages];
  alignas(1024) uint8_t stg[8][2048];  // BF16 epilogue staging: one 32 x 32 box per epilogue warp
  FpSf sf[2];
  uint64_t full[kGStages];
  uint64_t empty[kGStages];
  uint64_t sffull[2];          // a slot's raw scales landed (TMA)
  uint64_t sfready[2];         // its scale-factor chunks are expanded
  uint64_t sfempty[2];         // the MMAs that read it completed (tcgen05.commit)
  uint64_t tmem_full;          // accumulator complete (tcgen05.commit)
  uint64_t tmem_empty;         // accumulator read out by the 8 epilogue warps
  uint32_t tmem_base;
  uint32_t red[kGThreads / 32];
  int32_t seg_off[kGMaxGroups + 1];
  int32_t blk_prefix[kGMaxGroups + 1];
  int32_t total_rb;
};

// ---- tcgen05 wrappers ------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t cta_mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(cta_mask)
               : "memory");
}
// TMA 2D load multicast to the CTAs of `cta_mask` (same shared-memory offsets and mbarrier in each)
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0, int32_t c1,
                                               uint16_t cta_mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void tc_cp_32x128b_warpx4(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sdesc));
}
__device__ __forceinline__ void tc_mma_mxf8(uint32_t d_taddr, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate, uint32_t sfa_taddr, uint32_t sfb_taddr) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d_taddr),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sfa_taddr), "r"(sfb_taddr));
}
// four 32-column loads in flight, one wait (the epilogue holds the accumulator for less time)
__device__ __forceinline__ void tc_ld_128cols(uint32_t taddr, uint32_t (&v)[4][32]) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[c][0]), "=r"(v[c][1]), "=r"(v[c][2]), "=r"(v[c][3]), "=r"(v[c][4]), "=r"(v[c][5]), "=r"(v[c][6]),
          "=r"(v[c][7]), "=r"(v[c][8]), "=r"(v[c][9]), "=r"(v[c][10]), "=r"(v[c][11]), "=r"(v[c][12]),
          "=r"(v[c][13]), "=r"(v[c][14]), "=r"(v[c][15]), "=r"(v[c][16]), "=r"(v[c][17]), "=r"(v[c][18]),
          "=r"(v[c][19]), "=r"(v[c][20]), "=r"(v[c][21]), "=r"(v[c][22]), "=r"(v[c][23]), "=r"(v[c][24]),
          "=r"(v[c][25]), "=r"(v[c][26]), "=r"(v[c][27]), "=r"(v[c][28]), "=r"(v[c][29]), "=r"(v[c][30]),
          "=r"(v[c][31])
        : "r"(taddr + static_cast<uint32_t>(32 * c)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// shared-memory matrix descriptors (sm_100 "version 1" format)
__device__ __forceinline__ uint64_t desc_kmajor_sw128(const void* p) {
  // K-major, 128-byte swizzle: 8-row core-matrix groups 1024 B apart (SBO), LBO unused (1)
  const uint64_t addr = smem_u32(p);
  return ((addr & 0x3FFFFull) >> 4) | (1ull << 16) | ((1024ull >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t desc_sf_chunk(const void* p) {
  // 32 rows x 16 B, no swizzle: core matrices (8 rows x 16 B) 128 B apart (SBO)
  const uint64_t addr = smem_u32(p);
  return ((addr & 0x3FFFFull) >> 4) | ((128ull >> 4) << 32) | (1ull << 46);
}
// instruction descriptor: kind::mxf8f6f4.block_scale, E4M3 x E4M3, fp32 accumulate, K-major A and
// B, M = 128, N = 256, UE8M0 scales, scale-factor byte `sf_id` of each 32-bit TMEM word
__host__ __device__ constexpr uint32_t idesc_mxf8(uint32_t sf_id) {
  return (sf_id << 4) | (static_cast<uint32_t>(kGN >> 3) << 17) | (1u << 23) | (static_cast<uint32_t>(kGM >> 4) << 24) |
         (sf_id << 29);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// BF16 epilogue of one warp: its 32 accumulator rows (lane = row) x 128 columns (v[c][j] = column
// 32c + j) leave through shared memory as four 32x32 TMA box stores -- full 64-byte row segments
// instead of 32 scattered 16-byte stores per instruction.  NBUF staging buffers of 2 KB (32 rows x
// 64 B); a buffer is rewritten only after the TMA engine has read it.
template <int NBUF>
__device__ __forceinline__ void epilogue_bf16_tma(const CUtensorMap* tmap_d, uint8_t* stage, const uint32_t (&v)[4][32],
                                                  int col0, int row0, int lane, int& pending) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint8_t* buf = stage + (c % NBUF) * 2048;
    if (pending >= NBUF) {
      if (lane == 0) bulk_wait_read<NBUF - 1>();
      __syncwarp();
    }
    uint4* dst = reinterpret_cast<uint4*>(buf + lane * 64);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      dst[j] = make_uint4(pack_bf16x2(__uint_as_float(v[c][8 * j]), __uint_as_float(v[c][8 * j + 1])),
                          pack_bf16x2(__uint_as_float(v[c][8 * j + 2]), __uint_as_float(v[c][8 * j + 3])),
                          pack_bf16x2(__uint_as_float(v[c][8 * j + 4]), __uint_as_float(v[c][8 * j + 5])),
                          pack_bf16x2(__uint_as_float(v[c][8 * j + 6]), __uint_as_float(v[c][8 * j + 7])));
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(tmap_d, buf, col0 + 32 * c, row0);
      bulk_commit();
    }
    pending = pending < NBUF ? pending + 1 : NBUF;
  }
}

// BF16 epilogue of one warp through two 128-byte-swizzled 32 x 64 staging boxes (4 KB each; the
// swizzle keeps the row-per-lane writes bank-conflict free): 128-byte row segments per TMA store.
// Each buffer is rewritten only after the TMA engine has read it.
__device__ __forceinline__ void epilogue_bf16_tma_sw(const CUtensorMap* tmap_d, uint8_t* stage, const uint32_t (&v)[4][32],
                                                     int col0, int row0, int lane, int& pending) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint8_t* buf = stage + h * 4096;
    if (pending >= 2) {
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // 16-byte chunk j = columns 64h + 8j .. +7
      const uint32_t* w = &v[2 * h + (j >> 2)][8 * (j & 3)];
      *reinterpret_cast<uint4*>(buf + lane * 128 + ((j ^ (lane & 7)) * 16)) =
          make_uint4(pack_bf16x2(__uint_as_float(w[0]), __uint_as_float(w[1])),
                     pack_bf16x2(__uint_as_float(w[2]), __uint_as_float(w[3])),
                     pack_bf16x2(__uint_as_float(w[4]), __uint_as_float(w[5])),
                     pack_bf16x2(__uint_as_float(w[6]), __uint_as_float(w[7])));
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(tmap_d, buf, col0 + 64 * h, row0);
      bulk_commit();
    }
    pending = pending < 2 ? pending + 1 : 2;
  }
}

// tile t -> (group, first row, valid rows, first column)
struct GemmTile {
  int g, r0, rows, n0;
};
__device__ __forceinline__ GemmTile gemm_tile(const GemmSmem& sm, int ngroups, int n_nt, int t) {
  const int rb = t / n_nt, nt = t - rb * n_nt;
  const int g = find_segment(sm.blk_prefix, ngroups, rb);
  const int r0 = sm.seg_off[g] + (rb - sm.blk_prefix[g]) * kGM;
  return {g, r0, min(kGM, sm.seg_off[g + 1] - r0), nt * kGN};
}

// the i-th tile of this CTA (-1 when done).  CL = 1: t = blockIdx.x + i * gridDim.x.  CL = 2: the
// two CTAs of a cluster take the two column tiles (2p', 2p'+1) of the same row block, so they share
// the A tile (each loads one half and multicasts it to both).
template <int CL>
__device__ __forceinline__ int cta_tile(int i, int total_rb, int n_nt) {
  if (CL == 1) {
    const int t = static_cast<int>(blockIdx.x) + i * static_cast<int>(gridDim.x);
    return t < total_rb * n_nt ? t : -1;
  }
  const int pairs_per_rb = n_nt / 2;
  const int p = static_cast<int>(blockIdx.x) / 2 + i * static_cast<int>(gridDim.x / 2);
  if (p >= total_rb * pairs_per_rb) return -1;
  const int rb = p / pairs_per_rb;
  return rb * n_nt + 2 * (p - rb * pairs_per_rb) + static_cast<int>(blockIdx.x & 1);
}

template <int CL>
__global__ void __launch_bounds__(kGThreads, 1)
    gemm_blockscaled_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                            const __grid_constant__ CUtensorMap tmap_d, const __grid_constant__ CUtensorMap tmap_sa,
                            const __grid_constant__ CUtensorMap tmap_sb, int64_t M, int64_t N, int64_t K,
                            const int32_t* __restrict__ seg_offsets,
                            int32_t num_groups, void* __restrict__ D, int32_t d_f32) {
  extern __shared__ __align__(1024) uint8_t smem_gemm[];
  // 128-byte-swizzled TMA destinations need 1024-byte alignment: align the base explicitly
  GemmSmem& sm = *reinterpret_cast<GemmSmem*>((reinterpret_cast<uintptr_t>(smem_gemm) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ngroups = seg_offsets == nullptr ? 1 : num_groups;

  if (warp == 0) tmem_alloc(&sm.tmem_base, kTmemCols);
  if (tid == 32) {
    for (int i = 0; i < kGStages; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], CL);  // the MMA commits of every CTA that reads the stage's A tile
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.sffull[i], 1);
      mbar_init(&sm.sfready[i], 32);  // every lane of the scale-expansion warp
      mbar_init(&sm.sfempty[i], 1);
    }
    mbar_init(&sm.tmem_full, 1);
    mbar_init(&sm.tmem_empty, 8 * 32);  // every epilogue thread
    mbar_init_fence();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_b)) : "memory");
  }
  tc_fence_before();
  load_segments<kGThreads>(sm, seg_offsets, ngroups, M);  // ends with a CTA barrier
  if (CL > 1) cluster_sync_all();  // the peer's barriers exist before any multicast targets them
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int n_nt = static_cast<int>(N / kGN);
  const int nk = static_cast<int>(K / kGK);

  if (warp == 0) {  // --------------------------------------------------------- TMA producer
    if (lane == 0) {
      int st = 0, n = 0, ss = 0, ns = 0;
      uint32_t parity = 0, sparity = 0;
      const int half = CL > 1 ? static_cast<int>(cluster_ctarank()) : 0;
      const int kt = static_cast<int>(K / kGK);  // scale rows per group of B
      for (int i = 0, t; (t = cta_tile<CL>(i, sm.total_rb, n_nt)) >= 0; ++i) {
        const GemmTile T = gemm_tile(sm, ngroups, n_nt, t);
        for (int kb = 0; kb < nk; ++kb, ++n) {
          if (kb % kSfGroup == 0) {  // scales of K steps kb .. kb+3 (rows past the end: zero / unused)
            if (ns >= 2) mbar_wait(&sm.sfempty[ss], sparity ^ 1u);
            mbar_expect_tx(&sm.sffull[ss], kSfGroup * (kGM + kGN));
            tma_load_2d(sm.sf[ss].sa, &tmap_sa, &sm.sffull[ss], T.r0, kb);
            tma_load_2d(sm.sf[ss].sb, &tmap_sb, &sm.sffull[ss], T.n0, T.g * kt + kb);
            ++ns;
            if (++ss == 2) {
              ss = 0;
              sparity ^= 1u;
            }
          }
          if (n >= kGStages) mbar_wait(&sm.empty[st], parity ^ 1u);
          FpStage& S = sm.st[st];
          mbar_expect_tx(&sm.full[st], kGM * kGK + kGN * kGK);
          if (CL == 1)
            tma_load_2d(S.a, &tmap_a, &sm.full[st], kb * kGK, T.r0);
          else  // this CTA's half of the shared A tile, into both CTAs of the pair
            tma_load_2d_mc(S.a + half * (kGM / 2) * kGK, &tmap_a, &sm.full[st], kb * kGK, T.r0 + half * (kGM / 2),
                           0x3);
          tma_load_2d(S.b, &tmap_b, &sm.full[st], kb * kGK, static_cast<int32_t>(T.g * N + T.n0));
          if (++st == kGStages) {
            st = 0;
            parity ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {  // ------------------------------------------------------ MMA issue
    int st = 0, ss = 0, ng = 0;
    uint32_t parity = 0, sparity = 0;
    for (int i = 0; cta_tile<CL>(i, sm.total_rb, n_nt) >= 0; ++i) {
      if (i > 0) mbar_wait(&sm.tmem_empty, (i - 1) & 1);  // the previous tile has been read out
      tc_fence_after();
      uint32_t sfa_t = 0, sfb_t = 0;
      for (int kb = 0; kb < nk; ++kb) {
        const int j = kb % kSfGroup;
        if (j == 0) {  // one set of scale-factor copies per four K steps
          mbar_wait(&sm.sfready[ss], sparity);
          tc_fence_after();
          sfa_t = tmem + kSfCol + 16u * (ng & 1);
          sfb_t = sfa_t + 4u;
          if (lane == 0) {
            tc_cp_32x128b_warpx4(sfa_t, desc_sf_chunk(sm.sf[ss].sfa));
            tc_cp_32x128b_warpx4(sfb_t, desc_sf_chunk(sm.sf[ss].sfb[0]));
            tc_cp_32x128b_warpx4(sfb_t + 4u, desc_sf_chunk(sm.sf[ss].sfb[1]));
          }
        }
        mbar_wait(&sm.full[st], parity);
        tc_fence_after();
        if (lane == 0) {
          FpStage& S = sm.st[st];
          const uint64_t adesc = desc_kmajor_sw128(S.a), bdesc = desc_kmajor_sw128(S.b);
#pragma unroll
          for (int k = 0; k < kGK / 32; ++k)  // +32 bytes (one K=32 slice) inside the swizzle atom
            tc_mma_mxf8(tmem, adesc + 2u * k, bdesc + 2u * k, idesc_mxf8(static_cast<uint32_t>(j)),
                        (kb | k) != 0 ? 1u : 0u, sfa_t, sfb_t);
          // the stage is free when these MMAs complete -- in every CTA of the pair, since the
          // peer multicasts its half of A into this stage too
          if (CL == 1) tc_commit(&sm.empty[st]);
          else tc_commit_mc(&sm.empty[st], 0x3);
          if (j == kSfGroup - 1 || kb == nk - 1) tc_commit(&sm.sfempty[ss]);  // the scale slot too
        }
        __syncwarp();
        if (++st == kGStages) {
          st = 0;
          parity ^= 1u;
        }
        if (j == kSfGroup - 1 || kb == nk - 1) {
          ++ng;
          if (++ss == 2) {
            ss = 0;
            sparity ^= 1u;
          }
        }
      }
      if (lane == 0) tc_commit(&sm.tmem_full);
      __syncwarp();
    }
  } else if (warp == 2) {  // --------------------------------------------- scale expansion
    int ss = 0;
    uint32_t sparity = 0;
    for (int i = 0; cta_tile<CL>(i, sm.total_rb, n_nt) >= 0; ++i) {
      for (int kb = 0; kb < nk; kb += kSfGroup) {
        mbar_wait(&sm.sffull[ss], sparity);
        FpSf& S = sm.sf[ss];
        // chunk byte (r % 32) * 16 + (r / 32) * 4 + j = row r's scale for K step kb + j (one
        // 1x128 scale covers the four 32-wide MX blocks of its step: the MMAs of step kb + j all
        // read byte j)
        uint32_t w[4];
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2) {
          const int r = lane + 32 * i2;
          w[i2] = S.sa[0][r] | (S.sa[1][r] << 8) | (S.sa[2][r] << 16) | (static_cast<uint32_t>(S.sa[3][r]) << 24);
        }
        *reinterpret_cast<uint4*>(&S.sfa[lane * 16]) = make_uint4(w[0], w[1], w[2], w[3]);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
          for (int i2 = 0; i2 < 4; ++i2) {
            const int r = 128 * c + lane + 32 * i2;
            w[i2] = S.sb[0][r] | (S.sb[1][r] << 8) | (S.sb[2][r] << 16) | (static_cast<uint32_t>(S.sb[3][r]) << 24);
          }
          *reinterpret_cast<uint4*>(&S.sfb[c][lane * 16]) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        fence_proxy_async_smem();  // generic-proxy writes -> visible to tcgen05.cp (async proxy)
        __syncwarp();
        mbar_arrive(&sm.sfready[ss]);
        if (++ss == 2) {
          ss = 0;
          sparity ^= 1u;
        }
      }
    }
  } else {  // ------------------------------------------------------------------- epilogue
    const int q = warp & 3;           // TMEM lane quadrant this warp may access
    const int half = (warp - 3) >> 2;  // columns [128 half, 128 half + 128)
    int pending = 0;
    for (int i = 0, t; (t = cta_tile<CL>(i, sm.total_rb, n_nt)) >= 0; ++i) {
      const GemmTile T = gemm_tile(sm, ngroups, n_nt, t);
      mbar_wait(&sm.tmem_full, i & 1);
      tc_fence_after();
      uint32_t v[4][32];
      tc_ld_128cols(tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(128 * half), v);
      tc_fence_before();
      __syncwarp();
      mbar_arrive(&sm.tmem_empty);  // the MMAs of the next tile may start
      const int row = 32 * q + lane;
      if (!d_f32 && 32 * q + 32 <= T.rows) {  // all 32 rows of this warp belong to the group
        epilogue_bf16_tma<1>(&tmap_d, sm.stg[warp - 3], v, T.n0 + 128 * half, T.r0 + 32 * q, lane, pending);
      } else if (row < T.rows) {
        const int64_t grow = static_cast<int64_t>(T.r0) + row;
        const int col0 = T.n0 + 128 * half;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (d_f32) {
            float* dp = static_cast<float*>(D) + grow * N + col0 + 32 * c;
#pragma unroll
            for (int j = 0; j < 32; j += 4) st_v4(dp + j, make_uint4(v[c][j], v[c][j + 1], v[c][j + 2], v[c][j + 3]));
          } else {
            __nv_bfloat16* dp = static_cast<__nv_bfloat16*>(D) + grow * N + col0 + 32 * c;
#pragma unroll
            for (int j = 0; j < 32; j += 8)
              st_v4(dp + j, make_uint4(pack_bf16x2(__uint_as_float(v[c][j]), __uint_as_float(v[c][j + 1])),
                                       pack_bf16x2(__uint_as_float(v[c][j + 2]), __uint_as_float(v[c][j + 3])),
                                       pack_bf16x2(__uint_as_float(v[c][j + 4]), __uint_as_float(v[c][j + 5])),
                                       pack_bf16x2(__uint_as_float(v[c][j + 6]), __uint_as_float(v[c][j + 7]))));
          }
        }
      }
    }
  }
  if (warp >= 3 && lane == 0) bulk_wait_all();  // TMA stores of the epilogue
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // no multicast or remote commit may target an exited CTA
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

// =============================================================================================
// Wgrad: groups split K (the tokens of each expert), e.g. dW1_e = dH_e^T X_e.  Both operands are
// A2's column-wise outputs: per segment e a [rows][m_e] K-major matrix at byte offset rows * o_e,
// scales sT rows P_e .. P_e + ceil(m_e/128) - 1 (A2's layout).  The row stride m_e changes per
// group, so no single host-encoded TMA map addresses them: wgrad_maps_kernel writes two maps per
// group into the caller's workspace (a host-encoded template with the base address, the K extent
// m_e and the row stride m_e replaced by tensormap.replace, published by tensormap.cp_fenceproxy),
// and the GEMM's producer acquires a group's maps when it reaches the group.  TMA zero-fills K past
// the segment's last token; a group with no tokens gets D_e = 0.
// CTA pairs (clusters of 2) take the two 128-row halves of a 256-row block of D_e with the same 256
// columns: each loads its own A rows and half of the shared B tile, multicast into both (per SM a
// K step issues 32 KB of loads instead of 48 KB; the stage is released by both CTAs' MMA commits).
// An odd last 128-row block is paired with zero-filled rows past Ma that are not stored.
// Warps: 0 TMEM + TMA producer, 1 MMA issuer, 2 scale expansion, 3-10 epilogue (BF16 through
// 128-byte-swizzled 32 x 64 staging boxes).  At ~500 tokens per expert the operand loads bound
// it (the L2 -> SM traffic of re-reading each operand tile once per output tile); r01/r02 loaded
// them with 64 threads of 16-byte cp.async (1.25 ms at the EP8 shape, now 0.68 ms:
// profiles/r02_gemm_wgrad.txt).
// =============================================================================================
constexpr int kWThreads = 352;

template <int STAGES, int NBUF>
struct WgradSmem {
  GemmStage st[STAGES];
  alignas(1024) uint8_t stg[8][NBUF * 2048];  // BF16 epilogue staging: NBUF 32 x 32 boxes per warp
  uint64_t full[STAGES];     // operand boxes + scale runs landed (TMA transaction bytes)
  uint64_t empty[STAGES];    // the stage's MMAs completed (tcgen05.commit)
  uint64_t sfready[STAGES];  // the stage's scale-factor chunks are expanded
  uint64_t tmem_full;
  uint64_t tmem_empty;
  uint32_t tmem_base;
  uint32_t red[kWThreads / 32];
  int32_t seg_off[kGMaxGroups + 1];
  int32_t blk_prefix[kGMaxGroups + 1];
  int32_t total_rb;
};

// maps[2g] (A operand of group g) and maps[2g + 1] (B operand): one warp per map
__global__ void __launch_bounds__(256) wgrad_maps_kernel(const __grid_constant__ CUtensorMap tmpl_a,
                                                         const __grid_constant__ CUtensorMap tmpl_b,
                                                         const uint8_t* AT, int64_t Ma, const uint8_t* BT, int64_t Nb,
                                                         const int32_t* __restrict__ seg_offsets, int32_t num_groups,
                                                         CUtensorMap* __restrict__ maps) {
  __shared__ alignas(128) CUtensorMap tm[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = static_cast<int>(blockIdx.x) * 8 + warp; i < 2 * num_groups; i += static_cast<int>(gridDim.x) * 8) {
    const int g = i >> 1;
    const bool is_b = (i & 1) != 0;
    const int o = seg_offsets[g], me = seg_offsets[g + 1] - o;
    const uint32_t ext = me > 0 ? static_cast<uint32_t>(me) : 16u;  // an empty group's maps are never used
    const CUtensorMap* src = is_b ? &tmpl_b : &tmpl_a;
    if (lane < 8) reinterpret_cast<uint4*>(&tm[warp])[lane] = reinterpret_cast<const uint4*>(src)[lane];
    __syncwarp();
    if (lane == 0) {
      const uint32_t a = smem_u32(&tm[warp]);
      const uint64_t base = reinterpret_cast<uint64_t>(is_b ? BT + Nb * o : AT + Ma * o);
      asm volatile("tensormap.replace.tile.global_address.shared::cta.b1024.b64 [%0], %1;" ::"r"(a), "l"(base)
                   : "memory");
      asm volatile("tensormap.replace.tile.global_dim.shared::cta.b1024.b32 [%0], 0, %1;" ::"r"(a), "r"(ext)
                   : "memory");
      asm volatile("tensormap.replace.tile.global_stride.shared::cta.b1024.b64 [%0], 0, %1;" ::"r"(a),
                   "l"(static_cast<uint64_t>(ext))
                   : "memory");
    }
    __syncwarp();
    asm volatile(
        "tensormap.cp_fenceproxy.global.shared::cta.tensormap::generic.release.gpu.sync.aligned [%0], [%1], 128;" ::"l"(
            reinterpret_cast<uint64_t>(maps + i)),
        "r"(smem_u32(&tm[warp]))
        : "memory");
    __syncwarp();
  }
}

template <int STAGES, int NBUF>
__global__ void __launch_bounds__(kWThreads, 1)
    gemm_wgrad_kernel(const __grid_constant__ CUtensorMap tmap_d, const CUtensorMap* __restrict__ maps,
                      const uint8_t* __restrict__ saT, int64_t Ma, const uint8_t* __restrict__ sbT, int64_t Nb,
                      const int32_t* __restrict__ seg_offsets, int32_t num_groups, void* __restrict__ D,
                      int32_t d_f32) {
  extern __shared__ __align__(1024) uint8_t smem_wg[];
  using Smem = WgradSmem<STAGES, NBUF>;
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_wg) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (warp == 0) tmem_alloc(&sm.tmem_base, kTmemCols);
  if (tid == 32) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], 2);     // both CTAs' MMA commits (the peer multicasts half of B here)
      mbar_init(&sm.sfready[i], 32);  // every lane of the scale-expansion warp
    }
    mbar_init(&sm.tmem_full, 1);
    mbar_init(&sm.tmem_empty, 8 * 32);  // every epilogue thread
    mbar_init_fence();
  }
  tc_fence_before();
  load_segments<kWThreads>(sm, seg_offsets, num_groups, 0);  // blk_prefix[e] = P_e (scale-tile rows)
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int rank = static_cast<int>(cluster_ctarank());
  const int n_mp = static_cast<int>((Ma / kGM + 1) / 2), n_nt = static_cast<int>(Nb / kGN);
  const int per_group = n_mp * n_nt;
  const int total_tiles = num_groups * per_group;
  const int c0 = static_cast<int>(blockIdx.x) / 2, ncl = static_cast<int>(gridDim.x) / 2;
  auto tile_of = [&](int t, int& e, int& m0, int& n0) {  // m0: this CTA's rows
    e = t / per_group;
    const int r = t - e * per_group;
    m0 = (r / n_nt) * 2 * kGM + kGM * rank;
    n0 = (r % n_nt) * kGN;
  };

  if (warp == 0) {  // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int st = 0, n = 0, cur = -1;
      uint32_t parity = 0;
      for (int t = c0; t < total_tiles; t += ncl) {
        int e, m0, n0;
        tile_of(t, e, m0, n0);
        const int nk = (sm.seg_off[e + 1] - sm.seg_off[e] + kGK - 1) / kGK;
        if (nk == 0) continue;
        const CUtensorMap* ma = maps + 2 * e;
        const CUtensorMap* mb = ma + 1;
        if (e != cur) {  // the group's maps, written by wgrad_maps_kernel (generic proxy)
          asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(ma))
                       : "memory");
          asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(mb))
                       : "memory");
          cur = e;
        }
        for (int kb = 0; kb < nk; ++kb, ++n) {
          if (n >= STAGES) mbar_wait(&sm.empty[st], parity ^ 1u);
          GemmStage& S = sm.st[st];
          mbar_expect_tx(&sm.full[st], kGM * kGK + kGN * kGK + kGM + kGN);
          tma_load_2d(S.a, ma, &sm.full[st], kb * kGK, m0);
          // this CTA's half of the shared B tile, into both CTAs of the pair
          tma_load_2d_mc(S.b + rank * (kGN / 2) * kGK, mb, &sm.full[st], kb * kGK, n0 + (kGN / 2) * rank, 0x3);
          const int64_t srow = sm.blk_prefix[e] + kb;  // this K block's row of sT
          bulk_load_1d(S.sa, saT + srow * Ma + min(static_cast<int64_t>(m0), Ma - kGM), kGM, &sm.full[st]);
          bulk_load_1d(S.sb, sbT + srow * Nb + n0, kGN, &sm.full[st]);
          if (++st == STAGES) {
            st = 0;
            parity ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {  // ------------------------------------------------------ MMA issue
    int st = 0, step = 0;
    uint32_t parity = 0;
    for (int t = c0, i = 0; t < total_tiles; t += ncl, ++i) {
      int e, m0, n0;
      tile_of(t, e, m0, n0);
      const int me = sm.seg_off[e + 1] - sm.seg_off[e];
      const int nk = (me + kGK - 1) / kGK;
      if (i > 0) mbar_wait(&sm.tmem_empty, (i - 1) & 1);
      tc_fence_after();
      for (int kb = 0; kb < nk; ++kb, ++step) {
        mbar_wait(&sm.sfready[st], parity);  // implies full: the expansion warp waited for it
        tc_fence_after();
        if (lane == 0) {
          GemmStage& S = sm.st[st];
          const uint32_t sfa_t = tmem + kSfCol + 16u * (step & 1);
          const uint32_t sfb_t = sfa_t + 4u;
          tc_cp_32x128b_warpx4(sfa_t, desc_sf_chunk(S.sfa));
          tc_cp_32x128b_warpx4(sfb_t, desc_sf_chunk(S.sfb[0]));
          tc_cp_32x128b_warpx4(sfb_t + 4u, desc_sf_chunk(S.sfb[1]));
          const uint64_t adesc = desc_kmajor_sw128(S.a), bdesc = desc_kmajor_sw128(S.b);
          const int kv = me - kb * kGK;
          const int slices = kv >= kGK ? kGK / 32 : (kv + 31) / 32;  // zero-filled past the segment
          for (int k = 0; k < slices; ++k)
            tc_mma_mxf8(tmem, adesc + 2u * k, bdesc + 2u * k, idesc_mxf8(static_cast<uint32_t>(k)),
                        (kb | k) != 0 ? 1u : 0u, sfa_t, sfb_t);
          tc_commit_mc(&sm.empty[st], 0x3);
        }
        __syncwarp();
        if (++st == STAGES) {
          st = 0;
          parity ^= 1u;
        }
      }
      if (lane == 0) tc_commit(&sm.tmem_full);
      __syncwarp();
    }
  } else if (warp == 2) {  // --------------------------------------------- scale expansion
    int st = 0;
    uint32_t parity = 0;
    for (int t = c0; t < total_tiles; t += ncl) {
      int e, m0, n0;
      tile_of(t, e, m0, n0);
      const int nk = (sm.seg_off[e + 1] - sm.seg_off[e] + kGK - 1) / kGK;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&sm.full[st], parity);
        GemmStage& S = sm.st[st];
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = S.sa[lane + 32 * i] * 0x01010101u;
        *reinterpret_cast<uint4*>(&S.sfa[lane * 16]) = make_uint4(w[0], w[1], w[2], w[3]);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
          for (int i = 0; i < 4; ++i) w[i] = S.sb[128 * c + lane + 32 * i] * 0x01010101u;
          *reinterpret_cast<uint4*>(&S.sfb[c][lane * 16]) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        mbar_arrive(&sm.sfready[st]);
        if (++st == STAGES) {
          st = 0;
          parity ^= 1u;
        }
      }
    }
  } else {  // ------------------------------------------------------------------- epilogue
    const int q = warp & 3;
    const int half = (warp - 3) >> 2;
    int pending = 0;
    for (int t = c0, i = 0; t < total_tiles; t += ncl, ++i) {
      int e, m0, n0;
      tile_of(t, e, m0, n0);
      const bool empty_group = sm.seg_off[e + 1] == sm.seg_off[e];
      mbar_wait(&sm.tmem_full, i & 1);
      tc_fence_after();
      uint32_t v[4][32];
      tc_ld_128cols(tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(128 * half), v);
      tc_fence_before();
      __syncwarp();
      mbar_arrive(&sm.tmem_empty);
      if (empty_group) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int j = 0; j < 32; ++j) v[c][j] = 0u;  // no tokens: dW_e = 0
      }
      if (m0 >= Ma) continue;  // the zero-filled half of an odd last row pair
      const int64_t grow = static_cast<int64_t>(e) * Ma + m0 + 32 * q + lane;
      const int col0 = n0 + 128 * half;
      if (!d_f32) {
        epilogue_bf16_tma_sw(&tmap_d, sm.stg[warp - 3], v, col0, static_cast<int>(grow - lane), lane, pending);
        continue;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float* dp = static_cast<float*>(D) + grow * Nb + col0 + 32 * c;
#pragma unroll
        for (int j = 0; j < 32; j += 4) st_v4(dp + j, make_uint4(v[c][j], v[c][j + 1], v[c][j + 2], v[c][j + 3]));
      }
    }
  }
  if (warp >= 3 && lane == 0) bulk_wait_all();  // TMA stores of the epilogue
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

}  // namespace

cudaError_t launch_gemm_blockscaled(const uint8_t* A, const uint8_t* sa, int64_t ld_sa, const uint8_t* B,
                                    const uint8_t* sb, int64_t ld_sb, int64_t M, int64_t N, int64_t K,
                                    const int32_t* seg_offsets, int32_t num_groups, void* D, int32_t d_f32,
                                    cudaStream_t stream, int num_sms) {
  PFN_encodeTiled encode = tensor_map_encoder();
  if (!encode) return cudaErrorNotSupported;
  static KernelSetup setup1, setup2;
  if (prepare_kernel(setup1, gemm_blockscaled_kernel<1>, kGThreads, sizeof(GemmSmem) + 1024, sizeof(GemmSmem) + 1024) ==
          0 ||
      prepare_kernel(setup2, gemm_blockscaled_kernel<2>, kGThreads, sizeof(GemmSmem) + 1024, sizeof(GemmSmem) + 1024) ==
          0)
    return cudaErrorInvalidValue;
  // CTA pairs (clusters of 2) share the A tile of a row block when N has an even number of tiles
  const int cl = (N / kGN) % 2 == 0 ? 2 : 1;
  const int groups = seg_offsets == nullptr ? 1 : num_groups;
  CUtensorMap ma, mb, md;
  {  // BF16 output boxes of 32 rows x 32 columns (unused for fp32 output)
    const cuuint64_t gdim_d[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M > 0 ? M : 1)};
    const cuuint64_t gstr_d[1] = {static_cast<cuuint64_t>(N) * 2};
    const cuuint32_t box_d[2] = {32, 32};
    const cuuint32_t es[2] = {1, 1};
    if (encode(&md, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, gdim_d, gstr_d, box_d, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const cuuint32_t estride[2] = {1, 1};
  const cuuint64_t gdim_a[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M)};
  const cuuint64_t gstr_a[1] = {static_cast<cuuint64_t>(K)};
  const cuuint32_t box_a[2] = {kGK, static_cast<cuuint32_t>(kGM / cl)};  // a pair loads half each
  const cuuint64_t gdim_b[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(N) * groups};
  const cuuint64_t gstr_b[1] = {static_cast<cuuint64_t>(K)};
  const cuuint32_t box_b[2] = {kGK, kGN};
  if (encode(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(A), gdim_a, gstr_a, box_a, estride,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
      encode(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(B), gdim_b, gstr_b, box_b, estride,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  // MN-major scale tensors as 2D maps: sa [K/128][ld_sa], sb [groups * K/128][ld_sb]; boxes of four
  // K steps x 128 (A rows) / 256 (B rows) bytes
  CUtensorMap msa, msb;
  {
    const cuuint64_t gdim_sa[2] = {static_cast<cuuint64_t>(ld_sa), static_cast<cuuint64_t>(K / kGK)};
    const cuuint64_t gstr_sa[1] = {static_cast<cuuint64_t>(ld_sa)};
    const cuuint32_t box_sa[2] = {kGM, kSfGroup};
    const cuuint64_t gdim_sb[2] = {static_cast<cuuint64_t>(ld_sb), static_cast<cuuint64_t>(K / kGK) * groups};
    const cuuint64_t gstr_sb[1] = {static_cast<cuuint64_t>(ld_sb)};
    const cuuint32_t box_sb[2] = {kGN, kSfGroup};
    if (encode(&msa, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(sa), gdim_sa, gstr_sa, box_sa, estride,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        encode(&msb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(sb), gdim_sb, gstr_sb, box_sb, estride,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  // persistent: at most one CTA per SM, tiles walked with a static stride (pairs of tiles for cl = 2)
  const int64_t tiles_ub = (M / kGM + groups) * (N / kGN);
  int64_t grid = tiles_ub < num_sms ? tiles_ub : num_sms;
  if (cl == 1) {
    gemm_blockscaled_kernel<1><<<static_cast<unsigned>(grid), kGThreads, sizeof(GemmSmem) + 1024, stream>>>(
        ma, mb, md, msa, msb, M, N, K, seg_offsets, num_groups, D, d_f32);
    return cudaGetLastError();
  }
  grid = grid / 2 * 2;
  if (grid < 2) grid = 2;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kGThreads);
  cfg.dynamicSmemBytes = sizeof(GemmSmem) + 1024;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_blockscaled_kernel<2>, ma, mb, md, msa, msb, M, N, K, seg_offsets, num_groups,
                            D, d_f32);
}

}  // namespace fp8flow

namespace fp8flow {

cudaError_t launch_gemm_wgrad(const uint8_t* AT, const uint8_t* saT, int64_t Ma, const uint8_t* BT, const uint8_t* sbT,
                              int64_t Nb, const int32_t* seg_offsets, int32_t num_groups, void* D, int32_t d_f32,
                              void* workspace, cudaStream_t stream, int num_sms) {
  constexpr int kStages = 3, kNbuf = 4;
  using Smem = WgradSmem<kStages, kNbuf>;
  static KernelSetup setup;
  if (prepare_kernel(setup, gemm_wgrad_kernel<kStages, kNbuf>, kWThreads, sizeof(Smem) + 1024, sizeof(Smem) + 1024) == 0)
    return cudaErrorInvalidValue;
  PFN_encodeTiled encode = tensor_map_encoder();
  if (!encode) return cudaErrorNotSupported;
  const cuuint32_t es[2] = {1, 1};
  CUtensorMap md, ta, tb;
  const cuuint64_t gdim_d[2] = {static_cast<cuuint64_t>(Nb), static_cast<cuuint64_t>(num_groups) * Ma};
  const cuuint64_t gstr_d[1] = {static_cast<cuuint64_t>(Nb) * 2};
  const cuuint32_t box_d[2] = {64, 32};
  // operand templates: K extent and row stride 128 (replaced per group on the device), 128-byte
  // swizzled K-major boxes of 128 K x 128 rows (A; B: one CTA's half of the 256-row tile)
  const cuuint64_t gdim_a[2] = {128, static_cast<cuuint64_t>(Ma)}, gdim_b[2] = {128, static_cast<cuuint64_t>(Nb)};
  const cuuint64_t gstr_t[1] = {128};
  const cuuint32_t box_a[2] = {kGK, kGM}, box_b[2] = {kGK, kGN / 2};
  if (encode(&md, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, D, gdim_d, gstr_d, box_d, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
          CUDA_SUCCESS ||
      encode(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(AT), gdim_a, gstr_t, box_a, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
      encode(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(BT), gdim_b, gstr_t, box_b, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  CUtensorMap* maps = static_cast<CUtensorMap*>(workspace);
  wgrad_maps_kernel<<<(2 * num_groups + 7) / 8, 256, 0, stream>>>(ta, tb, AT, Ma, BT, Nb, seg_offsets, num_groups,
                                                                  maps);
  const int64_t pairs = static_cast<int64_t>(num_groups) * ((Ma / kGM + 1) / 2) * (Nb / kGN);
  int64_t grid = (pairs < num_sms / 2 ? pairs : num_sms / 2) * 2;
  if (grid < 2) grid = 2;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kWThreads);
  cfg.dynamicSmemBytes = sizeof(Smem) + 1024;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_wgrad_kernel<kStages, kNbuf>, md, static_cast<const CUtensorMap*>(maps), saT,
                            Ma, sbT, Nb, seg_offsets, num_groups, D, d_f32);
}

}  // namespace fp8flow
