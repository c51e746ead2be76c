// Tile-read probe (not product): how fast can 128x128-byte tiles of a row-major u8 matrix be read
// in A2's tile order (groups of 8 row blocks, column block then row block fastest), by
//   tma_read: persistent CTAs, one producer lane issuing one TMA box per tile into a STAGES ring,
//             8 consumer warps reading the stage (4 x LDS.128 per thread, as A2) and releasing it;
//   ldg_read: persistent CTAs of 8 warps, each warp reading 16 rows x 128 B of the tile with
//             coalesced 16-byte loads (4 rows x 128 B per instruction), U tiles in flight.
// Nothing is written unless the xor of everything read equals a magic value.
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(ph) : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint4 ldg16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void tile_of(int t, int n_jb, int n_ib, int& ib, int& jb) {
  const int g = t / (n_jb * 8), gsz = min(8, n_ib - g * 8), u = t - g * n_jb * 8;
  jb = u / gsz;
  ib = g * 8 + (u - jb * gsz);
}

template <int STAGES>
__global__ void __launch_bounds__(288) tma_read(const __grid_constant__ CUtensorMap map, int rows, int cols, uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * 16384);
  uint64_t* empty = full + STAGES;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 256); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int n_jb = cols / 128, n_ib = rows / 128, total = n_jb * n_ib;
  const int n_local = blockIdx.x < total ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (tid >= 256) {
    if (tid == 256) {
      for (int i = 0; i < n_local; ++i) {
        const int st = i % STAGES;
        if (i >= STAGES) mbar_wait(&empty[st], ((i / STAGES) - 1) & 1);
        int ib, jb;
        tile_of(blockIdx.x + i * gridDim.x, n_jb, n_ib, ib, jb);
        mbar_expect_tx(&full[st], 16384);
        tma2d(sm + st * 16384, &map, &full[st], jb * 128, ib * 128);
      }
    }
    return;
  }
  const int g = tid >> 3, c = tid & 7;
  uint32_t acc = 0;
  for (int i = 0; i < n_local; ++i) {
    const int st = i % STAGES;
    mbar_wait(&full[st], (i / STAGES) & 1);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint4 v = *reinterpret_cast<const uint4*>(sm + st * 16384 + (4 * g + r) * 128 + 16 * c);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    mbar_arrive(&empty[st]);
  }
  if (acc == 0x9E3779B9u) out[0] = acc;
}

template <int U>
__global__ void __launch_bounds__(256) ldg_read(const uint8_t* __restrict__ q, int rows, int cols, uint32_t* out) {
  const int n_jb = cols / 128, n_ib = rows / 128, total = n_jb * n_ib;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t acc = 0;
  for (int t0 = blockIdx.x; t0 < total; t0 += U * gridDim.x) {
    uint4 v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u * gridDim.x;
      if (t < total) {
        int ib, jb;
        tile_of(t, n_jb, n_ib, ib, jb);
        const uint8_t* base = q + (static_cast<int64_t>(ib) * 128 + 16 * w + (lane >> 3)) * cols + jb * 128 + 16 * (lane & 7);
#pragma unroll
        for (int k = 0; k < 4; ++k) v[u][k] = ldg16(base + static_cast<int64_t>(4 * k) * cols);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) v[u][k] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc ^= v[u][k].x ^ v[u][k].y ^ v[u][k].z ^ v[u][k].w;
  }
  if (acc == 0x9E3779B9u) out[0] = acc;
}

typedef CUresult (*PFN_enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" int probe_tma_read(const void* q, int rows, int cols, void* out, int stages, int ctas_per_sm, void* stream) {
  static PFN_enc enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &qr);
  }
  CUtensorMap map;
  const cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t gstr[1] = {(cuuint64_t)cols};
  const cuuint32_t box[2] = {128, 128}, es[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(q), gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  const int grid = 148 * ctas_per_sm;
  const size_t smem = stages * 16384 + 256;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
#define L(S)                                                                                  \
  case S:                                                                                     \
    cudaFuncSetAttribute(tma_read<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    tma_read<S><<<grid, 288, smem, s>>>(map, rows, cols, static_cast<uint32_t*>(out));        \
    break;
  switch (stages) { L(1) L(2) L(3) L(4) L(6) L(8) L(12) default: return -2; }
  return static_cast<int>(cudaGetLastError());
}
extern "C" int probe_ldg_read(const void* q, int rows, int cols, void* out, int u, int ctas_per_sm, void* stream) {
  const int grid = 148 * ctas_per_sm;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint8_t* p = static_cast<const uint8_t*>(q);
  uint32_t* o = static_cast<uint32_t*>(out);
  if (u == 1) ldg_read<1><<<grid, 256, 0, s>>>(p, rows, cols, o);
  else if (u == 2) ldg_read<2><<<grid, 256, 0, s>>>(p, rows, cols, o);
  else ldg_read<4><<<grid, 256, 0, s>>>(p, rows, cols, o);
  return static_cast<int>(cudaGetLastError());
}
