// swiglu_bwd.cu -- NEXT-1: fused SwiGLU backward + 1x128 power-of-two E4M3 quantization.
//
// The activation's gradient sits at the BF16 boundary of the backward pass (the
// nonlinear transformation keeps BF16, everything around it stays FP8).  From the saved fc1 output
// h = [a | b] (BF16) and the upstream gradient dA (BF16, fc2 dgrad output):
//     da = dA * b * silu'(a),  silu'(a) = sig(a) (1 + a (1 - sig(a))),   db = dA * silu(a)
// and dH = [da | db] leaves as row-wise FP8 (1x128 tiles along 2F) for the fc1 dgrad / wgrad GEMMs.
// Reference (oracle orc_swiglu_bwd_quant, reading R31): fp64 evaluation rounded once to fp32, then
// A1's quantization; acceptance as A5: codes within 1 E4M3 ULP on <= 1e-4 of elements, identical
// scale bytes.
//
// Kernel: A5's TMA producer/consumer pipeline with three boxes per stage (a, b, dA: 32 rows x 256
// columns each, 3 stages).  Fast fp32 path with MUFU ex2/rcp; 1 - sig is computed as e*sig (no
// cancellation).  silu' has a root near a = -1.28, so relative error bounds do not exist there:
// every element carries an ABSOLUTE error bound D (derived below), and every decision is checked
// against it -- the tile scale (scale byte of amax' - Dmax and amax' + Dmax must agree, else the
// candidates for the max are recomputed in fp64) and each code (the codes of y' - D and y' + D must
// agree, else the element is recomputed in fp64).  Tile-rows with |a| > 64 or an amax outside
// [2^-60, 2^100] are evaluated entirely in fp64.
#include <cuda.h>

#include "async.cuh"
#include "common.cuh"
#include "kernels.h"

namespace fp8flow {

namespace {

constexpr float kL2E = 1.4426950408889634f;
constexpr int kBwCons = 8;               // consumer warps (4 rows each)
constexpr int kBwRows = 4 * kBwCons;     // rows per TMA tile
constexpr int kBwCols = 256;             // F-columns per TMA tile
constexpr int kBwStages = 3;
constexpr int kBwBox = kBwRows * kBwCols * 2;

struct BwdSmem {
  uint8_t a[kBwStages][kBwBox];
  uint8_t b[kBwStages][kBwBox];
  uint8_t d[kBwStages][kBwBox];
  uint64_t full[kBwStages];
  uint64_t empty[kBwStages];
};

__device__ __forceinline__ float ex2f_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// fp64 reference values (the oracle's definition), rounded once to fp32
__device__ __noinline__ void bwd_exact(float a, float b, float g, float& da, float& db) {
  const double ad = a, bd = b, gd = g;
  const double sig = 1.0 / (1.0 + exp(-ad));
  da = static_cast<float>(gd * bd * (sig * (1.0 + ad * (1.0 - sig))));
  db = static_cast<float>(gd * (ad * sig));
}

// quantization decisions of one half-warp's 1x128 tile row from fp32 values y' with absolute error
// bounds D; exact values (fp64) are recomputed where a decision cannot be certified.
// which: 0 -> da, 1 -> db
template <int WHICH>
__device__ __forceinline__ void quant_tile_row(float (&y)[8], const float (&D)[8], const float (&a)[8],
                                               const float (&b)[8], const float (&g)[8], int half, bool exotic_half,
                                               uint32_t (&c)[4], uint32_t& sb_out) {
  float ymax = 0.0f, dmax = 0.0f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    ymax = fmaxf(ymax, fabsf(y[j]));
    dmax = fmaxf(dmax, D[j]);
  }
  uint32_t mag = halfwarp_max_u32(__float_as_uint(ymax));
  float dm = __uint_as_float(halfwarp_max_u32(__float_as_uint(dmax)));
  // domain: exotic inputs, or amax outside [2^-60, 2^100] -> fp64 for the whole tile-row
  const bool exotic = exotic_half || mag > 0x71800000u || (mag != 0u && mag < 0x21800000u);
  const uint32_t exb = __ballot_sync(0xffffffffu, exotic);
  bool exact = false;
  if (exb != 0u) {
    if ((exb >> (16 * half)) & 0xFFFFu) {
      float m2 = 0.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float da, db;
        bwd_exact(a[j], b[j], g[j], da, db);
        y[j] = WHICH == 0 ? da : db;
        m2 = fmaxf(m2, fabsf(y[j]));
      }
      mag = __float_as_uint(m2);
      exact = true;
    }
    mag = halfwarp_max_u32(mag);
    dm = __uint_as_float(halfwarp_max_u32(exact ? 0u : __float_as_uint(dm)));
  }
  // scale: certified iff amax' - Dmax and amax' + Dmax give the same scale byte
  const float am = __uint_as_float(mag);
  const uint32_t s_lo = scale_byte_from_f32_mag(__float_as_uint(fmaxf(am - dm, 0.0f)));
  const uint32_t s_hi = scale_byte_from_f32_mag(__float_as_uint(am + dm));
  if (__any_sync(0xffffffffu, !exact && s_lo != s_hi)) {
    if (!exact && s_lo != s_hi) {
      const float thr = am - 2.0f * dm;  // elements that can be the true max
      float m2 = 0.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (fabsf(y[j]) + D[j] >= thr) {
          float da, db;
          bwd_exact(a[j], b[j], g[j], da, db);
          y[j] = WHICH == 0 ? da : db;
        }
        m2 = fmaxf(m2, fabsf(y[j]));
      }
      mag = __float_as_uint(m2);
    }
    mag = halfwarp_max_u32(mag);
  }
  const uint32_t sb = scale_byte_from_f32_mag(mag);
  const float inv = inv_scale_from_byte(sb);
  uint32_t need = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float d0 = exact ? 0.0f : D[2 * j], d1 = exact ? 0.0f : D[2 * j + 1];
    const uint32_t lo = cvt_e4m3x2_f32((y[2 * j] - d0) * inv, (y[2 * j + 1] - d1) * inv);
    const uint32_t hi = cvt_e4m3x2_f32((y[2 * j] + d0) * inv, (y[2 * j + 1] + d1) * inv);
    c[j] = exact ? cvt_e4m3x2_f32(y[2 * j] * inv, y[2 * j + 1] * inv) : lo;
    need |= (!exact && lo != hi ? 1u : 0u) << j;
  }
  if (__any_sync(0xffffffffu, need != 0u)) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if ((need >> j) & 1u) {
        float e0, f0, e1, f1;
        bwd_exact(a[2 * j], b[2 * j], g[2 * j], e0, f0);
        bwd_exact(a[2 * j + 1], b[2 * j + 1], g[2 * j + 1], e1, f1);
        c[j] = WHICH == 0 ? cvt_e4m3x2_f32(e0 * inv, e1 * inv) : cvt_e4m3x2_f32(f0 * inv, f1 * inv);
      }
    }
  }
  sb_out = sb;
}

__global__ void __launch_bounds__(32 * (1 + kBwCons), 1)
    swiglu_bwd_quant_kernel(const __grid_constant__ CUtensorMap tmap_h, const __grid_constant__ CUtensorMap tmap_d,
                            int64_t rows_max, const int32_t* __restrict__ rows_dev, int64_t F,
                            uint8_t* __restrict__ q, uint8_t* __restrict__ s, int64_t ld_s) {
  extern __shared__ __align__(1024) uint8_t smem_bw[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_bw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rows = rows_dev != nullptr ? static_cast<int64_t>(*rows_dev) : rows_max;
  const int col_tiles = static_cast<int>((F + kBwCols - 1) / kBwCols);
  const int64_t n_tiles = ((rows + kBwRows - 1) / kBwRows) * col_tiles;
  if (tid == 0) {
    for (int i = 0; i < kBwStages; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], kBwCons);
    }
    mbar_init_fence();
  }
  __syncthreads();

  if (warp == 0) {  // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int st = 0;
      uint32_t parity = 0;
      int64_t n = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++n) {
        if (n >= kBwStages) mbar_wait(&sm.empty[st], parity ^ 1u);
        const int64_t rg = t / col_tiles;
        const int c0 = static_cast<int>(t - rg * col_tiles) * kBwCols;
        const int32_t r0 = static_cast<int32_t>(rg * kBwRows);
        mbar_expect_tx(&sm.full[st], 3 * kBwBox);
        tma_load_2d(sm.a[st], &tmap_h, &sm.full[st], c0, r0);
        tma_load_2d(sm.b[st], &tmap_h, &sm.full[st], static_cast<int32_t>(F) + c0, r0);
        tma_load_2d(sm.d[st], &tmap_d, &sm.full[st], c0, r0);
        if (++st == kBwStages) {
          st = 0;
          parity ^= 1u;
        }
      }
    }
    return;
  }
  // ------------------------------------------------------------------------ consumers
  const int cw = warp - 1;
  const int half = lane >> 4, sub = lane & 15;
  int st = 0;
  uint32_t parity = 0;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const int64_t rg = t / col_tiles;
    const int64_t c0 = (t - rg * col_tiles) * kBwCols;
    const int64_t col = c0 + half * 128 + sub * 8;  // column in [0, F)
    const bool col_ok = col < F;
    const int64_t row0 = rg * kBwRows + 4 * cw;
    const int nrows = static_cast<int>(min64(4, rows - row0));
    mbar_wait(&sm.full[st], parity);
    uint4 va[4], vb[4], vd[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int off = ((4 * cw + i) * kBwCols + half * 128 + sub * 8) * 2;
      va[i] = *reinterpret_cast<const uint4*>(&sm.a[st][off]);
      vb[i] = *reinterpret_cast<const uint4*>(&sm.b[st][off]);
      vd[i] = *reinterpret_cast<const uint4*>(&sm.d[st][off]);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[st]);
    if (++st == kBwStages) {
      st = 0;
      parity ^= 1u;
    }
    uint32_t packed_a = 0, packed_b = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t wa[4] = {va[i].x, va[i].y, va[i].z, va[i].w};
      const uint32_t wb[4] = {vb[i].x, vb[i].y, vb[i].z, vb[i].w};
      const uint32_t wd[4] = {vd[i].x, vd[i].y, vd[i].z, vd[i].w};
      float a[8], b[8], g[8], da[8], db[8], Da[8], Db[8];
      float amax_abs = 0.0f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        a[2 * j] = bf16lo_to_f32(wa[j]);
        a[2 * j + 1] = bf16hi_to_f32(wa[j]);
        b[2 * j] = bf16lo_to_f32(wb[j]);
        b[2 * j + 1] = bf16hi_to_f32(wb[j]);
        g[2 * j] = bf16lo_to_f32(wd[j]);
        g[2 * j + 1] = bf16hi_to_f32(wd[j]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float e = ex2f_approx(-a[j] * kL2E);
        const float sig = __fdividef(1.0f, 1.0f + e);
        const float oms = e * sig;  // 1 - sig without cancellation
        const float aom = a[j] * oms;
        const float gg = 1.0f + aom;
        const float dab = g[j] * b[j];  // exact (two 8-bit significands)
        const float daa = g[j] * a[j];  // exact
        da[j] = dab * (sig * gg);
        db[j] = daa * sig;
        // absolute error bounds (|a| <= 64): eps covers the MUFU approximations and the
        // argument rounding of ex2 (~|a| 2^-24), each further operation adds <= 2^-24 relative
        const float eps = (fabsf(a[j]) + 6.0f) * 1.1920928955078125e-07f;  // (|a| + 6) 2^-23
        Da[j] = 4.0f * eps * fabsf(dab) * sig * (fabsf(aom) + fabsf(gg) + 1.0f);
        Db[j] = 4.0f * eps * fabsf(db[j]);
        amax_abs = fmaxf(amax_abs, fabsf(a[j]));
      }
      const bool exotic = !(amax_abs <= 64.0f);
      const uint32_t exh = __ballot_sync(0xffffffffu, exotic);
      const bool exotic_half = ((exh >> (16 * half)) & 0xFFFFu) != 0u;
      uint32_t ca[4], cb[4], sba, sbb;
      quant_tile_row<0>(da, Da, a, b, g, half, exotic_half, ca, sba);
      quant_tile_row<1>(db, Db, a, b, g, half, exotic_half, cb, sbb);
      if (i < nrows && col_ok) {
        uint8_t* qrow = q + (row0 + i) * (2 * F);
        st_v2(qrow + col, ca[0] | (ca[1] << 16), ca[2] | (ca[3] << 16));
        st_v2(qrow + F + col, cb[0] | (cb[1] << 16), cb[2] | (cb[3] << 16));
      }
      packed_a |= sba << (8 * i);
      packed_b |= sbb << (8 * i);
    }
    if (sub == 0 && col_ok && nrows > 0) {
      uint8_t* spa = s + (col / 128) * ld_s + row0;
      uint8_t* spb = s + ((F + col) / 128) * ld_s + row0;
      if (nrows == 4) {
        *reinterpret_cast<uint32_t*>(spa) = packed_a;
        *reinterpret_cast<uint32_t*>(spb) = packed_b;
      } else {
        for (int r = 0; r < nrows; ++r) {
          spa[r] = static_cast<uint8_t>(packed_a >> (8 * r));
          spb[r] = static_cast<uint8_t>(packed_b >> (8 * r));
        }
      }
    }
  }
}

typedef CUresult (*PFN_encodeTiled_bw)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

cudaError_t launch_swiglu_bwd_quant(const void* h, const void* dA, int64_t rows_max, const int32_t* rows_dev,
                                    int64_t ffn, uint8_t* q, uint8_t* s, int64_t ld_s, cudaStream_t stream,
                                    int num_sms) {
  static PFN_encodeTiled_bw encode = nullptr;
  if (!encode) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qres;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qres) != cudaSuccess ||
        qres != cudaDriverEntryPointSuccess)
      return cudaErrorNotSupported;
    encode = reinterpret_cast<PFN_encodeTiled_bw>(p);
    cudaFuncSetAttribute(swiglu_bwd_quant_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(BwdSmem)));
  }
  CUtensorMap mh, md;
  const cuuint32_t box[2] = {kBwCols, kBwRows};
  const cuuint32_t estride[2] = {1, 1};
  const cuuint64_t gdim_h[2] = {static_cast<cuuint64_t>(2 * ffn), static_cast<cuuint64_t>(rows_max)};
  const cuuint64_t gstr_h[1] = {static_cast<cuuint64_t>(4 * ffn)};
  const cuuint64_t gdim_d[2] = {static_cast<cuuint64_t>(ffn), static_cast<cuuint64_t>(rows_max)};
  const cuuint64_t gstr_d[1] = {static_cast<cuuint64_t>(2 * ffn)};
  if (encode(&mh, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(h), gdim_h, gstr_h, box, estride,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
      encode(&md, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(dA), gdim_d, gstr_d, box, estride,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const int64_t tiles_ub = ((rows_max + kBwRows - 1) / kBwRows) * ((ffn + kBwCols - 1) / kBwCols);
  int64_t grid = tiles_ub < num_sms ? tiles_ub : num_sms;
  if (grid < 1) grid = 1;
  swiglu_bwd_quant_kernel<<<static_cast<unsigned>(grid), 32 * (1 + kBwCons), sizeof(BwdSmem), stream>>>(
      mh, md, rows_max, rows_dev, ffn, q, s, ld_s);
  return cudaGetLastError();
}

}  // namespace fp8flow
