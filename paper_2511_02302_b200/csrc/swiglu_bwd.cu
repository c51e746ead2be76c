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
// Kernel: a TMA producer warp and 16 consumer warps (1 CTA per SM).  A stage holds three boxes
// (a, b, dA: 64 rows x 128 columns each), so one warp-row is exactly one 1x128 scale tile of da and
// one of db: lane l holds columns 4l..4l+3, and every tile maximum is one warp-wide redux.sync
// (no shuffles).  Fast fp32 path with MUFU ex2/rcp; 1 - sig is computed as e*sig (no
// cancellation).  silu' has a root near a = -1.28, so relative error bounds do not exist there:
// the tile maximum carries an ABSOLUTE error bound Dm (derived below) and the scale byte is
// certified when the bytes of amax' - Dm and amax' + Dm agree; otherwise (and for rows with
// |a| > 64, NaN/Inf, or an amax outside [2^-60, 2^100]) the whole warp-row is recomputed in fp64.
// Scale bytes are therefore always the oracle's; codes come from the fp32 values (<= 1 E4M3 ULP,
// the A5 bar).  All decisions are warp-uniform (they depend only on redux results).
#include <cuda.h>

#include "async.cuh"
#include "common.cuh"
#include "kernels.h"

namespace fp8flow {

namespace {

constexpr float kL2E = 1.4426950408889634f;
constexpr int kBwCons = 16;              // consumer warps
constexpr int kBwSub = 4;                // warp-rows (128 columns each) per consumer item
constexpr int kBwHalves = 2;             // 128-column scale tiles per box row
constexpr int kBwRpw = kBwSub / kBwHalves;  // rows per consumer warp and tile
constexpr int kBwRows = kBwRpw * kBwCons;   // rows per TMA tile
constexpr int kBwCols = 128 * kBwHalves;    // F-columns per TMA tile
constexpr int kBwStages = 4;
constexpr int kBwBox = kBwRows * kBwCols * 2;
static_assert(kBwSub == 4, "lanes 0-7 take the 2 x kBwSub tile-row decisions");

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
__device__ __forceinline__ float rcpf_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// max that propagates NaN (a NaN anywhere must reach the domain check)
__device__ __forceinline__ float fmax_nan(float x, float y) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ void unpack4(uint2 w, float (&x)[4]) {
  x[0] = bf16lo_to_f32(w.x);
  x[1] = bf16hi_to_f32(w.x);
  x[2] = bf16lo_to_f32(w.y);
  x[3] = bf16hi_to_f32(w.y);
}

// fp64 reference values (the oracle's definition), rounded once to fp32
__device__ __forceinline__ void bwd_exact(float a, float b, float g, float& da, float& db) {
  const double ad = a, bd = b, gd = g;
  const double sig = 1.0 / (1.0 + exp(-ad));
  da = static_cast<float>(gd * bd * (sig * (1.0 + ad * (1.0 - sig))));
  db = static_cast<float>(gd * (ad * sig));
}

// one warp-row (lane: 4 columns) evaluated exactly; amax ignores NaN like the oracle
// returns {da codes, db codes, da scale byte, db scale byte}
__device__ __noinline__ uint4 row_exact(uint2 wa, uint2 wb, uint2 wg) {
  float a[4], b[4], g[4], ya[4], yb[4];
  unpack4(wa, a);
  unpack4(wb, b);
  unpack4(wg, g);
  float ma = 0.0f, mb = 0.0f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    bwd_exact(a[j], b[j], g[j], ya[j], yb[j]);
    ma = fmaxf(ma, fabsf(ya[j]));
    mb = fmaxf(mb, fabsf(yb[j]));
  }
  const uint32_t sba = scale_byte_from_f32_mag(__reduce_max_sync(0xffffffffu, __float_as_uint(ma)));
  const uint32_t sbb = scale_byte_from_f32_mag(__reduce_max_sync(0xffffffffu, __float_as_uint(mb)));
  const float ia = inv_scale_from_byte(sba), ib = inv_scale_from_byte(sbb);
  return make_uint4(cvt_e4m3x2_f32(ya[0] * ia, ya[1] * ia) | (cvt_e4m3x2_f32(ya[2] * ia, ya[3] * ia) << 16),
                    cvt_e4m3x2_f32(yb[0] * ib, yb[1] * ib) | (cvt_e4m3x2_f32(yb[2] * ib, yb[3] * ib) << 16), sba, sbb);
}

__global__ void __launch_bounds__(32 * (1 + kBwCons), 1)
    swiglu_bwd_quant_kernel(const __grid_constant__ CUtensorMap tmap_h, const __grid_constant__ CUtensorMap tmap_d,
                            int64_t rows_max, const int32_t* __restrict__ rows_dev, int64_t F,
                            uint8_t* __restrict__ q, uint8_t* __restrict__ s, int64_t ld_s, uint32_t sleep_ns) {
  extern __shared__ __align__(1024) uint8_t smem_bw[];
  BwdSmem& sm = *reinterpret_cast<BwdSmem*>(smem_bw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rows = rows_dev != nullptr ? min64(static_cast<int64_t>(*rows_dev), rows_max) : rows_max;  // clamped: an overflowed plan reports its true total
  const int col_tiles = static_cast<int>((F + kBwCols - 1) / kBwCols);
  const int64_t n_rg = (rows + kBwRows - 1) / kBwRows;
  // tile t = (row group rg, column tile ct), t = rg * col_tiles + ct, strided by gridDim.x; the
  // divisions happen once, the walk is incremental
  const int step_c = static_cast<int>(gridDim.x % col_tiles);
  const int64_t step_r = gridDim.x / col_tiles;
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
      int ct = static_cast<int>(blockIdx.x % col_tiles);
      for (int64_t rg = blockIdx.x / col_tiles; rg < n_rg; ++n) {
        if (n >= kBwStages) {
          if (sleep_ns) mbar_wait_sleep(&sm.empty[st], parity ^ 1u, sleep_ns);
          else mbar_wait(&sm.empty[st], parity ^ 1u);
        }
        const int c0 = ct * kBwCols;
        const int32_t r0 = static_cast<int32_t>(rg * kBwRows);
        ct += step_c;
        rg += step_r;
        if (ct >= col_tiles) {
          ct -= col_tiles;
          ++rg;
        }
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
  int st = 0;
  uint32_t parity = 0;
  int ct = static_cast<int>(blockIdx.x % col_tiles);
  for (int64_t rg = blockIdx.x / col_tiles; rg < n_rg;) {
    const int c0 = ct * kBwCols;  // sub-row i: row i / kBwHalves, 128-col tile i % kBwHalves
    const int64_t row0 = rg * kBwRows + kBwRpw * cw;
    const int nrows = static_cast<int>(min64(kBwRpw, rows - row0));
    ct += step_c;
    rg += step_r;
    if (ct >= col_tiles) {
      ct -= col_tiles;
      ++rg;
    }
    mbar_wait(&sm.full[st], parity);
    uint2 wa[kBwSub], wb[kBwSub], wg[kBwSub];
#pragma unroll
    for (int i = 0; i < kBwSub; ++i) {
      const int off = ((kBwRpw * cw + i / kBwHalves) * kBwCols + (i % kBwHalves) * 128 + 4 * lane) * 2;
      wa[i] = *reinterpret_cast<const uint2*>(&sm.a[st][off]);
      wb[i] = *reinterpret_cast<const uint2*>(&sm.b[st][off]);
      wg[i] = *reinterpret_cast<const uint2*>(&sm.d[st][off]);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[st]);
    if (++st == kBwStages) {
      st = 0;
      parity ^= 1u;
    }
    // phase 1: fp32 values (packed f32x2 arithmetic, MUFU scalar) and the four warp maxima of
    // every row (independent across rows)
    float2 da[kBwSub][2], db[kBwSub][2];
    uint32_t mA[kBwSub], mB[kBwSub], mP[kBwSub], mX[kBwSub];
#pragma unroll
    for (int i = 0; i < kBwSub; ++i) {
      const uint32_t aw[2] = {wa[i].x, wa[i].y}, bw[2] = {wb[i].x, wb[i].y}, gw[2] = {wg[i].x, wg[i].y};
      float xa = 0.0f, ya = 0.0f, yb = 0.0f, yp = 0.0f;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const float2 a = make_float2(bf16lo_to_f32(aw[j]), bf16hi_to_f32(aw[j]));
        const float2 b = make_float2(bf16lo_to_f32(bw[j]), bf16hi_to_f32(bw[j]));
        const float2 g = make_float2(bf16lo_to_f32(gw[j]), bf16hi_to_f32(gw[j]));
        const float2 x = __fmul2_rn(a, make_float2(-kL2E, -kL2E));
        const float2 e = make_float2(ex2f_approx(x.x), ex2f_approx(x.y));
        const float2 e1 = __fadd2_rn(e, make_float2(1.0f, 1.0f));
        const float2 sig = make_float2(rcpf_approx(e1.x), rcpf_approx(e1.y));
        const float2 aom = __fmul2_rn(a, __fmul2_rn(e, sig));  // a (1 - sig), no cancellation
        const float2 tt = __fmul2_rn(__fmul2_rn(g, b), sig);   // g b exact (two 8-bit significands)
        const float2 pp = __fmul2_rn(tt, aom);
        da[i][j] = __fadd2_rn(tt, pp);                         // t (1 + a (1 - sig))
        db[i][j] = __fmul2_rn(__fmul2_rn(g, a), sig);
        xa = fmax_nan(xa, fmax_nan(fabsf(a.x), fabsf(a.y)));
        ya = fmax_nan(ya, fmax_nan(fabsf(da[i][j].x), fabsf(da[i][j].y)));
        yb = fmax_nan(yb, fmax_nan(fabsf(db[i][j].x), fabsf(db[i][j].y)));
        yp = fmax_nan(yp, fmax_nan(fabsf(pp.x), fabsf(pp.y)));
      }
      mX[i] = __reduce_max_sync(0xffffffffu, __float_as_uint(xa));
      mA[i] = __reduce_max_sync(0xffffffffu, __float_as_uint(ya));
      mB[i] = __reduce_max_sync(0xffffffffu, __float_as_uint(yb));
      mP[i] = __reduce_max_sync(0xffffffffu, __float_as_uint(yp));
    }
    // phase 2: the item's 8 tile-row decisions (da of rows 0-3, db of rows 0-3) are taken in
    // parallel by lanes 0-7 (lane k: tile-row k), then broadcast.  Error bounds (|a| <= 64): eps
    // covers the MUFU approximations and the argument rounding of ex2 (~|a| 2^-24);
    // with t = g b sig and p = t a (1 - sig): |da - da'| <= 4.25 eps (|t'| + |p'|) and, as
    // |t'| <= |da'| + |p'| (to rounding), the row bound 8.75 eps (max|da'| + 2 max|p'|) holds with
    // a factor-2 margin; |db - db'| <= 4.25 eps |db'| (roundings included).
    const int r = lane & 3;
    const bool is_b = (lane & 4) != 0;
    uint32_t mx = mX[0], mp = mP[0], mm = is_b ? mB[0] : mA[0];
#pragma unroll
    for (int i = 1; i < kBwSub; ++i) {
      if (r == i) {
        mx = mX[i];
        mp = mP[i];
        mm = is_b ? mB[i] : mA[i];
      }
    }
    const float eps = (__uint_as_float(mx) + 6.0f) * 1.1920928955078125e-07f;  // (max|a| + 6) 2^-23
    const float M = __uint_as_float(mm);
    const float dm = is_b ? 4.25f * eps * M : 8.75f * eps * (M + 2.0f * __uint_as_float(mp));
    // domain: |a| <= 64 (no NaN), amax 0 or in [2^-60, 2^100]
    const bool exotic = mx > 0x42800000u || (mm != 0u && mm - 0x21800000u > 0x50000000u);
    // scale byte of a magnitude: exponent field - 8 + [mantissa > 0.75] = ((bits + 0x1FFFFF) >> 23) - 8
    const uint32_t hi = __float_as_uint(M + dm), lo = __float_as_uint(fmaxf(M - dm, 0.0f));
    const uint32_t fh = (hi + 0x1FFFFFu) >> 23;
    const bool sure = !exotic && fh == ((lo + 0x1FFFFFu) >> 23);
    uint32_t sbyte = hi == 0u ? 0u : fh - 8u;
    const float inv = __uint_as_float((254u - sbyte) << 23);
    uint32_t ca[kBwSub], cb[kBwSub];
#pragma unroll
    for (int i = 0; i < kBwSub; ++i) {
      const float ia = __shfl_sync(0xffffffffu, inv, i), ib = __shfl_sync(0xffffffffu, inv, 4 + i);
      const float2 a0 = __fmul2_rn(da[i][0], make_float2(ia, ia)), a1 = __fmul2_rn(da[i][1], make_float2(ia, ia));
      const float2 b0 = __fmul2_rn(db[i][0], make_float2(ib, ib)), b1 = __fmul2_rn(db[i][1], make_float2(ib, ib));
      ca[i] = cvt_e4m3x2_f32(a0.x, a0.y) | (cvt_e4m3x2_f32(a1.x, a1.y) << 16);
      cb[i] = cvt_e4m3x2_f32(b0.x, b0.y) | (cvt_e4m3x2_f32(b1.x, b1.y) << 16);
    }
    const uint32_t unsure = __ballot_sync(0xffffffffu, !sure) & 0xFFu;
    if (unsure != 0u) {  // rare, warp-uniform: recompute whole warp-rows exactly
#pragma unroll
      for (int i = 0; i < kBwSub; ++i) {
        if ((unsure >> i) & 0x11u) {
          const uint4 x = row_exact(wa[i], wb[i], wg[i]);
          ca[i] = x.x;
          cb[i] = x.y;
          if (r == i) sbyte = is_b ? x.w : x.z;
        }
      }
    }
    const bool second_ok = c0 + 128 < F;  // the box's second 128-column tile exists (F % 256 == 128)
    uint8_t* qp = q + row0 * (2 * F) + c0 + 4 * lane;
#pragma unroll
    for (int i = 0; i < kBwSub; ++i) {
      if (i / kBwHalves < nrows && (i % kBwHalves == 0 || second_ok)) {
        uint8_t* p = qp + (i / kBwHalves) * (2 * F) + (i % kBwHalves) * 128;
        *reinterpret_cast<uint32_t*>(p) = ca[i];
        *reinterpret_cast<uint32_t*>(p + F) = cb[i];
      }
    }
    if (lane < 2 * kBwSub && r / kBwHalves < nrows && (r % kBwHalves == 0 || second_ok)) {
      const int tile = (c0 >> 7) + r % kBwHalves + (is_b ? static_cast<int>(F >> 7) : 0);
      s[tile * ld_s + row0 + r / kBwHalves] = static_cast<uint8_t>(sbyte);
    }
  }
}

}  // namespace

cudaError_t launch_swiglu_bwd_quant(const void* h, const void* dA, int64_t rows_max, const int32_t* rows_dev,
                                    int64_t ffn, uint8_t* q, uint8_t* s, int64_t ld_s, cudaStream_t stream,
                                    int num_sms) {
  constexpr uint32_t kSleepNs = 128;  // producer's ring poll interval
  static KernelSetup setup;
  if (prepare_kernel(setup, swiglu_bwd_quant_kernel, 32 * (1 + kBwCons), sizeof(BwdSmem), sizeof(BwdSmem)) == 0)
    return cudaErrorInvalidValue;
  CUtensorMap mh, md;
  if (!encode_2d(&mh, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, h, static_cast<uint64_t>(2 * ffn),
                 static_cast<uint64_t>(rows_max), static_cast<uint64_t>(4 * ffn), kBwCols, kBwRows) ||
      !encode_2d(&md, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, dA, static_cast<uint64_t>(ffn),
                 static_cast<uint64_t>(rows_max), static_cast<uint64_t>(2 * ffn), kBwCols, kBwRows))
    return cudaErrorInvalidValue;
  const int64_t tiles_ub = ((rows_max + kBwRows - 1) / kBwRows) * ((ffn + kBwCols - 1) / kBwCols);
  int64_t grid = tiles_ub < num_sms ? tiles_ub : num_sms;
  if (grid < 1) grid = 1;
  swiglu_bwd_quant_kernel<<<static_cast<unsigned>(grid), 32 * (1 + kBwCons), sizeof(BwdSmem), stream>>>(
      mh, md, rows_max, rows_dev, ffn, q, s, ld_s, kSleepNs);
  return cudaGetLastError();
}

}  // namespace fp8flow
