/*
 * fp8flow_oracle.c -- plain, slow, obviously-correct CPU oracle for the FP8-Flow-MoE hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no source with the CUDA path
 * (paper_2511_02302_b200/csrc) and must never be called by the product path.
 *
 * Citations: "P:n" = line n of the paper's LaTeX source (arXiv 2511.02302, PAPER.md);
 * readings of ambiguous passages are the ones listed in DESIGN.md §3 (numbered R1..R27, the
 * same numbering as SURVEY.md §8(c) "Ambiguities").
 *
 * Style: scalar loops, fp64 arithmetic wherever the paper does not fix a precision, every
 * result computed from its definition (no bit tricks, no blocking, no fusion).  Compiled with
 * -O2 -ffp-contract=off (no FMA contraction, no fast-math) so that every fp32 expression below
 * is evaluated exactly as written.
 *
 * Parity status of each function (pins live in tests/test_oracle_*.py):
 *   orc_decode_e4m3            pinned (torch + ml_dtypes tables, Eq. 10 P:179, 448 max P:143)
 *   orc_encode_e4m3            pinned (torch cast for |v|<=448, round-trip/idempotence/monotone)
 *   orc_scale_exponent         pinned (exact rational brute force over all positive BF16)
 *   orc_shift_e4m3             pinned (torch cast brute force 254 codes x k=0..40, Eq. 11)
 *   orc_quantize_rows_*        pinned (Eqs. 5-8 idempotence, torch cast of x*2^-T, examples)
 *   orc_scaling_aware_transpose pinned (exactness theorem P:186-198, scale alignment, k=0
 *                               identity, T∘T∘T = T, T∘T = id on block-uniform input)
 *   orc_naive_transpose        pinned (constant / block-uniform cases; Eq. 1 demo)
 *   orc_permute_plan/_pad      pinned (worked example, bijection, multiple-of-align sizes)
 *   orc_unpermute              pinned (top_k=1 inverse, convex gates, K·X identity)
 *   orc_swiglu_f32             pinned against torch float64 silu (library routine)
 *   orc_swiglu_quant           partly pinned (H=0, special cases); beyond that the fp64
 *                               definition + tolerance governs -- "parity partly unpinned"
 *   orc_swiglu_bwd_f32         pinned against torch float64 autograd of silu(a)*b (library) and
 *                               central finite differences of the fp64 forward
 *   orc_swiglu_bwd_quant       as orc_swiglu_quant: the fp64 definition + tolerance beyond pins
 *   orc_checksum64             closed form (DESIGN.md §4 C11)
 *   orc_gemm_blockscaled       pinned (torch float64 matmul of torch-decoded operands, one-hot
 *                               rows = scaled B columns, linearity in the scale exponents)
 *   orc_combine                pinned (n = 1 reduces to C9; one-hot gates = the expert row;
 *                               combine(dispatch(Q)) = K * dequant(Q) exactly for any rank count)
 * NEXT-3's dispatch is the composition gather-in-rank-order -> C8 plan -> C8 move (oracle/__init__.py
 * dispatch_permute_pad), pinned by the routing-pair partition over ranks and byte equality of every
 * row with its source token.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------
 * C1  decode(c)  -- Eq. 10: (-1)^SN * 2^(E-7) * (1 + M/8); subnormals at E = 0
 *     (value (-1)^SN * M * 2^-9); E = 15 and M = 7 is NaN; maximum 448.
 * ------------------------------------------------------------------------------------------ */
double orc_decode_e4m3(uint8_t c)
{
    int sn = (c >> 7) & 1;
    int e = (c >> 3) & 15;
    int m = c & 7;
    double sign = sn ? -1.0 : 1.0;
    if (e == 15 && m == 7) return NAN;
    if (e == 0) return sign * ldexp((double)m, -9);              /* 2^-6 * (M/8) */
    return sign * ldexp(1.0 + (double)m / 8.0, e - 7);            /* 2^(E-7)(1+M/8) */
}

/* ------------------------------------------------------------------------------------------
 * C2  encode(v) -- the grid snap of Eq. 3: nearest E4M3 value, ties to even mantissa
 *     (RtN read as round-half-even, R8); finite overflow saturates to +-448 (R9);
 *     the sign is kept, so negative values that round to zero give 0x80 (R10).
 * ------------------------------------------------------------------------------------------ */
uint8_t orc_encode_e4m3(double v)
{
    uint8_t sign = (v < 0.0 || (v == 0.0 && signbit(v))) ? 0x80 : 0x00;
    double a = fabs(v);
    if (isnan(v)) return (uint8_t)(sign | 0x7F);
    if (a > 448.0) a = 448.0;                                   /* satfinite (R9) */

    /* grid spacing at |v|: 2^(e-3) in the normal binade [2^e, 2^(e+1)), 2^-9 below 2^-6 */
    double ulp;
    if (a >= ldexp(1.0, -6)) {
        int ex;
        frexp(a, &ex);                                          /* a = f * 2^ex, f in [0.5,1) */
        ulp = ldexp(1.0, (ex - 1) - 3);
    } else {
        ulp = ldexp(1.0, -9);
    }
    double n = a / ulp;                                         /* exact: power-of-two divide */
    double fl = floor(n);
    double frac = n - fl;
    double r;
    if (frac > 0.5) r = fl + 1.0;
    else if (frac < 0.5) r = fl;
    else r = (fmod(fl, 2.0) == 0.0) ? fl : fl + 1.0;            /* tie -> even */
    double q = r * ulp;                                         /* the chosen grid value */
    if (q > 448.0) q = 448.0;                                   /* a 448 < a' rounding up: clamp */

    /* bits of the chosen value */
    if (q == 0.0) return sign;
    if (q < ldexp(1.0, -6)) {                                   /* subnormal: E = 0, M = q/2^-9 */
        int m = (int)(q / ldexp(1.0, -9));
        return (uint8_t)(sign | m);
    }
    int ex;
    double f = frexp(q, &ex);                                   /* q = f*2^ex, f in [0.5,1) */
    int e = (ex - 1) + 7;                                       /* biased exponent */
    int m = (int)((f * 2.0 - 1.0) * 8.0);                       /* exact: q has 4 sig. bits */
    return (uint8_t)(sign | (e << 3) | m);
}

/* ------------------------------------------------------------------------------------------
 * C3  scale exponent -- Eq. 2 with power-of-two scales s = 2^T:
 *     T = the least integer with amax <= 448 * 2^T (ceil, R3), clamped to [-127, 127] (R13);
 *     amax = 0 gives T = -127 (R11).  Stored as the UE8M0 byte T + 127 (R12).
 * ------------------------------------------------------------------------------------------ */
int orc_scale_exponent(double amax)
{
    if (!(amax > 0.0)) return -127;
    int ex;
    frexp(amax / 448.0, &ex);
    int t = ex;                                                 /* start near log2(amax/448) */
    while (t > -127 && amax <= 448.0 * ldexp(1.0, t - 1)) t--;  /* make t the LEAST such T  */
    while (amax > 448.0 * ldexp(1.0, t)) t++;                   /* ... that still covers amax */
    if (t < -127) t = -127;
    if (t > 127) t = 127;
    return t;
}

/* ------------------------------------------------------------------------------------------
 * C5  shift(c, k) = encode(decode(c) * 2^-k), k >= 0.  The exponent-bit edit E' = E - D of the
 *     derivation after Eq. 11 is this operation whenever no underflow occurs; on
 *     underflow the value is re-rounded into the subnormal grid (R7).  NaN propagates.
 * ------------------------------------------------------------------------------------------ */
uint8_t orc_shift_e4m3(uint8_t c, int k)
{
    double v = orc_decode_e4m3(c);
    if (isnan(v)) return c;
    if (v == 0.0) return c;                                     /* +-0 keeps its sign */
    return orc_encode_e4m3(v * ldexp(1.0, -k));
}

/* BF16 helpers (inputs are BF16 bit patterns; BF16 -> double is exact) */
static double bf16_to_double(uint16_t b)
{
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* round a finite double to the nearest BF16 value, ties to even (also used for fp32 -> BF16).
 * Written from the definition: take the two neighbouring BF16 values and pick the nearer. */
uint16_t orc_round_bf16(double v)
{
    if (isnan(v)) return 0x7FC0;
    float f = (float)v;                        /* callers pass values that are already fp32 */
    uint32_t u;
    memcpy(&u, &f, 4);
    uint32_t lo = u & 0xFFFF0000u;             /* toward zero */
    uint32_t hi = lo + 0x00010000u;            /* away from zero (next BF16 magnitude) */
    float flo, fhi;
    memcpy(&flo, &lo, 4);
    memcpy(&fhi, &hi, 4);
    double dlo = fabs((double)f - (double)flo);
    double dhi = fabs((double)fhi - (double)f);
    uint32_t pick;
    if (dlo < dhi) pick = lo;
    else if (dhi < dlo) pick = hi;
    else pick = ((lo >> 16) & 1) ? hi : lo;    /* tie -> even last mantissa bit */
    return (uint16_t)(pick >> 16);
}

/* ------------------------------------------------------------------------------------------
 * C4  row-wise 1x128 quantization, Eqs. 2-3 with pow2 scales:
 *     per tile of 128 contiguous elements along a row: T = scale(amax), q = encode(x * 2^-T).
 *     Scales are stored MN-major: s[tile][row], ld_s bytes per tile column (ABI layout).
 *     A ragged last tile (cols % 128 != 0) covers the elements present (used by the naive
 *     comparator's column-wise pass over partial 128-row blocks, R14).
 * ------------------------------------------------------------------------------------------ */
static void quantize_row_f64(const double* x, int64_t cols, uint8_t* q, uint8_t* s_col, int64_t ld_s,
                             int64_t row)
{
    for (int64_t t0 = 0, tile = 0; t0 < cols; t0 += 128, tile++) {
        int64_t t1 = t0 + 128 < cols ? t0 + 128 : cols;
        double amax = 0.0;
        for (int64_t j = t0; j < t1; j++)
            if (fabs(x[j]) > amax) amax = fabs(x[j]);
        int t = orc_scale_exponent(amax);
        s_col[tile * ld_s + row] = (uint8_t)(t + 127);
        for (int64_t j = t0; j < t1; j++) q[j] = orc_encode_e4m3(x[j] * ldexp(1.0, -t));
    }
}

void orc_quantize_rows_f64(const double* x, int64_t rows, int64_t cols, uint8_t* q, uint8_t* s,
                           int64_t ld_s)
{
    for (int64_t i = 0; i < rows; i++) quantize_row_f64(x + i * cols, cols, q + i * cols, s, ld_s, i);
}

/* A1 entry quantize: BF16 input (bit patterns) */
void orc_quantize_rowwise_bf16(const uint16_t* x, int64_t rows, int64_t cols, uint8_t* q, uint8_t* s,
                               int64_t ld_s)
{
    double* row = (double*)malloc(sizeof(double) * (size_t)cols);
    for (int64_t i = 0; i < rows; i++) {
        for (int64_t j = 0; j < cols; j++) row[j] = bf16_to_double(x[i * cols + j]);
        quantize_row_f64(row, cols, q + i * cols, s, ld_s, i);
    }
    free(row);
}

/* Eq. 4 dequantize with pow2 scales: x = decode(q) * 2^T  (exact in double) */
void orc_dequantize_rows(const uint8_t* q, const uint8_t* s, int64_t ld_s, int64_t rows, int64_t cols,
                         double* x)
{
    for (int64_t i = 0; i < rows; i++)
        for (int64_t j = 0; j < cols; j++)
            x[i * cols + j] = orc_decode_e4m3(q[i * cols + j]) * ldexp(1.0, (int)s[(j / 128) * ld_s + i] - 127);
}

/* Real-valued-scale variant of Eqs. 2-4 (s = amax/448 exactly as printed), used only
 * for the Eq. 1 double-quantization demonstration (C7).  s_real[tile][row]; amax=0 -> s=1. */
void orc_quantize_rows_real(const double* x, int64_t rows, int64_t cols, uint8_t* q, double* s_real)
{
    int64_t tiles = cols / 128;
    for (int64_t i = 0; i < rows; i++) {
        for (int64_t tile = 0; tile < tiles; tile++) {
            double amax = 0.0;
            for (int64_t j = tile * 128; j < tile * 128 + 128; j++)
                if (fabs(x[i * cols + j]) > amax) amax = fabs(x[i * cols + j]);
            double sc = amax > 0.0 ? amax / 448.0 : 1.0;
            s_real[tile * rows + i] = sc;
            for (int64_t j = tile * 128; j < tile * 128 + 128; j++)
                q[i * cols + j] = orc_encode_e4m3(x[i * cols + j] / sc);
        }
    }
}

/* ------------------------------------------------------------------------------------------
 * C6  Algorithm 1, scaling-aware transpose, as read in R5-R7, R14, R15, R23:
 *     for each segment [o, o+m) and each block (ib, jb) = rows o+128ib .. (partial at the end)
 *     x columns 128jb .. 128jb+127:
 *        T_max = max over the block's rows of T[i][jb]                      (line "S_max = max")
 *        sT[ib][j] = T_max for every j of the block                          (line "S_col = S_max")
 *        qT[j][i-o] = shift(q[i][j], T_max - T[i][jb])   (k = log2(S_max / S_row(i)), E_new = E-k)
 *     Output placement per segment e: qT_e = qT + N*o_e, row stride m_e; sT_e = sT + N*P_e with
 *     P_e = sum_{e'<e} ceil(m_e'/128).  seg_offsets is a HOST array of num_segs+1 entries; NULL
 *     means one segment [0, rows).
 * ------------------------------------------------------------------------------------------ */
void orc_scaling_aware_transpose(const uint8_t* q, const uint8_t* s, int64_t ld_s, int64_t rows,
                                 int64_t cols, const int32_t* seg_offsets, int32_t num_segs,
                                 uint8_t* qT, uint8_t* sT)
{
    int32_t one[2] = {0, (int32_t)rows};
    if (!seg_offsets) { seg_offsets = one; num_segs = 1; }
    int64_t tile_base = 0;
    for (int32_t e = 0; e < num_segs; e++) {
        int64_t o = seg_offsets[e], m = seg_offsets[e + 1] - seg_offsets[e];
        uint8_t* qTe = qT + cols * o;
        uint8_t* sTe = sT + cols * tile_base;
        int64_t nblk = (m + 127) / 128;
        for (int64_t ib = 0; ib < nblk; ib++) {
            int64_t r0 = o + 128 * ib, r1 = r0 + 128 < o + m ? r0 + 128 : o + m;
            for (int64_t jb = 0; jb < cols / 128; jb++) {
                int tmax = -1000;
                for (int64_t i = r0; i < r1; i++) {
                    int t = (int)s[jb * ld_s + i] - 127;
                    if (t > tmax) tmax = t;
                }
                for (int64_t j = jb * 128; j < jb * 128 + 128; j++) {
                    sTe[ib * cols + j] = (uint8_t)(tmax + 127);
                    for (int64_t i = r0; i < r1; i++) {
                        int k = tmax - ((int)s[jb * ld_s + i] - 127);
                        qTe[j * m + (i - o)] = orc_shift_e4m3(q[i * cols + j], k);
                    }
                }
            }
        }
        tile_base += nblk;
    }
}

/* ------------------------------------------------------------------------------------------
 * C7  naive comparator: dequantize -> transpose -> quantize column-wise.
 *     Dequantization lands in BF16 (the dtype the naive path materialises; R-naive in DESIGN.md),
 *     the column-wise pass recomputes a fresh pow2 scale per (column j, 128-row block) of each
 *     segment from the BF16 values.  Same output layout as orc_scaling_aware_transpose.
 * ------------------------------------------------------------------------------------------ */
void orc_naive_transpose(const uint8_t* q, const uint8_t* s, int64_t ld_s, int64_t rows, int64_t cols,
                         const int32_t* seg_offsets, int32_t num_segs, uint8_t* qT, uint8_t* sT)
{
    int32_t one[2] = {0, (int32_t)rows};
    if (!seg_offsets) { seg_offsets = one; num_segs = 1; }
    int64_t tile_base = 0;
    double* col = (double*)malloc(sizeof(double) * (size_t)(rows > 0 ? rows : 1));
    for (int32_t e = 0; e < num_segs; e++) {
        int64_t o = seg_offsets[e], m = seg_offsets[e + 1] - seg_offsets[e];
        uint8_t* qTe = qT + cols * o;
        uint8_t* sTe = sT + cols * tile_base;
        for (int64_t j = 0; j < cols; j++) {
            for (int64_t i = 0; i < m; i++) {
                double v = orc_decode_e4m3(q[(o + i) * cols + j]) *
                           ldexp(1.0, (int)s[(j / 128) * ld_s + (o + i)] - 127);
                col[i] = bf16_to_double(orc_round_bf16(v));   /* D(.) materialised in BF16 */
            }
            /* column j of segment e becomes row j of qT_e; 1x128 tiles along it, MN-major
               scales sT_e[tile][j] (ld = cols) */
            quantize_row_f64(col, m, qTe + j * m, sTe, cols, j);
        }
        tile_base += (m + 127) / 128;
    }
    free(col);
}

/* ------------------------------------------------------------------------------------------
 * C8  permute plan (R16): local experts e in [e0, e0+E_loc);
 *     count_e = #{(t,k): idx[t][k] = e}; padded_e = ceil(count_e/align)*align;
 *     offsets = exclusive prefix sum of padded_e in expert order; inside an expert the rows are
 *     the (t,k) pairs in ascending t, followed by the PAD rows.
 *     row_map[t][k] = output row or -1 (expert not local); src_of_row[r] = t or -1 (PAD / unused
 *     up to max_rows).  Returns 0, or -1 if the padded total exceeds max_rows.
 * ------------------------------------------------------------------------------------------ */
int orc_permute_plan(const int32_t* topk_idx, int64_t T, int32_t K, int32_t e0, int32_t E_loc,
                     int32_t align, int32_t* row_map, int32_t* src_of_row, int64_t max_rows,
                     int32_t* offsets)
{
    offsets[0] = 0;
    for (int32_t le = 0; le < E_loc; le++) {
        int64_t count = 0;
        for (int64_t t = 0; t < T; t++)
            for (int32_t k = 0; k < K; k++)
                if (topk_idx[t * K + k] == e0 + le) count++;
        int64_t padded = (count + align - 1) / align * align;
        offsets[le + 1] = (int32_t)(offsets[le] + padded);
    }
    if (offsets[E_loc] > max_rows) return -1;
    for (int64_t r = 0; r < max_rows; r++) src_of_row[r] = -1;
    for (int64_t t = 0; t < T; t++)
        for (int32_t k = 0; k < K; k++) row_map[t * K + k] = -1;
    for (int32_t le = 0; le < E_loc; le++) {
        int64_t next = offsets[le];
        for (int64_t t = 0; t < T; t++)
            for (int32_t k = 0; k < K; k++)
                if (topk_idx[t * K + k] == e0 + le) {
                    row_map[t * K + k] = (int32_t)next;
                    src_of_row[next] = (int32_t)t;
                    next++;
                }
    }
    return 0;
}

/* C8 move: out[r] = tok[src_of_row[r]] (codes and 1x128 scales), PAD rows = code 0x00 and
 * scale byte 0x00 (R11, R17).  Rows r >= offsets[E_loc] are not written. */
void orc_permute_pad(const uint8_t* q_tok, const uint8_t* s_tok, int64_t ld_s_tok, int64_t T, int64_t H,
                     const int32_t* src_of_row, const int32_t* offsets, int32_t E_loc, int64_t max_rows,
                     uint8_t* q_out, uint8_t* s_out)
{
    (void)T;
    int64_t R = offsets[E_loc];
    for (int64_t r = 0; r < R; r++) {
        int32_t src = src_of_row[r];
        for (int64_t h = 0; h < H; h++) q_out[r * H + h] = src >= 0 ? q_tok[(int64_t)src * H + h] : 0x00;
        for (int64_t tile = 0; tile < H / 128; tile++)
            s_out[tile * max_rows + r] = src >= 0 ? s_tok[tile * ld_s_tok + src] : 0x00;
    }
}

/* ------------------------------------------------------------------------------------------
 * C9  unpermute + unpad (R21, R22): y[t][h] = BF16_RNE( sum over k with
 *     row_map[t][k] >= 0 of p[t][k] * x[row_map[t][k]][h] ), accumulated in fp32 with one
 *     fused multiply-add per term in k order starting from +0.0 (p = 1, plain add, when probs
 *     is NULL).  PAD rows are never read.
 * ------------------------------------------------------------------------------------------ */
void orc_unpermute(const uint16_t* x, int64_t H, const int32_t* row_map, const float* probs, int64_t T,
                   int32_t K, uint16_t* y)
{
    for (int64_t t = 0; t < T; t++) {
        for (int64_t h = 0; h < H; h++) {
            float acc = 0.0f;
            for (int32_t k = 0; k < K; k++) {
                int32_t r = row_map[t * K + k];
                if (r < 0) continue;
                float xv = (float)bf16_to_double(x[(int64_t)r * H + h]);
                if (probs) acc = fmaf(probs[t * K + k], xv, acc);
                else acc = acc + xv;
            }
            y[t * H + h] = orc_round_bf16((double)acc);
        }
    }
}

/* ------------------------------------------------------------------------------------------
 * C10 SwiGLU (R18-R20): a = h[:, :F] (gate), b = h[:, F:];
 *     y = silu(a) * b = a*b / (1 + e^-a), evaluated in double, rounded once to fp32.
 * ------------------------------------------------------------------------------------------ */
void orc_swiglu_f32(const uint16_t* h, int64_t rows, int64_t F, float* y)
{
    for (int64_t i = 0; i < rows; i++)
        for (int64_t j = 0; j < F; j++) {
            double a = bf16_to_double(h[i * 2 * F + j]);
            double b = bf16_to_double(h[i * 2 * F + F + j]);
            y[i * F + j] = (float)(a * b / (1.0 + exp(-a)));
        }
}

/* C10 fused SwiGLU + quantize: C4 applied to the fp32 SwiGLU output (amax over fp32 values). */
void orc_swiglu_quant(const uint16_t* h, int64_t rows, int64_t F, uint8_t* q, uint8_t* s, int64_t ld_s)
{
    float* yf = (float*)malloc(sizeof(float) * (size_t)F);
    double* yd = (double*)malloc(sizeof(double) * (size_t)F);
    for (int64_t i = 0; i < rows; i++) {
        orc_swiglu_f32(h + i * 2 * F, 1, F, yf);
        for (int64_t j = 0; j < F; j++) yd[j] = (double)yf[j];
        quantize_row_f64(yd, F, q + i * F, s, ld_s, i);
    }
    free(yf);
    free(yd);
}

/* ------------------------------------------------------------------------------------------
 * NEXT-1 SwiGLU backward (the activation's gradient at the BF16 boundary; R31):
 *     y = silu(a) * b, silu(a) = a * sig(a), sig(a) = 1 / (1 + e^-a)
 *     da = dA * b * silu'(a),  silu'(a) = sig(a) * (1 + a * (1 - sig(a)))
 *     db = dA * silu(a)
 *     dH = [da | db]  (the gate half first, the same column order as h)
 *     evaluated in double, each rounded once to fp32.
 * ------------------------------------------------------------------------------------------ */
void orc_swiglu_bwd_f32(const uint16_t* h, const uint16_t* dA, int64_t rows, int64_t F, float* dh)
{
    for (int64_t i = 0; i < rows; i++)
        for (int64_t j = 0; j < F; j++) {
            double a = bf16_to_double(h[i * 2 * F + j]);
            double b = bf16_to_double(h[i * 2 * F + F + j]);
            double g = bf16_to_double(dA[i * F + j]);
            double sig = 1.0 / (1.0 + exp(-a));
            double silu = a * sig;
            double dsilu = sig * (1.0 + a * (1.0 - sig));
            dh[i * 2 * F + j] = (float)(g * b * dsilu);
            dh[i * 2 * F + F + j] = (float)(g * silu);
        }
}

/* NEXT-1 fused SwiGLU backward + quantize: C4 applied to each row of the fp32 dH (1x128 tiles along
 * 2F, fp32 amax).  q [rows][2F], s [2F/128][ld_s]. */
void orc_swiglu_bwd_quant(const uint16_t* h, const uint16_t* dA, int64_t rows, int64_t F, uint8_t* q, uint8_t* s,
                          int64_t ld_s)
{
    float* yf = (float*)malloc(sizeof(float) * (size_t)(2 * F));
    double* yd = (double*)malloc(sizeof(double) * (size_t)(2 * F));
    for (int64_t i = 0; i < rows; i++) {
        orc_swiglu_bwd_f32(h + i * 2 * F, dA + i * F, 1, F, yf);
        for (int64_t j = 0; j < 2 * F; j++) yd[j] = (double)yf[j];
        quantize_row_f64(yd, 2 * F, q + i * 2 * F, s, ld_s, i);
    }
    free(yf);
    free(yd);
}

/* C11 checksum64: sum_i b_i * (i * 0x9E3779B97F4A7C15 + 1) mod 2^64 over the bytes. */
uint64_t orc_checksum64(const uint8_t* buf, int64_t nbytes)
{
    uint64_t acc = 0;
    for (int64_t i = 0; i < nbytes; i++) acc += (uint64_t)buf[i] * ((uint64_t)i * 0x9E3779B97F4A7C15ull + 1ull);
    return acc;
}


/* NEXT-2 (R33): the GEMM that consumes the FP8 operands, by its plain
 * definition -- dequantize both operands exactly (Eq. 4) and sum the products in fp64:
 *     D[m][n] = sum_k decode(A[m][k]) 2^(sa[k/128][m]-127) * decode(B_g[n][k]) 2^(sb_g[k/128][n]-127)
 * A [M][K], B [groups][N][K] (K contiguous), sa [K/128][ld_sa], sb [groups][K/128][ld_sb];
 * group g covers rows [seg[g], seg[g+1]) (seg = NULL: one group of M rows).  Rows outside every
 * group are left untouched.  D [M][N] fp64. */
void orc_gemm_blockscaled(const uint8_t* A, const uint8_t* sa, int64_t ld_sa, const uint8_t* B, const uint8_t* sb,
                          int64_t ld_sb, int64_t M, int64_t N, int64_t K, const int32_t* seg, int32_t groups,
                          int64_t m_lo, int64_t m_hi, double* D)
{
    for (int32_t g = 0; g < (seg ? groups : 1); g++) {
        int64_t r_begin = seg ? seg[g] : 0, r_end = seg ? seg[g + 1] : M;
        if (r_begin < m_lo) r_begin = m_lo;
        if (r_end > m_hi) r_end = m_hi;
        const uint8_t* Bg = B + (int64_t)g * N * K;
        const uint8_t* sbg = sb + (int64_t)g * (K / 128) * ld_sb;
        for (int64_t m = r_begin; m < r_end; m++) {
            for (int64_t n = 0; n < N; n++) {
                double acc = 0.0;
                for (int64_t k = 0; k < K; k++) {
                    double a = orc_decode_e4m3(A[m * K + k]) * ldexp(1.0, (int)sa[(k / 128) * ld_sa + m] - 127);
                    double b = orc_decode_e4m3(Bg[n * K + k]) * ldexp(1.0, (int)sbg[(k / 128) * ld_sb + n] - 127);
                    acc += a * b;
                }
                D[m * N + n] = acc;
            }
        }
    }
}

/* ------------------------------------------------------------------------------------------
 * NEXT-3 (R34) combine: the owner of a token gathers its top_k expert
 * outputs from the ranks that computed them and sums them as C9 does ("unpermutation, and
 * combination"; BF16 at this boundary).  Rank d owns experts [d*E_per, (d+1)*E_per) and
 * holds x_d [rows_d][H] BF16 with its plan's row_map_d [T_global][K] (the C8 plan over every
 * rank's tokens, global token id = rank * tokens_per_rank + t).  For the owner's tokens
 * t = 0..T-1 (global id token_begin + t):
 *     y[t][h] = BF16_RNE( sum over k = 0..K-1 of p[t][k] * x_d[row_map_d[gt][k]][h] ),
 *     d = topk_idx[t][k] / E_per, gt = token_begin + t,
 * fp32 accumulation with one fused multiply-add per term in k order from +0.0 (p = 1, plain add,
 * when probs is NULL), exactly C9's arithmetic.  x[d] / row_map[d] are arrays of n pointers.
 * ------------------------------------------------------------------------------------------ */
void orc_combine(const uint16_t* const* x, const int32_t* const* row_map, int64_t H, const int32_t* topk_idx,
                 int32_t E_per, const float* probs, int64_t token_begin, int64_t T, int32_t K, uint16_t* y)
{
    for (int64_t t = 0; t < T; t++) {
        int64_t gt = token_begin + t;
        for (int64_t h = 0; h < H; h++) {
            float acc = 0.0f;
            for (int32_t k = 0; k < K; k++) {
                int32_t d = topk_idx[t * K + k] / E_per;
                int32_t r = row_map[d][gt * K + k];
                float xv = (float)bf16_to_double(x[d][(int64_t)r * H + h]);
                if (probs) acc = fmaf(probs[t * K + k], xv, acc);
                else acc = acc + xv;
            }
            y[t * H + h] = orc_round_bf16((double)acc);
        }
    }
}
