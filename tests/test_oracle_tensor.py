"""Pins for the oracle's tensor operations: A1 quantize (C4), A2 scaling-aware transpose (C6),
the naive comparator and Eq. 1 demonstration (C7).

What pins them (besides the scalar codec pins): Eqs. 5-8 idempotence, the exactness
theorem of the exponent-shift derivation, Algorithm 1's scale alignment,
special cases (k = 0 pure byte transpose, constant matrices), library casts of exact products,
T∘T∘T = T and T∘T = id on block-uniform input (R24), and the double-quantization error of
Eq. 1 / Eq. 9 being visible on the naive path.
"""
import json
import os

import numpy as np
import pytest
import torch

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def lib_decode(codes: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(codes)).view(torch.float8_e4m3fn).to(torch.float64).numpy()


def lib_encode(v: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).to(torch.float8_e4m3fn).view(torch.uint8).numpy()


def tile_dequant(q, s):
    """decode(q) * 2^(s-127), rows tiled along the columns (independent numpy + torch decode)."""
    rows, cols = q.shape
    T = s[: cols // 128, :rows].astype(np.int64).T - 127            # [rows, tiles]
    return lib_decode(q) * np.exp2(np.repeat(T, 128, axis=1)).astype(np.float64)


# ------------------------------------------------------------------------------ A1 / C4
@pytest.mark.parametrize("dist", ["normal", "uniform", "lognormal", "activations"])
def test_quantize_idempotent_eqs5to8(orc, dist):
    rng = np.random.default_rng(hash(dist) % 2 ** 32)
    rows, cols = 96, 512                                              # 384 tiles per draw
    if dist == "normal":
        x = rng.standard_normal((rows, cols))
    elif dist == "uniform":
        x = rng.uniform(-3, 3, (rows, cols))
    elif dist == "lognormal":
        x = np.exp(rng.normal(0, 3, (rows, cols))) * rng.choice([-1, 1], (rows, cols))
    else:
        x = synth.activations_bf16(rows, cols, 7).to(torch.float64).numpy()
    q, s = orc.quantize_rows_f64(x)
    d = orc.dequantize_rows(q, s)
    q2, s2 = orc.quantize_rows_f64(d)
    # Eqs. 5-8 at value level: D(Q(D(Q(X)))) == D(Q(X)) exactly
    assert np.array_equal(orc.dequantize_rows(q2, s2), d)
    # bitwise wherever the tile scale is unchanged.  With ceil-pow2 scales (R3) a tile whose amax
    # lies in (224, 232) * 2^T rounds its max down onto 448 * 2^(T-1), so the second pass picks
    # T-1 and re-expresses the same values one binade up (R28 in DESIGN.md).
    same = (s2 == s).T                                                # [rows, tiles]
    assert np.array_equal(q[np.repeat(same, 128, axis=1)], q2[np.repeat(same, 128, axis=1)])
    assert np.all((s2 == s) | (s2.astype(int) == s.astype(int) - 1))
    assert not np.any((q & 0x7F) == 0x7F)                             # never NaN: no overflow
    # each code is the library RNE cast of the exact product x * 2^-T (one rounding, |.| <= 448)
    T = s.astype(np.int64).T - 127
    prod = x * np.exp2(-np.repeat(T, 128, axis=1).astype(np.float64))
    assert np.all(np.abs(prod) <= 448.0)
    f32 = prod.astype(np.float32)
    exact = f32.astype(np.float64) == prod
    assert np.array_equal(q[exact], lib_encode(f32[exact]))
    # the scale covers the tile and is the least such power of two (Eq. 2, R3)
    amax = np.abs(x).reshape(rows, cols // 128, 128).max(-1)
    nz = amax > 0
    assert np.all(amax[nz] <= 448.0 * np.exp2(T[nz])) and np.all(amax[nz] > 448.0 * np.exp2(T[nz] - 1.0))


def test_quantize_idempotent_real_scales_bitwise(orc):
    """Eqs. 5-8 with the real-valued scale of Eq. 2 (s = amax/448): the tile max maps exactly
    onto 448, so s is unchanged and the second quantization is bit-identical."""
    rng = np.random.default_rng(21)
    for x in (rng.standard_normal((64, 512)), np.exp(rng.normal(0, 3, (64, 512)))):
        q, s = orc.quantize_rows_real(x)
        d = lib_decode(q) * np.repeat(s.T, 128, axis=1)
        q2, s2 = orc.quantize_rows_real(d)
        assert np.array_equal(q, q2) and np.array_equal(s, s2)


def test_quantize_examples(orc):
    x = 448.0 * np.eye(128)                                           # SPEC tile_quant S:154
    q, s = orc.quantize_rows_f64(x)
    assert np.all(s == 127) and np.all(np.diag(q) == 0x7E) and np.all(q[~np.eye(128, dtype=bool)] == 0)
    q, s = orc.quantize_rows_f64(np.zeros((2, 256)))                  # zero tile: T = -127 (R11)
    assert np.all(s == 0) and np.all(q == 0)


def test_quantize_bf16_entry_matches_f64_path(orc):
    x = synth.activations_bf16(64, 1024, 11)
    q, s = orc.quantize_rowwise_bf16(synth.bf16_bits(x))
    q2, s2 = orc.quantize_rows_f64(x.to(torch.float64).numpy())
    assert np.array_equal(q, q2) and np.array_equal(s, s2)
    # threaded split is schedule-independent
    q3, s3 = orc.quantize_rowwise_bf16(synth.bf16_bits(x), threads=5)
    assert np.array_equal(q, q3) and np.array_equal(s, s3)


# ------------------------------------------------------------------------------ A2 / C6
def make_rowwise(rows, cols, seed, k_span=6, min_E=None):
    """Construct a row-wise FP8 tensor directly (codes + per-tile exponents), not via quantize.
    min_E: smallest exponent field of nonzero codes (to control underflow)."""
    rng = np.random.default_rng(seed)
    E = rng.integers(1 if min_E is None else min_E, 16, (rows, cols))
    M = rng.integers(0, 8, (rows, cols))
    M[E == 15] = rng.integers(0, 7, int(np.sum(E == 15)))             # avoid the NaN code
    S = rng.integers(0, 2, (rows, cols))
    q = ((S << 7) | (E << 3) | M).astype(np.uint8)
    T = rng.integers(-10, -10 + k_span + 1, (cols // 128, rows))
    s = (T + 127).astype(np.uint8)
    return q, s


def seg_view(qT, sT, cols, seg):
    """Split the flat A2 output into per-segment [cols, m_e] codes and [tiles_e, cols] scales."""
    out, tb = [], 0
    for e in range(len(seg) - 1):
        o, m = int(seg[e]), int(seg[e + 1] - seg[e])
        nt = (m + 127) // 128
        out.append((qT[cols * o: cols * (o + m)].reshape(cols, m), sT[tb: tb + nt]))
        tb += nt
    return out


def test_transpose_exactness_theorem(orc):
    """with no underflow, dequant(T(Q)) == transpose(dequant(Q)) elementwise."""
    k_span = 5
    q, s = make_rowwise(256, 384, 1, k_span=k_span, min_E=k_span + 1)
    qT, sT = orc.scaling_aware_transpose(q, s)
    qT = qT.reshape(384, 256)
    x = tile_dequant(q, s)                                            # [256, 384]
    TT = sT.astype(np.int64) - 127                                    # [2 row blocks, 384]
    xT = lib_decode(qT) * np.exp2(np.repeat(TT.T, 128, axis=1))       # [384, 256]
    assert np.array_equal(xT, x.T)


def test_transpose_scale_alignment_and_brute_force(orc):
    q, s = make_rowwise(256, 256, 2, k_span=12)
    qT, sT = orc.scaling_aware_transpose(q, s)
    qT = qT.reshape(256, 256)
    for ib in range(2):
        for jb in range(2):
            tmax = int(s[jb, ib * 128:(ib + 1) * 128].max())
            assert np.all(sT[ib, jb * 128:(jb + 1) * 128] == tmax)   # Alg. 1: S_col = S_max
            # every element: library RNE cast of decode * 2^-(k) with k = Tmax - T_row (R5)
            rows = np.arange(ib * 128, ib * 128 + 128)
            k = tmax - s[jb, rows].astype(np.int64)
            blk = q[rows][:, jb * 128:(jb + 1) * 128]
            vals = lib_decode(blk) * np.exp2(-k.astype(np.float64))[:, None]
            nan = np.isnan(vals)
            ref = lib_encode(np.where(nan, 0, vals)).reshape(blk.shape)
            got = qT[jb * 128:(jb + 1) * 128, ib * 128:(ib + 1) * 128].T
            assert np.array_equal(got[~nan], ref[~nan])


def test_transpose_k0_is_pure_byte_transpose(orc):
    q, s = make_rowwise(256, 256, 3, k_span=0)                        # uniform scales
    qT, sT = orc.scaling_aware_transpose(q, s)
    assert np.array_equal(qT.reshape(256, 256), q.T)


def test_transpose_worked_example(orc):
    ex = json.load(open(os.path.join(GOLDEN, "worked_examples.json")))["transpose_block"]
    q = np.full((128, 128), int(ex["in_code"], 16), np.uint8)
    s = np.full((1, 128), ex["row_T_default"] + 127, np.uint8)
    s[0, 3] = ex["row3_T"] + 127
    qT, sT = orc.scaling_aware_transpose(q, s)
    qT = qT.reshape(128, 128)
    assert np.all(sT == ex["out_T"] + 127)
    assert np.all(qT[:, 3] == int(ex["out_code_row3"], 16))
    assert np.all(np.delete(qT, 3, axis=1) == int(ex["out_code_other_rows"], 16))


def test_transpose_involution_properties(orc):
    """R24: T∘T∘T = T always; T∘T = id iff each block's row scales are uniform."""
    q, s = make_rowwise(256, 256, 4, k_span=8)
    q1, s1 = orc.scaling_aware_transpose(q, s)
    q2, s2 = orc.scaling_aware_transpose(q1.reshape(256, 256), s1)
    q3, s3 = orc.scaling_aware_transpose(q2.reshape(256, 256), s2)
    assert np.array_equal(q3, q1) and np.array_equal(s3, s1)
    qu, su = make_rowwise(256, 256, 5, k_span=0)
    a, b = orc.scaling_aware_transpose(qu, su)
    a2, b2 = orc.scaling_aware_transpose(a.reshape(256, 256), b)
    assert np.array_equal(a2.reshape(256, 256), qu) and np.array_equal(b2, su)
    # value-level identity except underflowed elements
    x = tile_dequant(q, s)
    y = tile_dequant(q2.reshape(256, 256), s2)
    lost = x != y
    # an element may change only if its first shift underflowed: nonzero code with E <= k
    tmax = s.reshape(2, 2, 128).max(-1)                                # [jb, ib]
    k = np.repeat(np.repeat(tmax, 128, axis=1), 128, axis=0).T.astype(int) - np.repeat(s.T, 128, axis=1)
    E = (q >> 3) & 15
    under = ((q & 0x7F) != 0) & (E <= k)
    assert lost.any() and not np.any(lost & ~under)


def test_transpose_segments_ragged(orc):
    """R14/R15: blocks never straddle segments; a partial last block aligns to the max over the
    rows present; the segmented result equals transposing each segment as its own tensor."""
    m = [16, 0, 144, 128, 112, 272]
    seg = np.concatenate([[0], np.cumsum(m)]).astype(np.int32)
    rows, cols = int(seg[-1]), 256
    q, s = make_rowwise(rows, cols, 6, k_span=10)
    qT, sT = orc.scaling_aware_transpose(q, s, seg)
    nbytes, ntiles = orc.transpose_out_sizes(rows, cols, seg)
    assert qT.size == nbytes and sT.shape[0] == ntiles == sum((x + 127) // 128 for x in m)
    for e, (qe, se) in enumerate(seg_view(qT, sT, cols, seg)):
        o, me = int(seg[e]), m[e]
        if me == 0:
            continue
        qs = np.ascontiguousarray(q[o:o + me])
        ss = np.ascontiguousarray(s[:, o:o + me])
        q_ref, s_ref = orc.scaling_aware_transpose(qs, ss)
        assert np.array_equal(qe, q_ref.reshape(cols, me)) and np.array_equal(se, s_ref)
        # last partial block: T_max over the rows present only
        ib = (me - 1) // 128
        assert np.all(se[ib, :128] == ss[0, ib * 128:].max())


# ------------------------------------------------------------------------------ C7 naive / Eq. 1
def test_naive_constant_and_block_uniform_cases(orc):
    # constant matrix -> naive == direct (s' = s)
    x = np.full((256, 256), 3.25)
    q, s = orc.quantize_rows_f64(x)
    a, sa = orc.naive_transpose(q, s)
    b, sb = orc.scaling_aware_transpose(q, s)
    assert np.array_equal(a, b) and np.array_equal(sa, sb)
    # every row of each block has the same max -> s' = s, E = 0 at value level
    rng = np.random.default_rng(8)
    x = rng.uniform(-1, 1, (128, 128))
    x[:, 0] = 1.0                                                      # column 0 carries the max
    x[0, :] = 1.0                                                      # row 0 carries the max
    q, s = orc.quantize_rows_f64(x)
    a, sa = orc.naive_transpose(q, s)
    b, sb = orc.scaling_aware_transpose(q, s)
    va = lib_decode(a.reshape(128, 128)) * np.exp2(sa[0].astype(np.float64) - 127)[:, None]
    vb = lib_decode(b.reshape(128, 128)) * np.exp2(sb[0].astype(np.float64) - 127)[:, None]
    assert np.array_equal(va, vb)


def test_naive_fresh_scale_per_column_block(orc):
    """P:130 / P:224 (R29): the naive route dequantizes, transposes and re-quantizes column-wise,
    with a FRESH pow2 scale for every (column, 128-row block of a segment).  Hand-built input
    whose column maxima differ between the blocks of one segment and between columns, so any other
    grouping of the amax (whole column, whole segment, blocks counted from the tensor's row 0,
    the wrong source tile's row scale) changes scales and codes.

    Value of local row l (segment e, block b = l // 128) at column j:
        X = sgn * v(l) * 2^a,   a = (j + 3b + e) mod 8 - 4,   v(l) = [1, 0.75, 0.5, 0.625][l % 4]
    (every block contains v = 1 rows, so the (column, block) amax is exactly 2^a).  Closed form of
    the expected result, from Eq. 2 with the least-T pow2 rule (R3): amax 2^a <= 448 * 2^T  <=>
    T = a - 8; the code is E4M3(X * 2^-T) = E4M3(sgn * 256 * v(l)), cast here by torch.
    The row-wise input is built directly: codes = torch E4M3 of X * 2^-T_row with per-row,
    per-tile T_row in {-2, -1, 0} (all values exact, no underflow)."""
    m = [16, 256, 144]                                   # partial block, two full blocks, 128 + 16
    seg = np.concatenate([[0], np.cumsum(m)]).astype(np.int32)
    rows, cols = int(seg[-1]), 256
    vtab = np.array([1.0, 0.75, 0.5, 0.625])
    X = np.zeros((rows, cols))
    A = np.zeros((rows, cols), np.int64)                 # the exponent a of each element
    for e in range(3):
        for l in range(m[e]):
            i = int(seg[e]) + l
            j = np.arange(cols)
            A[i] = (j + 3 * (l // 128) + e) % 8 - 4
            sgn = np.where((i * 7 + j) % 3 == 0, -1.0, 1.0)
            X[i] = sgn * vtab[l % 4] * np.exp2(A[i])
    Trow = (np.arange(rows)[None, :] + np.arange(cols // 128)[:, None]) % 3 - 2      # [tiles, rows]
    s = (Trow + 127).astype(np.uint8)
    q = lib_encode(X * np.exp2(-np.repeat(Trow.T, 128, axis=1)))
    assert np.array_equal(tile_dequant(q, s), X)                                      # exact input

    qT, sT = orc.naive_transpose(q, s, seg)
    for e, (qe, se) in enumerate(seg_view(qT, sT, cols, seg)):
        o = int(seg[e])
        for b in range((m[e] + 127) // 128):
            lo, hi = o + 128 * b, o + min(128 * (b + 1), m[e])
            a_blk = A[lo, :]                                                          # [cols]
            assert np.all(A[lo:hi] == a_blk)
            assert np.array_equal(se[b], (a_blk - 8 + 127).astype(np.uint8)), (e, b)
            want = lib_encode((X[lo:hi] * np.exp2(8 - a_blk)[None, :]).T)             # [cols, rows]
            assert np.all(np.isin(np.abs(X[lo:hi] * np.exp2(8 - a_blk)), 256 * vtab))
            assert np.array_equal(qe[:, lo - o: hi - o], want), (e, b)


def test_double_quantization_error_eq1_real_scales(orc):
    """Eq. 1 / Eq. 9: with real-valued scales (Eq. 2 literal) the naive
    dequantize -> transpose -> column-wise requantize differs from single quantization Q_col(X)."""
    rng = np.random.default_rng(9)
    x = rng.standard_normal((256, 256))
    q, sr = orc.quantize_rows_real(x)                                  # Q_row(X)
    d = lib_decode(q) * np.repeat(sr.T, 128, axis=1)                  # D(Q_row(X))
    qc, sc = orc.quantize_rows_real(np.ascontiguousarray(d.T))        # Q_col(D(Q_row(X)))
    qx, sx = orc.quantize_rows_real(np.ascontiguousarray(x.T))        # Q_col(X)
    v1 = lib_decode(qc) * np.repeat(sc.T, 128, axis=1)
    v2 = lib_decode(qx) * np.repeat(sx.T, 128, axis=1)
    E = v1 - v2
    frac = np.mean(E != 0)
    assert frac > 0.01, frac                                           # error is visible
    # and the naive path drifts from the values D(Q_row(X)) it started from
    assert np.mean(v1 != d.T) > 0.5


def test_direct_path_has_no_drift_without_underflow_pow2(orc):
    """SPEC S:233 / AC4: pow2 scales, no underflow -> direct path drift vs D(Q_row(X)) is zero,
    while the naive path's per-column requantization re-rounds."""
    x = synth.activations_bf16(256, 256, 12, gain_sigma=0.2).to(torch.float64).numpy()
    q, s = orc.quantize_rows_f64(x)
    d = tile_dequant(q, s)
    b, sb = orc.scaling_aware_transpose(q, s)
    vb = lib_decode(b.reshape(256, 256)) * np.exp2(np.repeat((sb.astype(np.float64) - 127).T, 128, axis=1))
    under = vb != d.T
    # every mismatch is an underflow (the shifted code left the normal range)
    assert np.all(np.abs(lib_decode(b.reshape(256, 256))[under]) <= 2.0 ** -6)
    assert under.mean() < 0.01
