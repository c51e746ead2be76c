"""Pins for the oracle's MoE data-movement ops: A3 permute plan + move (C8), A4 unpermute (C9),
A5 SwiGLU + quant (C10).

Pins: the SPEC worked example, multiple-of-16 padding, bijection of the plan,
permute/unpermute round trips that reduce to exact arithmetic identities, convex-gate and top-1
special cases, SwiGLU special cases and a library routine
(torch float64 silu) for the fp32 SwiGLU values.  Beyond those, SwiGLU+quant's parity is the
fp64 definition plus the tolerance ("parity partly unpinned").
"""
import json
import os

import numpy as np
import torch

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def bits_to_f64(b):
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).to(torch.float64).numpy()


def f32_to_bits(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


# ------------------------------------------------------------------------------ A3 plan
def test_permute_worked_example(orc):
    ex = json.load(open(os.path.join(GOLDEN, "worked_examples.json")))["permute"]
    idx = np.array(ex["topk_idx"], np.int32)
    row_map, src, off = orc.permute_plan(idx, 0, 2, align=ex["align"], max_rows=len(ex["src_of_row"]))
    assert src.tolist() == ex["src_of_row"] and off.tolist() == ex["offsets"]
    assert row_map[:, 0].tolist() == [16, 0, 17]


def _check_plan(idx, e0, E_loc, align, row_map, src, off):
    T, K = idx.shape
    local = (idx >= e0) & (idx < e0 + E_loc)
    counts = np.array([np.sum(idx == e0 + e) for e in range(E_loc)])
    padded = -(-counts // align) * align
    assert np.array_equal(np.diff(off), padded) and off[0] == 0          # P:319 multiples of align
    assert np.all(row_map[~local] == -1) and np.all(row_map[local] >= 0)
    rows = row_map[local]
    assert len(np.unique(rows)) == rows.size                             # injective
    tt = np.repeat(np.arange(T)[:, None], K, axis=1)[local]
    assert np.array_equal(src[rows], tt)                                 # inverse map (bijection)
    assert np.sum(src >= 0) == rows.size                                 # every other row is PAD
    for e in range(E_loc):                                               # R16: ascending tokens,
        seg = src[off[e]:off[e + 1]]                                     # PAD rows at the end
        real = seg[: counts[e]]
        assert np.all(np.diff(real) > 0) and np.all(seg[counts[e]:] == -1)
        exp_of_rows = idx[real]
        assert np.all((exp_of_rows == e0 + e).any(axis=1))


def test_permute_plan_invariants_routing(orc):
    idx, _ = synth.routing(512, 5, num_experts=64, top_k=6, num_groups=8, topk_groups=4)
    for e0, E_loc, align in [(0, 64, 16), (16, 16, 16), (8, 8, 128), (60, 4, 1)]:
        row_map, src, off = orc.permute_plan(idx.numpy(), e0, E_loc, align=align)
        _check_plan(idx.numpy(), e0, E_loc, align, row_map, src, off)


def test_permute_plan_empty_and_tiny_experts(orc):
    idx = np.array([[0, 3], [3, 1], [1, 0]], np.int32)                    # expert 2 receives none
    row_map, src, off = orc.permute_plan(idx, 0, 4, align=16)
    assert off.tolist() == [0, 16, 32, 32, 48]
    _check_plan(idx, 0, 4, 16, row_map, src, off)


# ------------------------------------------------------------------------------ A3 move + A4
def test_permute_move_copies_rows_and_scales(orc):
    T, H = 200, 512
    x = synth.activations_bf16(T, H, 3)
    q, s = orc.quantize_rowwise_bf16(synth.bf16_bits(x))
    idx, _ = synth.routing(T, 4, num_experts=16, top_k=4, num_groups=4, topk_groups=2)
    row_map, src, off = orc.permute_plan(idx.numpy(), 0, 16)
    qo, so = orc.permute_pad(q, s, src, off)
    R = off[-1]
    real = src[:R] >= 0
    assert np.array_equal(qo[:R][real], q[src[:R][real]])
    assert np.array_equal(so[:, :R][:, real], s[:, src[:R][real]])
    assert np.all(qo[:R][~real] == 0) and np.all(so[:, :R][:, ~real] == 0)   # PAD: 0x00 / 0x00
    # threaded split is schedule-independent
    qo2, so2 = orc.permute_pad(q, s, src, off, threads=3)
    assert np.array_equal(qo, qo2) and np.array_equal(so, so2)


def test_unpermute_of_permute_is_K_times_X(orc):
    """All experts local, probs NULL, K a power of two: summing K identical BF16 copies in fp32
    is exact, so unpermute(dequant(permute(Q))) == K * dequant(Q) bit for bit."""
    T, H, K = 96, 256, 4
    x = synth.activations_bf16(T, H, 5)
    xb = synth.bf16_bits(x)
    idx, _ = synth.routing(T, 6, num_experts=16, top_k=K, num_groups=4, topk_groups=2)
    row_map, src, off = orc.permute_plan(idx.numpy(), 0, 16)
    # move BF16 rows by hand through src_of_row (the A3 move on 2-byte elements)
    xp = np.zeros((len(src), H), np.uint16)
    xp[src >= 0] = xb[src[src >= 0]]
    y = orc.unpermute(xp, row_map)
    assert np.array_equal(bits_to_f64(y), K * bits_to_f64(xb))


def test_unpermute_top1_inverse_and_convex_gates(orc):
    T, H = 64, 256
    xb = synth.bf16_bits(synth.normal_bf16(T, H, 8))
    idx = (np.arange(T) % 4).astype(np.int32)[:, None]                   # top-1, 4 experts
    row_map, src, off = orc.permute_plan(idx, 0, 4)
    xp = np.zeros((len(src), H), np.uint16)
    xp[src >= 0] = xb[src[src >= 0]]
    assert np.array_equal(orc.unpermute(xp, row_map), xb)                 # S:305 exact inverse
    assert np.array_equal(orc.unpermute(xp, row_map, np.ones((T, 1), np.float32)), xb)
    # gates [0.25, 0.75] over two equal expert outputs -> the same value
    idx2 = np.stack([np.zeros(T), np.ones(T)], 1).astype(np.int32)
    rm2, src2, _ = orc.permute_plan(idx2, 0, 2)
    xp2 = np.zeros((len(src2), H), np.uint16)
    xp2[src2 >= 0] = xb[src2[src2 >= 0]]
    p = np.tile(np.array([[0.25, 0.75]], np.float32), (T, 1))
    assert np.array_equal(orc.unpermute(xp2, rm2, p), xb)
    # tokens whose experts are all non-local -> +0
    rm3 = np.full((T, 2), -1, np.int32)
    assert np.all(orc.unpermute(xp2, rm3, p) == 0)


def test_unpermute_weighted_sum_fp32_order(orc):
    """y = BF16(sum_k fma(p, x, acc)) in k order: check against numpy fp32 fma emulated exactly
    in float64 (p*x is exact in fp64 for fp32 p and BF16 x; one rounding to fp32 per step)."""
    T, H, K = 32, 128, 8
    xb = synth.bf16_bits(synth.normal_bf16(T * K, H, 9))
    row_map = np.arange(T * K, dtype=np.int32).reshape(T, K)
    row_map[::3, 2] = -1
    p = np.random.default_rng(0).random((T, K)).astype(np.float32)
    y = orc.unpermute(xb, row_map, p)
    xv = bits_to_f64(xb)
    acc = np.zeros((T, H), np.float32)
    for k in range(K):
        r = row_map[:, k]
        term = p[:, k].astype(np.float64)[:, None] * xv[np.maximum(r, 0)]
        new = (term + acc.astype(np.float64)).astype(np.float32)        # exact sum, one rounding
        acc = np.where((r >= 0)[:, None], new, acc)
    assert np.array_equal(y, f32_to_bits(acc))


def test_unpermute_k_order_half_ulp_tie(orc):
    """R21: the terms are summed in fp32 in k order from +0, then rounded once to
    BF16.  Hand-built terms where that order is visible in the BF16 result:
        1, 2^-8, 2^-24, 2^-24  (all exact BF16)
    k order: 1 + 2^-8 is exact; + 2^-24 is an fp32 tie (ulp 2^-23 at 1) -> even -> 1 + 2^-8,
    twice; BF16(1 + 2^-8) is a BF16 tie (ulp 2^-7) -> even -> 1.0 = 0x3F80.
    The reverse order (or pairwise sums, or an fp64 accumulator) keeps 2^-23 and ends at
    1 + 2^-8 + 2^-23 -> rounds up to 1 + 2^-7 = 0x3F81.  A second token lists the same rows in
    the opposite order, so its k-order result is 0x3F81.  Checked through the plain-add path
    (probs NULL) and the fused multiply-add path (p = 1)."""
    H = 128
    vals = np.array([0x3F80, 0x3B80, 0x3380, 0x3380], np.uint16)         # 1, 2^-8, 2^-24, 2^-24
    assert np.array_equal(bits_to_f64(vals), [1.0, 2.0 ** -8, 2.0 ** -24, 2.0 ** -24])
    x = np.repeat(vals[:, None], H, axis=1)
    row_map = np.array([[0, 1, 2, 3], [3, 2, 1, 0]], np.int32)
    for probs in (None, np.ones((2, 4), np.float32)):
        y = orc.unpermute(x, row_map, probs)
        assert np.all(y[0] == 0x3F80) and np.all(y[1] == 0x3F81), (probs is None, y[:, 0])


# ------------------------------------------------------------------------------ A5
def test_swiglu_values_match_torch_float64(orc):
    h = synth.normal_bf16(256, 1024, 10, sigma=1.5)
    y = orc.swiglu_f32(synth.bf16_bits(h))
    hd = h.to(torch.float64)
    ref = (torch.nn.functional.silu(hd[:, :512]) * hd[:, 512:]).to(torch.float32).numpy()
    diff = y != ref
    assert diff.mean() < 1e-4                                             # rounding-boundary cases only
    if diff.any():
        assert np.all(np.abs(y[diff].view(np.int32) - ref[diff].view(np.int32)) == 1)


def test_swiglu_quant_special_cases(orc):
    z = np.zeros((4, 512), np.uint16)
    q, s = orc.swiglu_quant(z)
    assert np.all(q == 0) and np.all(s == 0)                              # S:315 H = 0 -> zero codes
    # silu(0) = 0: a = 0, b arbitrary -> +-0 codes
    hb = synth.bf16_bits(synth.normal_bf16(4, 512, 11))
    hb[:, :256] = 0
    q, _ = orc.swiglu_quant(hb)
    assert np.all((q & 0x7F) == 0)
    # a = b = c large: silu(c) * c -> c^2; c = 16: y = 256 / (1 + e^-16) ~ 256 - 2.9e-5
    c = torch.full((2, 512), 16.0).to(torch.bfloat16)
    q, s = orc.swiglu_quant(synth.bf16_bits(c))
    assert np.all(s == 127) and np.all(q == 0x78)                          # T = 0, 256 = 0x78
    # the codes equal the quantization of the fp32 SwiGLU values (fused == quantize ∘ swiglu)
    h = synth.normal_bf16(64, 512, 12, sigma=1.5)
    q, s = orc.swiglu_quant(synth.bf16_bits(h))
    q2, s2 = orc.quantize_rows_f64(orc.swiglu_f32(synth.bf16_bits(h)).astype(np.float64))
    assert np.array_equal(q, q2) and np.array_equal(s, s2)


# ------------------------------------------------------------------------------ NEXT-1 SwiGLU backward
def test_swiglu_bwd_matches_torch_float64_autograd(orc):
    """Library pin: torch float64 autograd of silu(a) * b with upstream gradient dA."""
    rows, F = 128, 256
    h = synth.normal_bf16(rows, 2 * F, 20, sigma=1.5)
    dA = synth.normal_bf16(rows, F, 21, sigma=0.7)
    dh = orc.swiglu_bwd_f32(synth.bf16_bits(h), synth.bf16_bits(dA))
    hd = h.to(torch.float64).requires_grad_(True)
    y = torch.nn.functional.silu(hd[:, :F]) * hd[:, F:]
    y.backward(dA.to(torch.float64))
    ref = hd.grad.to(torch.float32).numpy()
    diff = dh != ref
    assert diff.mean() < 1e-4                       # fp32 rounding-boundary cases only
    if diff.any():
        assert np.all(np.abs(dh[diff].view(np.int32) - ref[diff].view(np.int32)) == 1)


def test_swiglu_bwd_central_differences(orc):
    """the analytic gradient agrees with central differences of the fp64 forward."""
    rng = np.random.default_rng(22)
    a = rng.normal(0, 2, 400)
    b = rng.normal(0, 1, 400)
    # BF16-representable inputs so the oracle sees exactly these values
    a = torch.tensor(a).to(torch.bfloat16).to(torch.float64).numpy()
    b = torch.tensor(b).to(torch.bfloat16).to(torch.float64).numpy()
    h = np.concatenate([a, b])[None, :].astype(np.float64)
    hb = synth.bf16_bits(torch.from_numpy(h).to(torch.bfloat16))
    one = synth.bf16_bits(torch.ones(1, 400, dtype=torch.bfloat16))
    dh = orc.swiglu_bwd_f32(hb, one).astype(np.float64)[0]
    f = lambda aa, bb: aa / (1 + np.exp(-aa)) * bb  # noqa: E731
    eps = 1e-4
    fd_a = (f(a + eps, b) - f(a - eps, b)) / (2 * eps)
    fd_b = (f(a, b + eps) - f(a, b - eps)) / (2 * eps)
    scale = np.maximum(1.0, np.abs(fd_a))
    assert np.all(np.abs(dh[:400] - fd_a) <= 1e-6 * scale + 2e-7 * np.abs(b) * 4)
    assert np.all(np.abs(dh[400:] - fd_b) <= 1e-6 * np.maximum(1.0, np.abs(fd_b)))


def test_swiglu_bwd_special_cases_and_quant(orc):
    # a = 0, b = 1, dY = 1 -> da = silu'(0) = 0.5, db = silu(0) = 0
    F = 128
    h = torch.zeros(1, 2 * F)
    h[0, F:] = 1.0
    dh = orc.swiglu_bwd_f32(synth.bf16_bits(h.to(torch.bfloat16)), synth.bf16_bits(torch.ones(1, F).to(torch.bfloat16)))
    assert np.all(dh[0, :F] == 0.5) and np.all(dh[0, F:] == 0.0)
    # dA = 0 -> dH = 0 -> zero codes and the neutral scale (R11)
    hb = synth.bf16_bits(synth.normal_bf16(4, 2 * F, 23))
    q, s = orc.swiglu_bwd_quant(hb, np.zeros((4, F), np.uint16))
    assert np.all((q & 0x7F) == 0) and np.all(s == 0)
    # fused = quantize(dH) on the fp32 values
    dA = synth.bf16_bits(synth.normal_bf16(4, F, 24))
    q, s = orc.swiglu_bwd_quant(hb, dA)
    q2, s2 = orc.quantize_rows_f64(orc.swiglu_bwd_f32(hb, dA).astype(np.float64))
    assert np.array_equal(q, q2) and np.array_equal(s, s2)


# ============================================================================ NEXT-2 GEMM oracle
def _torch_dequant(q, s):
    """Independent decode: torch's float8_e4m3fn reinterpretation (a library routine) times 2^T."""
    vals = torch.from_numpy(np.ascontiguousarray(q)).view(torch.float8_e4m3fn).to(torch.float64)
    K = q.shape[1]
    T = torch.from_numpy(s[: K // 128, : q.shape[0]].astype(np.int64) - 127).T          # [rows, K/128]
    return vals * torch.pow(2.0, T.repeat_interleave(128, dim=1).to(torch.float64))


def _rand_operand(rng, rows, K, ld):
    q = rng.integers(0, 256, (rows, K), dtype=np.uint8)
    q[(q & 0x7F) == 0x7F] = 0x3C                                                         # no NaN codes
    s = rng.integers(110, 140, (K // 128, ld), dtype=np.uint8)
    return q, s


def test_gemm_oracle_vs_torch_matmul(orc):
    """Pin: torch float64 matmul of torch-decoded, scaled operands, with groups over M."""
    rng = np.random.default_rng(41)
    M, N, K, G = 96, 48, 384, 3
    A, sa = _rand_operand(rng, M, K, 112)
    Bs = [_rand_operand(rng, N, K, 64) for _ in range(G)]
    B = np.stack([b[0] for b in Bs])
    sb = np.stack([b[1] for b in Bs])
    seg = np.array([0, 16, 16, 80], np.int32)                                            # empty group, rows 80.. none
    D = orc.gemm_blockscaled(A, sa, B, sb, seg)
    Ad = _torch_dequant(A, sa)
    for g in range(G):
        lo, hi = seg[g], seg[g + 1]
        ref = (Ad[lo:hi] @ _torch_dequant(B[g], sb[g]).T).numpy()
        np.testing.assert_allclose(D[lo:hi], ref, rtol=1e-12, atol=0)
    assert np.all(np.isnan(D[80:]))                                                      # outside every group


def test_gemm_oracle_one_hot_rows(orc):
    """Pin (closed form): a row of A holding the single code 0x38 (= 1.0) at column k with scale
    byte t selects 2^(t-127) * dequant(B)[:, k]."""
    rng = np.random.default_rng(42)
    M, N, K = 16, 32, 256
    A = np.zeros((M, K), np.uint8)
    sa = np.full((K // 128, M), 127, np.uint8)
    ks = rng.integers(0, K, M)
    for m in range(M):
        A[m, ks[m]] = 0x38
        sa[ks[m] // 128, m] = 120 + m
    B, sb = _rand_operand(rng, N, K, N)
    D = orc.gemm_blockscaled(A, sa, B, sb)
    Bd = orc.dequantize_rows(B, sb)
    for m in range(M):
        np.testing.assert_array_equal(D[m], 2.0 ** (120 + m - 127) * Bd[:, ks[m]])


def test_gemm_oracle_scale_linearity(orc):
    """Pin: adding d to every scale byte of A multiplies D by 2^d exactly (pow2 scales)."""
    rng = np.random.default_rng(43)
    A, sa = _rand_operand(rng, 32, 256, 32)
    B, sb = _rand_operand(rng, 16, 256, 16)
    D0 = orc.gemm_blockscaled(A, sa, B, sb)
    D1 = orc.gemm_blockscaled(A, sa + 3, B, sb)
    np.testing.assert_array_equal(D1, D0 * 8.0)
