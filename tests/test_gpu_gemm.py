"""NEXT-2 GPU parity: the tcgen05 block-scaled FP8 GEMM against the oracle's fp64 definition
(R33), fed with random E4M3 codes and UE8M0 scales and with the outputs of the hot path's own
kernels (A1 row-wise for Fprop, A2 column-wise for Wgrad).

Tolerance: the tensor core accumulates in fp32 (order unspecified), so |D - D_ref| is bounded by
a small multiple of 2^-23 * K * (|A| |B|^T); the test bound is 2^-14 * (|A| |B|^T)[m][n] (the
measured worst case is printed), plus BF16 rounding (2^-8 relative) for BF16 output."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_02302_b200 import fp8flow

    fp8flow.fp8flow_device_check()
    return fp8flow


def rand_operand(rng, rows, K, ld, scale_lo=120, scale_hi=134):
    q = rng.integers(0, 256, (rows, K), dtype=np.uint8)
    q[(q & 0x7F) == 0x7F] = 0x3C  # no NaN codes
    s = rng.integers(scale_lo, scale_hi, (K // 128, ld), dtype=np.uint8)
    return q, s


def run_gemm(F, A, sa, B, sb, seg=None, f32=True):
    M = A.shape[0]
    N = B.shape[-2]
    D = torch.full((M, N), float("nan"), dtype=torch.float32 if f32 else torch.bfloat16, device="cuda")
    F.fp8flow_gemm_blockscaled(torch.from_numpy(A).cuda(), torch.from_numpy(sa).cuda(), torch.from_numpy(B).cuda(),
                               torch.from_numpy(sb).cuda(), D,
                               seg_offsets=None if seg is None else torch.from_numpy(np.asarray(seg, np.int32)).cuda())
    torch.cuda.synchronize()
    return D.float().cpu().numpy()


def abs_ref(orc, A, sa, B, sb, seg=None):
    """(|A| |B|^T) per output, from the oracle on magnitude codes (sign bit cleared)."""
    return orc.gemm_blockscaled(A & 0x7F, sa, B & 0x7F, sb, seg)


def check(D, ref, mag, rows, bf16=False, what=""):
    err = np.abs(D[rows] - ref[rows])
    bound = 2.0 ** -14 * mag[rows] + (2.0 ** -8 * np.abs(ref[rows]) if bf16 else 0.0) + 1e-30
    rel = float(np.max(err / (mag[rows] + 1e-30)))
    print(f"{what}: max |D - ref| / (|A||B|^T) = {rel:.3e}")
    assert np.all(err <= bound), (np.argwhere(err > bound)[:5], rel)


@pytest.mark.parametrize("M,N,K", [(128, 256, 128), (256, 512, 512), (384, 256, 1024), (256, 768, 256)])
def test_gemm_single_group(F, orc, M, N, K):
    """N = 256 or 768 (odd number of 256-column tiles): one CTA per tile; N = 512: CTA pairs that
    share the A tile by TMA multicast."""
    rng = np.random.default_rng(M + N + K)
    A, sa = rand_operand(rng, M, K, M)
    B, sb = rand_operand(rng, N, K, N)
    D = run_gemm(F, A, sa, B, sb)
    ref = orc.gemm_blockscaled(A, sa, B, sb)
    check(D, ref, abs_ref(orc, A, sa, B, sb), slice(0, M), what=f"{M}x{N}x{K}")


def test_gemm_unit_scales_small_ints(F, orc):
    """Scale bytes 127 and codes of small integers: every product and partial sum is exact in fp32,
    so the result must be bit-exact (checks operand layout, descriptors and the epilogue)."""
    rng = np.random.default_rng(5)
    M, N, K = 128, 256, 256
    ints = np.array([0x00, 0x38, 0x40, 0x44, 0x48, 0xB8, 0xC0, 0xC4, 0xC8], np.uint8)  # 0, +-1, 2, 3, 4
    A = ints[rng.integers(0, len(ints), (M, K))]
    B = ints[rng.integers(0, len(ints), (N, K))]
    sa = np.full((K // 128, M), 127, np.uint8)
    sb = np.full((K // 128, N), 127, np.uint8)
    D = run_gemm(F, A, sa, B, sb)
    np.testing.assert_array_equal(D, orc.gemm_blockscaled(A, sa, B, sb))


def test_gemm_scale_layout(F, orc):
    """Distinct scale bytes per row and per K block on both operands, with a range narrow enough
    (products 2^-4..2^6, 512 terms) that every partial sum is exact in fp32: catches any mix-up of
    the tensor-memory scale-factor layout (bit-exact)."""
    rng = np.random.default_rng(6)
    M, N, K = 128, 256, 512
    A = np.full((M, K), 0x38, np.uint8)          # 1.0
    B = np.full((N, K), 0x38, np.uint8)
    sa = rng.integers(125, 131, (K // 128, M), dtype=np.uint8)
    sb = rng.integers(125, 131, (K // 128, N), dtype=np.uint8)
    D = run_gemm(F, A, sa, B, sb)
    np.testing.assert_array_equal(D, orc.gemm_blockscaled(A, sa, B, sb))


def test_gemm_groups_and_bf16(F, orc):
    """Expert groups over M (multiples of 16, an empty group, partial 128-row blocks) with
    per-group weights; rows outside every group untouched; BF16 output."""
    rng = np.random.default_rng(7)
    seg = np.array([0, 48, 48, 208, 400], np.int32)
    M, N, K, G = 416, 256, 256, 4
    A, sa = rand_operand(rng, M, K, M)
    Bs = [rand_operand(rng, N, K, N) for _ in range(G)]
    B = np.stack([b[0] for b in Bs])
    sb = np.stack([b[1] for b in Bs])
    ref = orc.gemm_blockscaled(A, sa, B, sb, seg)
    mag = abs_ref(orc, A, sa, B, sb, seg)
    D = run_gemm(F, A, sa, B, sb, seg)
    check(D, ref, mag, slice(0, 400), what="groups f32")
    assert np.all(np.isnan(D[400:]))
    Db = run_gemm(F, A, sa, B, sb, seg, f32=False)
    check(Db, ref, mag, slice(0, 400), bf16=True, what="groups bf16")


def test_gemm_consumes_hot_path_outputs(F, orc):
    """Casting-free end to end: Fprop on A1's row-wise output and Wgrad on A2's column-wise
    outputs, each against the oracle GEMM of the same FP8 operands and against the BF16 product
    of the unquantized inputs (quantization error only)."""
    rng = np.random.default_rng(8)
    T, H, N = 256, 512, 256
    x = synth.activations_bf16(T, H, 71)
    w = synth.normal_bf16(N, H, 72, sigma=0.05)
    qx, sx = orc.quantize_rowwise_bf16(synth.bf16_bits(x))
    qw, sw = orc.quantize_rowwise_bf16(synth.bf16_bits(w))
    D = run_gemm(F, qx, sx, qw, sw)
    check(D, orc.gemm_blockscaled(qx, sx, qw, sw), abs_ref(orc, qx, sx, qw, sw), slice(0, T), what="fprop")
    exact = x.double() @ w.double().T
    assert np.max(np.abs(D - exact.numpy())) <= 0.1 * np.max(np.abs(exact.numpy()))
    # Wgrad: dW[n][h] = sum_t dy[t][n] x[t][h] -> A = dy^T (A2 of dy), B = x^T (A2 of x), K = tokens
    dy = synth.normal_bf16(T, N, 73)
    qd, sd = orc.quantize_rowwise_bf16(synth.bf16_bits(dy))
    dT, sdT = orc.scaling_aware_transpose(qd, sd)
    xT, sxT = orc.scaling_aware_transpose(qx, sx)
    A2 = dT.reshape(N, T)
    B2 = xT.reshape(H, T)
    sA2 = np.ascontiguousarray(sdT)                                   # [T/128][N]
    sB2 = np.ascontiguousarray(sxT)                                   # [T/128][H]
    D2 = run_gemm(F, A2, sA2, B2[:256], sB2[:, :256])
    check(D2, orc.gemm_blockscaled(A2, sA2, B2[:256], sB2[:, :256]), abs_ref(orc, A2, sA2, B2[:256], sB2[:, :256]),
          slice(0, N), what="wgrad")


def test_gemm_dgrad_on_transposed_weights(F, orc):
    """Dgrad with the same kernel: dX = dY W contracts over N, so the B operand is W^T in K-major
    form -- exactly A2's column-wise output of the row-wise FP8 weights (no re-quantization)."""
    T, N, H = 256, 384, 256
    dy = synth.normal_bf16(T, N, 81)
    w = synth.normal_bf16(N, H, 82, sigma=0.05)
    qd, sd = orc.quantize_rowwise_bf16(synth.bf16_bits(dy))          # A: [T][N], K = N
    qw, sw = orc.quantize_rowwise_bf16(synth.bf16_bits(w))           # W: [N][H] row-wise along H
    wT, swT = orc.scaling_aware_transpose(qw, sw)                    # W^T: [H][N], scales [N/128][H]
    B = wT.reshape(H, N)
    D = run_gemm(F, qd, sd, B, np.ascontiguousarray(swT))
    check(D, orc.gemm_blockscaled(qd, sd, B, swT), abs_ref(orc, qd, sd, B, swT), slice(0, T), what="dgrad")
    exact = (dy.double() @ w.double()).numpy()
    assert np.max(np.abs(D - exact)) <= 0.1 * np.max(np.abs(exact))


@pytest.mark.parametrize("m,Ma,Nb,bf16", [([128, 256], 128, 256, False), ([16, 0, 144, 528, 48], 128, 256, False),
                                          ([16, 0, 144, 528, 48], 384, 512, False), ([272, 0, 32], 512, 768, True),
                                          ([16, 0, 144, 528, 48], 128, 1792, False), ([272, 0, 32], 256, 1792, True)])
def test_gemm_wgrad_grouped_k(F, orc, m, Ma, Nb, bf16):
    """Wgrad with groups over K (each expert's tokens, multiples of 16, an empty expert, partial K
    blocks): dW_e = dH_e^T X_e straight from A2's column-wise outputs of dH and X_perm.  Ma = 128
    and 384 leave the last CTA pair half outside Ma; fp32 and BF16 outputs; Nb = 1792 (7 column
    tiles: an odd count of 256-column tiles per 256-row block pair)."""
    seg = np.concatenate([[0], np.cumsum(m)]).astype(np.int32)
    R = int(seg[-1])
    dh = synth.normal_bf16(R, Ma, 91)
    x = synth.activations_bf16(R, Nb, 92)
    qd, sd = orc.quantize_rowwise_bf16(synth.bf16_bits(dh))
    qx, sx = orc.quantize_rowwise_bf16(synth.bf16_bits(x))
    dT, sdT = orc.scaling_aware_transpose(qd, sd, seg)
    xT, sxT = orc.scaling_aware_transpose(qx, sx, seg)
    G = len(m)
    D = torch.full((G, Ma, Nb), float("nan"), dtype=torch.bfloat16 if bf16 else torch.float32, device="cuda")
    F.fp8flow_gemm_wgrad(torch.from_numpy(dT).cuda(), torch.from_numpy(np.ascontiguousarray(sdT)).cuda(),
                         torch.from_numpy(xT).cuda(), torch.from_numpy(np.ascontiguousarray(sxT)).cuda(), D,
                         torch.from_numpy(seg).cuda())
    torch.cuda.synchronize()
    D = D.float().cpu().numpy()
    P = np.concatenate([[0], np.cumsum((np.asarray(m) + 127) // 128)])
    for e in range(G):
        o, me = int(seg[e]), int(m[e])
        if me == 0:
            assert np.all(D[e] == 0.0)
            continue
        A = dT[Ma * o: Ma * (o + me)].reshape(Ma, me)
        B = xT[Nb * o: Nb * (o + me)].reshape(Nb, me)
        sA, sB = sdT[P[e]:P[e + 1]], sxT[P[e]:P[e + 1]]
        check(D[e], orc.gemm_blockscaled(A, sA, B, sB), orc.gemm_blockscaled(A & 0x7F, sA, B & 0x7F, sB),
              slice(0, Ma), bf16=bf16, what=f"wgrad e{e} m_e={me}")
