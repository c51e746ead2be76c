"""GPU parity: every op of the hot path through the C ABI (libfp8flow via its binding) against the
CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): bit-exact codes and scales for quantize (A1), transpose (A2),
permute plan + move (A3) and unpermute (A4, BF16 bytes); SwiGLU+quant (A5) codes within 1 E4M3
ULP on <= 1e-4 of elements with byte-identical scales.  Sizes span several tiles with ragged
tails, plus the BASELINE.json full sizes (configs 1-4) and the edge cases of each method.
"""
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

    fp8flow.fp8flow_device_check()  # raises on anything but sm_100
    return fp8flow


def dev(a):
    t = torch.from_numpy(np.ascontiguousarray(a)) if isinstance(a, np.ndarray) else a
    return t.cuda()


def host(t):
    return t.cpu().numpy()


def bf16_dev(x_bits):
    return torch.from_numpy(np.ascontiguousarray(x_bits).view(np.int16)).view(torch.bfloat16).cuda()


def e4m3_ulp_dist(a, b):
    def ordv(c):
        c = c.astype(np.int32)
        return np.where(c < 0x80, c & 0x7F, -(c & 0x7F))
    return np.abs(ordv(a) - ordv(b))


# =========================================================================================== A1
def run_quantize(F, x_bf16, ld_s=None):
    rows, cols = x_bf16.shape
    ld_s = ld_s or ((rows + 15) // 16 * 16)
    q = torch.empty(rows, cols, dtype=torch.uint8, device="cuda")
    s = torch.full((cols // 128, ld_s), 0xAB, dtype=torch.uint8, device="cuda")
    F.fp8flow_quantize_rowwise(x_bf16, q, s)
    torch.cuda.synchronize()
    return host(q), host(s)


@pytest.mark.parametrize("rows,cols", [(256, 256), (1, 128), (33, 384), (1000, 1152), (4096, 7168)])
def test_quantize_parity(F, orc, rows, cols):
    x = synth.activations_bf16(rows, cols, 100 + rows)
    q, s = run_quantize(F, x.cuda())
    ld = s.shape[1]
    q_ref, s_ref = orc.quantize_rowwise_bf16(synth.bf16_bits(x), ld_s=ld)
    assert np.array_equal(q, q_ref)
    assert np.array_equal(s[:, :rows], s_ref[:, :rows])
    assert np.all(s[:, rows:] == 0xAB)                                  # padding bytes untouched


def test_quantize_edge_values(F, orc):
    """amax exactly 448*2^T and its BF16 successor, zeros, subnormal BF16, huge values, -0."""
    rows, cols = 64, 256
    rng = np.random.default_rng(0)
    x = (rng.standard_normal((rows, cols)) * 0.3).astype(np.float32)
    for i in range(rows):
        T = int(rng.integers(-30, 30))
        x[i, 5] = 448.0 * 2.0 ** T                                       # exactly on the boundary
        if i % 2:
            x[i, 6] = np.nextafter(np.float32(448.0 * 2.0 ** T), np.float32(np.inf))  # rounds up in bf16
    x[3] = 0.0                                                           # zero tile -> byte 0
    x[4, :128] = -0.0
    x[5, :] = 1e-40                                                      # bf16 subnormal
    x[6, 0] = 3.0e38                                                     # near bf16 max
    xb = torch.from_numpy(x).to(torch.bfloat16)
    q, s = run_quantize(F, xb.cuda())
    q_ref, s_ref = orc.quantize_rowwise_bf16(synth.bf16_bits(xb), ld_s=s.shape[1])
    assert np.array_equal(q, q_ref) and np.array_equal(s[:, :rows], s_ref[:, :rows])


def test_quantize_idempotent_on_gpu(F, orc):
    """AC2 / Eqs. 5-8 on the device: A1 of the dequantized codes reproduces the values
    exactly; the codes bit for bit wherever the tile scale is unchanged, else the scale drops by one
    binade (a tile max in (224, 232) * 2^T rounds onto 448 * 2^(T-1), R28)."""
    x = synth.activations_bf16(1024, 7168, 17).cuda()
    q, s = run_quantize(F, x)
    d = orc.dequantize_rows(q, s)                                    # exact: <= 4 significant bits
    d_bf16 = torch.from_numpy(d).to(torch.bfloat16)
    assert np.array_equal(d_bf16.to(torch.float64).numpy(), d)       # representable in BF16
    q2, s2 = run_quantize(F, d_bf16.cuda())
    assert np.array_equal(orc.dequantize_rows(q2, s2), d)
    same = (s2 == s).T
    assert np.array_equal(q[np.repeat(same, 128, axis=1)], q2[np.repeat(same, 128, axis=1)])
    assert np.all((s2 == s) | (s2.astype(int) == s.astype(int) - 1))


def test_quantize_deterministic(F):
    x = synth.activations_bf16(512, 2048, 7).cuda()
    a = run_quantize(F, x)
    b = run_quantize(F, x)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# =========================================================================================== A2
def run_transpose(F, q, s, seg=None, naive=False):
    rows, cols = q.shape
    nseg = 1 if seg is None else len(seg) - 1
    nbytes, ntiles = F.transpose_out_shapes(rows, cols, nseg)
    qT = torch.full((max(nbytes, 16),), 0xCD, dtype=torch.uint8, device="cuda")
    sT = torch.full((ntiles, cols), 0xCD, dtype=torch.uint8, device="cuda")
    seg_t = None if seg is None else dev(np.asarray(seg, np.int32))
    qd, sd = dev(q), dev(s)
    if naive:
        ws = torch.empty(F.fp8flow_naive_workspace_bytes(rows, cols, nseg), dtype=torch.uint8, device="cuda")
        F.fp8flow_naive_transpose(qd, sd, qT, sT, ws, seg_offsets=seg_t)
    else:
        F.fp8flow_scaling_aware_transpose(qd, sd, qT, sT, seg_offsets=seg_t)
    torch.cuda.synchronize()
    return host(qT), host(sT)


def check_transpose(F, orc, q, s, seg=None, naive=False):
    qT, sT = run_transpose(F, q, s, seg, naive)
    fn = orc.naive_transpose if naive else orc.scaling_aware_transpose
    qT_ref, sT_ref = fn(q, s, seg)
    n = qT_ref.size
    assert np.array_equal(qT[:n], qT_ref), np.argwhere(qT[:n] != qT_ref)[:5]
    assert np.array_equal(sT[:sT_ref.shape[0]], sT_ref)


def constructed_rowwise(rows, cols, seed, k_max=40, nan=False):
    """Row-wise FP8 built directly: all 254 non-NaN codes (all 256 codes with nan=True) appear in
    every row block and the block's row scales span k = 0..k_max (the adversarial all-codes x
    all-k suite)."""
    rng = np.random.default_rng(seed)
    codes = np.array([c for c in range(256) if nan or c not in (0x7F, 0xFF)], np.uint8)
    q = codes[rng.integers(0, codes.size, (rows, cols))]
    q[:, :codes.size] = codes[None, :]
    T = 100 - (np.arange(rows) % (k_max + 1))                            # block max 100 -> k = 0..k_max
    s = np.tile(T.astype(np.uint8), (cols // 128, 1))
    s = np.ascontiguousarray(np.roll(s, 3, axis=1))
    return q, s


@pytest.mark.parametrize("rows,cols", [(256, 256), (128, 128), (384, 640), (4096, 7168)])
def test_transpose_parity_quantized(F, orc, rows, cols):
    x = synth.activations_bf16(rows, cols, 200 + rows)
    q, s = orc.quantize_rowwise_bf16(synth.bf16_bits(x))
    check_transpose(F, orc, q, s)


def test_transpose_all_codes_all_k(F, orc):
    q, s = constructed_rowwise(512, 384, 1)
    check_transpose(F, orc, q, s)


def test_transpose_nan_codes_propagate(F, orc):
    """E4M3 NaN codes (0x7F, 0xFF; A1 emits them for NaN input) keep their bytes through the
    exponent shift for every k, as the oracle's shift does; the rest is unchanged."""
    q, s = constructed_rowwise(256, 384, 11, nan=True)
    check_transpose(F, orc, q, s)
    qT, _ = run_transpose(F, q, s)
    assert np.array_equal(qT.reshape(384, 256) == 0x7F, q.T == 0x7F)


def test_transpose_ragged_segments(F, orc):
    # per-expert token counts {0,1,15,16,17,127,128,129} padded to 16, plus larger ones
    m = [0, 16, 16, 16, 32, 128, 128, 144, 0, 256, 272, 16]
    seg = np.concatenate([[0], np.cumsum(m)]).astype(np.int32)
    rows, cols = int(seg[-1]), 512
    q, s = constructed_rowwise(rows, cols, 2, k_max=24)
    check_transpose(F, orc, q, s, seg)
    x = synth.activations_bf16(rows, cols, 3)
    q, s = orc.quantize_rowwise_bf16(synth.bf16_bits(x))
    check_transpose(F, orc, q, s, seg)


def test_transpose_involution_on_gpu(F, orc):
    """R24 on the device path: T∘T∘T == T bitwise."""
    q, s = constructed_rowwise(256, 256, 4, k_max=12)
    q1, s1 = run_transpose(F, q, s)
    q2, s2 = run_transpose(F, q1[: 256 * 256].reshape(256, 256), s1)
    q3, s3 = run_transpose(F, q2[: 256 * 256].reshape(256, 256), s2)
    assert np.array_equal(q3, q1) and np.array_equal(s3, s1)


@pytest.mark.parametrize("rows,cols", [(256, 256), (1024, 1024), (4096, 7168)])
def test_naive_transpose_parity(F, orc, rows, cols):
    x = synth.activations_bf16(rows, cols, 300 + rows)
    q, s = orc.quantize_rowwise_bf16(synth.bf16_bits(x))
    check_transpose(F, orc, q, s, naive=True)
    m = [16, 128, 0, rows - 144]
    seg = np.concatenate([[0], np.cumsum(m)]).astype(np.int32)
    check_transpose(F, orc, q, s, seg, naive=True)


def test_naive_transpose_ragged_segments(F, orc):
    """The comparator over expert segments {0, 16, ..., 272} rows (partial 128-row blocks, empty
    segments): fresh scales per (column, 128-row block of a segment), as the oracle (R29)."""
    m = [0, 16, 16, 16, 32, 128, 128, 144, 0, 256, 272, 16]
    seg = np.concatenate([[0], np.cumsum(m)]).astype(np.int32)
    x = synth.activations_bf16(int(seg[-1]), 512, 31)
    q, s = orc.quantize_rowwise_bf16(synth.bf16_bits(x))
    check_transpose(F, orc, q, s, seg, naive=True)


# =========================================================================================== A3
def run_plan(F, topk_idx, e0, E_loc, align=16, max_rows=None):
    T, K = topk_idx.shape
    max_rows = max_rows or F.permute_max_rows(T, K, E_loc, align)
    row_map = torch.empty(T, K, dtype=torch.int32, device="cuda")
    src = torch.full((max_rows,), -7, dtype=torch.int32, device="cuda")
    off = torch.empty(E_loc + 1, dtype=torch.int32, device="cuda")
    ws = torch.empty(F.fp8flow_permute_workspace_bytes(T, K, E_loc), dtype=torch.uint8, device="cuda")
    F.fp8flow_permute_plan(dev(topk_idx), e0, E_loc, align, row_map, src, off, ws)
    torch.cuda.synchronize()
    return host(row_map), host(src), host(off), int(host(ws[:4].view(torch.int32))[0])


@pytest.mark.parametrize("T,E,K,group,ngroups,align", [
    (16384, 256, 8, 0, 8, 16), (16384, 256, 8, 5, 8, 16), (16384, 256, 8, 0, 1, 16), (3000, 64, 6, 0, 1, 16),
    (777, 32, 4, 1, 4, 128), (5, 8, 2, 0, 2, 16), (200000, 64, 8, 3, 8, 16)])
def test_permute_plan_parity(F, orc, T, E, K, group, ngroups, align):
    """The single cooperative launch for token counts whose 512-token chunks fit on the GPU at once
    (<= 148 x its occupancy, ~75k tokens), and the two-kernel path (count, then place) beyond:
    200,000 tokens = 391 chunks.  (16384, 256 local experts) is the whole DeepSeek-V3 layer on one
    GPU."""
    idx, _ = synth.routing(T, 400 + T, num_experts=E, top_k=K, num_groups=min(8, E // 4), topk_groups=2)
    per = E // ngroups
    e0 = group * per
    rm, src, off, status = run_plan(F, idx.numpy(), e0, per, align)
    rm_ref, src_ref, off_ref = orc.permute_plan(idx.numpy(), e0, per, align=align, max_rows=len(src))
    assert status == 0
    assert np.array_equal(off, off_ref) and np.array_equal(rm, rm_ref)
    assert np.array_equal(src[: off[-1]], src_ref[: off[-1]])


def test_permute_plan_zero_tokens(F):
    idx = np.zeros((0, 8), np.int32)
    rm, src, off, status = run_plan(F, np.zeros((1, 8), np.int32)[:0], 0, 4, 16, max_rows=16)
    assert off.tolist() == [0, 0, 0, 0, 0] and status == 0
    del idx


def test_permute_plan_no_tokens_for_some_experts(F, orc):
    idx = np.array([[0, 3], [3, 1], [1, 0], [0, 1]], np.int32)
    rm, src, off, _ = run_plan(F, idx, 0, 6)
    rm_ref, src_ref, off_ref = orc.permute_plan(idx, 0, 6, max_rows=len(src))
    assert np.array_equal(off, off_ref) and np.array_equal(rm, rm_ref)
    assert np.array_equal(src[: off[-1]], src_ref[: off[-1]])


def test_permute_plan_overflow_status(F):
    idx = np.zeros((64, 1), np.int32)
    rm, src, off, status = run_plan(F, idx, 0, 1, 16, max_rows=32)
    assert status == 1 and off[-1] == 64 and np.all(rm[32:] == -1) and np.all(rm[:32, 0] == np.arange(32))


def test_overflowed_plan_consumers_stay_in_bounds(F):
    """a plan whose padded total (64) exceeds max_rows (32) reports the true total in
    expert_offsets[E_loc] and status 1; the move and SwiGLU+quant that consume it clamp to their
    capacity.  Guard bytes right after every output buffer must stay untouched."""
    T, H, FF, mr = 64, 256, 128, 32
    idx = np.zeros((T, 1), np.int32)
    rm, src, off, status = run_plan(F, idx, 0, 1, 16, max_rows=mr)
    assert status == 1 and off[-1] == 64
    q_tok = torch.randint(0, 0x7E, (T, H), dtype=torch.uint8, device="cuda")
    s_tok = torch.randint(100, 140, (H // 128, T), dtype=torch.uint8, device="cuda")
    guard = 4096
    qbuf = torch.full((mr * H + guard,), 0xEE, dtype=torch.uint8, device="cuda")
    sbuf = torch.full(((H // 128) * mr + guard,), 0xEE, dtype=torch.uint8, device="cuda")
    q_out, s_out = qbuf[: mr * H].view(mr, H), sbuf[: (H // 128) * mr].view(H // 128, mr)
    F.fp8flow_permute_pad(q_tok, s_tok, dev(rm), dev(src), dev(off), q_out, s_out)
    h = synth.normal_bf16(mr, 2 * FF, 77).cuda()
    abuf = torch.full((mr * FF + guard,), 0xEE, dtype=torch.uint8, device="cuda")
    sab = torch.full(((FF // 128) * mr + guard,), 0xEE, dtype=torch.uint8, device="cuda")
    F.fp8flow_swiglu_quant(h, abuf[: mr * FF].view(mr, FF), sab[: (FF // 128) * mr].view(FF // 128, mr),
                           rows_dev=dev(off)[1:])
    torch.cuda.synchronize()
    for buf, n in ((qbuf, mr * H), (sbuf, (H // 128) * mr), (abuf, mr * FF), (sab, (FF // 128) * mr)):
        assert torch.all(buf[n:] == 0xEE), "write past the capacity"
    assert torch.equal(q_out, q_tok[:mr]) and torch.equal(s_out, s_tok[:, :mr])   # rows 0..31 = tokens 0..31


def run_move(F, q_tok, s_tok, rm, src, off, max_rows):
    T, H = q_tok.shape
    q_out = torch.full((max_rows, H), 0xEE, dtype=torch.uint8, device="cuda")
    s_out = torch.full((H // 128, max_rows), 0xEE, dtype=torch.uint8, device="cuda")
    F.fp8flow_permute_pad(dev(q_tok), dev(s_tok), dev(rm), dev(src), dev(off), q_out, s_out)
    torch.cuda.synchronize()
    return host(q_out), host(s_out)


@pytest.mark.parametrize("T,H,group,ngroups", [(16384, 7168, 3, 8), (1000, 1024, 0, 8), (16384, 7168, 0, 1)])
def test_permute_pad_parity(F, orc, T, H, group, ngroups):
    """EP8 shards and the whole DeepSeek-V3 layer on one GPU (ngroups 1: 256 local experts, every
    token fanned out to its 8 rows, ~133k padded rows)."""
    x = synth.activations_bf16(T, H, 500 + T)
    q_tok, s_tok = orc.quantize_rowwise_bf16(synth.bf16_bits(x))
    idx, _ = synth.routing(T, 501 + T)
    sh = synth.expert_shard(idx, torch.zeros(idx.shape), group, ngroups)
    q_recv = np.ascontiguousarray(q_tok[sh.recv_tokens])
    s_recv = np.ascontiguousarray(s_tok[:, sh.recv_tokens])
    rm, src, off = orc.permute_plan(sh.topk_idx, sh.expert_begin, sh.num_local_experts)
    max_rows = (len(src) + 15) // 16 * 16
    src_p = np.full(max_rows, -1, np.int32)
    src_p[: len(src)] = src
    qo, so = run_move(F, q_recv, s_recv, rm, src_p, off, max_rows)
    qo_ref, so_ref = orc.permute_pad(q_recv, s_recv, src_p, off, max_rows=max_rows)
    R = int(off[-1])
    assert np.array_equal(qo[:R], qo_ref[:R]) and np.array_equal(so[:, :R], so_ref[:, :R])
    assert np.all(qo[R:] == 0xEE)                                        # rows >= R untouched


# =========================================================================================== A4
@pytest.mark.parametrize("with_probs", [True, False])
@pytest.mark.parametrize("T,H,K,E_loc", [(2000, 7168, 8, 32), (300, 256, 4, 16), (64, 1024, 16, 64)])
def test_unpermute_parity(F, orc, T, H, K, E_loc, with_probs):
    idx, probs = synth.routing(T, 600 + T, num_experts=max(E_loc * 2, K * 2), top_k=K,
                               num_groups=4, topk_groups=4)
    rm, src, off = orc.permute_plan(idx.numpy(), 0, E_loc)
    R = int(off[-1])
    xb = synth.bf16_bits(synth.normal_bf16(max(R, 1), H, 601))
    p = probs.numpy() if with_probs else None
    y_ref = orc.unpermute(xb, rm, p)
    y = torch.empty(T, H, dtype=torch.bfloat16, device="cuda")
    F.fp8flow_unpermute_unpad(bf16_dev(xb), dev(rm), dev(p) if with_probs else None, y)
    torch.cuda.synchronize()
    assert np.array_equal(host(y.view(torch.int16)).view(np.uint16), y_ref)


# =========================================================================================== A5
def run_swiglu(F, h_bits, rows_dev=None, ld_s=None):
    rows, F2 = h_bits.shape
    ld_s = ld_s or ((rows + 15) // 16 * 16)
    q = torch.empty(rows, F2 // 2, dtype=torch.uint8, device="cuda")
    s = torch.full((F2 // 256, ld_s), 0xAB, dtype=torch.uint8, device="cuda")
    F.fp8flow_swiglu_quant(bf16_dev(h_bits), q, s, rows_dev=None if rows_dev is None else dev(rows_dev))
    torch.cuda.synchronize()
    return host(q), host(s)


def check_swiglu(q, s, q_ref, s_ref, rows):
    assert np.array_equal(s[:, :rows], s_ref[:, :rows])                  # identical scales
    d = e4m3_ulp_dist(q[:rows], q_ref[:rows])
    assert d.max(initial=0) <= 1
    assert np.mean(d > 0) <= 1e-4


@pytest.mark.parametrize("rows,ffn,sigma", [(256, 256, 1.5), (100, 2048, 1.5), (2048, 2048, 4.0),
                                            (16640, 2048, 1.5)])
def test_swiglu_quant_parity(F, orc, rows, ffn, sigma):
    hb = synth.bf16_bits(synth.normal_bf16(rows, 2 * ffn, 700 + rows, sigma=sigma))
    q, s = run_swiglu(F, hb)
    q_ref, s_ref = orc.swiglu_quant(hb, ld_s=s.shape[1])
    check_swiglu(q, s, q_ref, s_ref, rows)


def test_swiglu_quant_near_boundaries_and_wild(F, orc):
    """Tiles whose SwiGLU amax sits at 448*2^T within a few ulp, huge |a| (exp overflow range),
    tiny products (subnormal range), zeros and PAD rows."""
    rows, ffn = 64, 256
    rng = np.random.default_rng(5)
    a = rng.normal(0, 1.5, (rows, ffn)).astype(np.float32)
    b = rng.normal(0, 1.5, (rows, ffn)).astype(np.float32)
    # a = 20: silu(a) = a (1 - 2e-9); b chosen so that a*b lands near 448*2^T * (1 +- eps)
    for i in range(0, 32):
        T = int(rng.integers(-6, 6))
        a[i, 7] = 20.0
        b[i, 7] = 448.0 * 2.0 ** T / 20.0 * (1 + (i - 16) * 2.0 ** -8)
    a[40, :] = -100.0
    a[41, :] = 90.0
    a[42, :], b[42, :] = 1e-20, 1e-20
    a[43, :], b[43, :] = 0.0, 0.0
    h = np.concatenate([a, b], axis=1)
    hb = synth.bf16_bits(torch.from_numpy(h).to(torch.bfloat16))
    q, s = run_swiglu(F, hb)
    q_ref, s_ref = orc.swiglu_quant(hb, ld_s=s.shape[1])
    check_swiglu(q, s, q_ref, s_ref, rows)


def test_swiglu_quant_rows_dev(F, orc):
    rows_max, ffn, rows = 256, 512, 176
    hb = synth.bf16_bits(synth.normal_bf16(rows_max, 2 * ffn, 9, sigma=1.5))
    q, s = run_swiglu(F, hb, rows_dev=np.array([rows], np.int32))
    q_ref, s_ref = orc.swiglu_quant(hb[:rows], ld_s=s.shape[1])
    check_swiglu(q, s, q_ref, s_ref, rows)
    assert np.all(s[:, rows:] == 0xAB)


# =========================================================================================== checksum
def test_checksum_matches_oracle(F, orc):
    rng = np.random.default_rng(1)
    for n in (16, 1000 * 16, 12345 * 16 + 16):
        b = rng.integers(0, 256, n, dtype=np.uint8)
        out = torch.zeros(1, dtype=torch.int64, device="cuda")
        F.fp8flow_checksum64(dev(b), out)
        torch.cuda.synchronize()
        got = int(np.array(out.cpu().numpy()).view(np.uint64)[0])
        assert got == orc.checksum64(b)


# =========================================================================================== NEXT-1
def run_swiglu_bwd(F, h_bits, dA_bits, rows_dev=None):
    rows, F2 = h_bits.shape
    ld_s = (rows + 15) // 16 * 16
    q = torch.empty(rows, F2, dtype=torch.uint8, device="cuda")
    s = torch.full((F2 // 128, ld_s), 0xAB, dtype=torch.uint8, device="cuda")
    F.fp8flow_swiglu_bwd_quant(bf16_dev(h_bits), bf16_dev(dA_bits), q, s,
                               rows_dev=None if rows_dev is None else dev(rows_dev))
    torch.cuda.synchronize()
    return host(q), host(s)


@pytest.mark.parametrize("rows,ffn,sigma", [(64, 128, 1.5), (77, 384, 2.0), (100, 2048, 1.5), (2048, 2048, 3.0),
                                            (15872, 2048, 1.5)])
def test_swiglu_bwd_quant_parity(F, orc, rows, ffn, sigma):
    hb = synth.bf16_bits(synth.normal_bf16(rows, 2 * ffn, 800 + rows, sigma=sigma))
    db = synth.bf16_bits(synth.normal_bf16(rows, ffn, 801 + rows, sigma=0.5))
    q, s = run_swiglu_bwd(F, hb, db)
    q_ref, s_ref = orc.swiglu_bwd_quant(hb, db, ld_s=s.shape[1])
    check_swiglu(q, s, q_ref, s_ref, rows)


def test_swiglu_bwd_quant_adversarial(F, orc):
    """a at the root of silu' (~ -1.2785), whole tiles near it, tile maxima at 448*2^T, |a| > 64,
    tiny gradients, zero rows, and rows_dev."""
    rows, ffn = 64, 256
    rng = np.random.default_rng(31)
    a = rng.normal(0, 1.5, (rows, ffn)).astype(np.float32)
    b = rng.normal(0, 1.0, (rows, ffn)).astype(np.float32)
    g = rng.normal(0, 1.0, (rows, ffn)).astype(np.float32)
    a[0:8, :] = -1.2785 + rng.normal(0, 1e-3, (8, ffn))            # whole tiles at the root of silu'
    a[8:16, ::3] = -1.2785
    for i in range(16, 40):                                          # db tile maxima near 448*2^T
        T = int(rng.integers(-4, 4))
        a[i, 5] = 30.0
        g[i, 5] = 448.0 * 2.0 ** T / 30.0 * (1 + (i - 28) * 2.0 ** -9)
    a[40, :] = -80.0
    a[41, :] = 70.0
    g[42, :] = 1e-30
    a[43, :], b[43, :], g[43, :] = 0.0, 0.0, 0.0
    h = np.concatenate([a, b], axis=1)
    hb = synth.bf16_bits(torch.from_numpy(h).to(torch.bfloat16))
    dbits = synth.bf16_bits(torch.from_numpy(g).to(torch.bfloat16))
    q, s = run_swiglu_bwd(F, hb, dbits)
    q_ref, s_ref = orc.swiglu_bwd_quant(hb, dbits, ld_s=s.shape[1])
    check_swiglu(q, s, q_ref, s_ref, rows)
    q2, s2 = run_swiglu_bwd(F, hb, dbits, rows_dev=np.array([48], np.int32))
    check_swiglu(q2, s2, q_ref, s_ref, 48)
    assert np.all(s2[:, 48:] == 0xAB)


# ============================================================================ NEXT-1 dual output
def run_dual(F, inp, seg, swiglu=False, rows_dev=None):
    """Returns (q, s, qT, sT) of the dual-output kernel, outputs pre-filled with sentinels."""
    rows, in_cols = inp.shape
    cols = in_cols // 2 if swiglu else in_cols
    nseg = 1 if seg is None else len(seg) - 1
    ld_s = (rows + 15) // 16 * 16
    nbytes, ntiles = F.transpose_out_shapes(rows, cols, nseg)
    q = torch.full((rows, cols), 0xAB, dtype=torch.uint8, device="cuda")
    s = torch.full((cols // 128, ld_s), 0xAB, dtype=torch.uint8, device="cuda")
    qT = torch.full((max(nbytes, 16),), 0xCD, dtype=torch.uint8, device="cuda")
    sT = torch.full((ntiles, cols), 0xCD, dtype=torch.uint8, device="cuda")
    seg_t = None if seg is None else dev(np.asarray(seg, np.int32))
    if swiglu:
        F.fp8flow_swiglu_quant_dual(inp, q, s, qT, sT, seg_offsets=seg_t,
                                    rows_dev=None if rows_dev is None else dev(np.asarray([rows_dev], np.int32)))
    else:
        F.fp8flow_quantize_dual(inp, q, s, qT, sT, seg_offsets=seg_t)
    torch.cuda.synchronize()
    return host(q), host(s), host(qT), host(sT)


DUAL_SEGS = [None, [0, 16, 16, 160, 288, 304, 560, 576]]


@pytest.mark.parametrize("seg", DUAL_SEGS)
@pytest.mark.parametrize("cols", [128, 384, 7168])
def test_quantize_dual_parity(F, orc, seg, cols):
    """q, s bit-exact vs the oracle's A1; qT, sT bit-exact vs the oracle's A2 of that (R32)."""
    rows = 576 if seg is not None else 320
    x = synth.activations_bf16(rows, cols, 900 + cols)
    q, s, qT, sT = run_dual(F, x.cuda(), seg)
    q_ref, s_ref = orc.quantize_rowwise_bf16(synth.bf16_bits(x), ld_s=s.shape[1])
    assert np.array_equal(q, q_ref)
    assert np.array_equal(s[:, :rows], s_ref[:, :rows])
    qT_ref, sT_ref = orc.scaling_aware_transpose(q_ref, s_ref[:, :rows], seg)
    assert np.array_equal(qT[: qT_ref.size], qT_ref)
    assert np.array_equal(sT[: sT_ref.shape[0]], sT_ref)


def test_quantize_dual_equals_composition(F, orc):
    """Bit-identical to A1 followed by A2 on the device at the bench's X shape class."""
    seg = np.concatenate([[0], np.cumsum([512, 16, 0, 1040, 2528])]).astype(np.int32)
    rows, cols = int(seg[-1]), 7168
    x = synth.activations_bf16(rows, cols, 77).cuda()
    q, s, qT, sT = run_dual(F, x, seg)
    q1, s1 = run_quantize(F, x, ld_s=s.shape[1])
    qT1, sT1 = run_transpose(F, q1, s1[:, :rows], seg)
    assert np.array_equal(q, q1) and np.array_equal(s[:, :rows], s1[:, :rows])
    assert np.array_equal(qT, qT1) and np.array_equal(sT, sT1)


@pytest.mark.parametrize("seg,ffn", [(None, 256), ([0, 16, 16, 160, 288, 304, 560, 576], 384),
                                     ([0, 528, 1040, 1056, 2048], 2048)])
def test_swiglu_quant_dual_parity(F, orc, seg, ffn):
    """q, s at the A5 bar vs the oracle; qT, sT bit-exact vs the oracle's A2 of the kernel's own
    q, s (the composition semantics, R32)."""
    rows = 320 if seg is None else seg[-1]
    hb = synth.bf16_bits(synth.normal_bf16(rows, 2 * ffn, 950 + ffn, sigma=1.5))
    q, s, qT, sT = run_dual(F, bf16_dev(hb), seg, swiglu=True)
    q_ref, s_ref = orc.swiglu_quant(hb, ld_s=s.shape[1])
    check_swiglu(q, s, q_ref, s_ref, rows)
    qT_ref, sT_ref = orc.scaling_aware_transpose(q, s[:, :rows], seg)
    assert np.array_equal(qT[: qT_ref.size], qT_ref)
    assert np.array_equal(sT[: sT_ref.shape[0]], sT_ref)


def test_swiglu_quant_dual_equals_composition(F, orc):
    """Bit-identical to A5 then A2 on the device, with the rows given by the last offset (PAD rows
    of h beyond it are never read into the outputs) and the wild inputs of A5's edge test."""
    seg = np.concatenate([[0], np.cumsum([528, 0, 16, 1024, 144])]).astype(np.int32)
    rows_max, ffn = int(seg[-1]) + 64, 2048
    rng = np.random.default_rng(12)
    a = rng.normal(0, 1.5, (rows_max, ffn)).astype(np.float32)
    b = rng.normal(0, 1.5, (rows_max, ffn)).astype(np.float32)
    a[5, :7] = [-70.0, -100.0, 90.0, -88.5, 0.0, -0.0, 1e-30]
    b[9, :] = 0.0
    h = torch.from_numpy(np.concatenate([a, b], 1)).to(torch.bfloat16).cuda()
    rows = int(seg[-1])
    q, s, qT, sT = run_dual(F, h, seg, swiglu=True)
    q1 = torch.full((rows_max, ffn), 0xAB, dtype=torch.uint8, device="cuda")
    s1 = torch.full((ffn // 128, s.shape[1]), 0xAB, dtype=torch.uint8, device="cuda")
    F.fp8flow_swiglu_quant(h, q1, s1, rows_dev=dev(np.asarray([rows], np.int32)))
    torch.cuda.synchronize()
    q1, s1 = host(q1), host(s1)
    assert np.array_equal(q[:rows], q1[:rows]) and np.array_equal(s[:, :rows], s1[:, :rows])
    qT1, sT1 = run_transpose(F, q1[:rows], s1[:, :rows], seg)
    assert np.array_equal(qT[: qT1.size], qT1) and np.array_equal(sT[: sT1.shape[0]], sT1)


# ======================================================================= CUDA-graph capturability
def test_all_ops_capture_into_a_cuda_graph(F, orc):
    """The header's promise: every call is asynchronous, never synchronises and keeps
    data-dependent sizes on the device, so a whole step captures into a CUDA graph; replays give
    the eager results bit for bit (and the oracle's)."""
    T, H, FF, K, E_loc = 96, 256, 256, 4, 8
    x = synth.activations_bf16(T, H, 11).cuda()
    g = torch.Generator().manual_seed(12)
    idx = torch.stack([torch.randperm(16, generator=g)[:K] for _ in range(T)]).to(torch.int32).cuda()
    probs = torch.rand(T, K, generator=g).cuda()
    max_rows = F.permute_max_rows(T, K, E_loc)
    h = synth.normal_bf16(max_rows, 2 * FF, 13, sigma=1.5).cuda()
    y_in = synth.normal_bf16(max_rows, H, 14).cuda()
    ws = torch.empty(F.fp8flow_permute_workspace_bytes(T, K, E_loc), dtype=torch.uint8, device="cuda")
    bufs = {
        "q": torch.empty(T, H, dtype=torch.uint8, device="cuda"), "s": torch.empty(H // 128, 96, dtype=torch.uint8, device="cuda"),
        "row_map": torch.empty(T, K, dtype=torch.int32, device="cuda"),
        "src": torch.empty(max_rows, dtype=torch.int32, device="cuda"),
        "off": torch.empty(E_loc + 1, dtype=torch.int32, device="cuda"),
        "q_out": torch.empty(max_rows, H, dtype=torch.uint8, device="cuda"),
        "s_out": torch.empty(H // 128, max_rows, dtype=torch.uint8, device="cuda"),
        "qa": torch.empty(max_rows, FF, dtype=torch.uint8, device="cuda"),
        "sa": torch.empty(FF // 128, max_rows, dtype=torch.uint8, device="cuda"),
        "y": torch.empty(T, H, dtype=torch.bfloat16, device="cuda"),
        "qT": torch.empty(max_rows * H, dtype=torch.uint8, device="cuda"),
        "sT": torch.empty(max_rows // 128 + E_loc, H, dtype=torch.uint8, device="cuda"),
    }

    def step():
        b = bufs
        F.fp8flow_quantize_rowwise(x, b["q"], b["s"])
        F.fp8flow_permute_plan(idx, 0, E_loc, 16, b["row_map"], b["src"], b["off"], ws)
        F.fp8flow_permute_pad(b["q"], b["s"], b["row_map"], b["src"], b["off"], b["q_out"], b["s_out"])
        F.fp8flow_swiglu_quant(h, b["qa"], b["sa"], rows_dev=b["off"][E_loc:])
        F.fp8flow_unpermute_unpad(y_in, b["row_map"], probs, b["y"])
        F.fp8flow_scaling_aware_transpose(b["q_out"], b["s_out"], b["qT"], b["sT"], seg_offsets=b["off"])

    step()
    torch.cuda.synchronize()
    eager = {k: v.clone() for k, v in bufs.items()}
    for v in bufs.values():
        v.zero_()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    for _ in range(2):
        graph.replay()
    torch.cuda.synchronize()
    R = int(eager["off"][-1])
    for k in ("q", "s", "row_map", "off", "y"):
        assert torch.equal(bufs[k], eager[k]), k
    assert torch.equal(bufs["src"][:R], eager["src"][:R])
    assert torch.equal(bufs["q_out"][:R], eager["q_out"][:R]) and torch.equal(bufs["s_out"][:, :R], eager["s_out"][:, :R])
    assert torch.equal(bufs["qa"][:R], eager["qa"][:R]) and torch.equal(bufs["sa"][:, :R], eager["sa"][:, :R])
    assert torch.equal(bufs["qT"][: R * H], eager["qT"][: R * H])
    q_ref, s_ref = orc.quantize_rowwise_bf16(synth.bf16_bits(x.cpu()), ld_s=96)
    assert np.array_equal(host(bufs["q"]), q_ref)
