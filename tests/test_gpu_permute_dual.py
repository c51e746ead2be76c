"""GPU parity of the A3 move fused with A2 (fp8flow_permute_pad_dual, NEXT-1 dual output, DESIGN.md
R37) through the C ABI, against the CPU oracle's composition permute_pad -> scaling_aware_transpose
(Algorithm 1) on the same seeded inputs: every output byte identical.
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

    fp8flow.fp8flow_device_check()
    return fp8flow


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_dual(F, q_tok, s_tok, src_p, off, max_rows, fill=0xEE):
    T, H = q_tok.shape
    E_loc = len(off) - 1
    q_out = torch.full((max_rows, H), fill, dtype=torch.uint8, device="cuda")
    s_out = torch.full((H // 128, max_rows), fill, dtype=torch.uint8, device="cuda")
    nbytes, ntiles = F.transpose_out_shapes(max_rows, H, E_loc)
    qT = torch.full((nbytes,), fill, dtype=torch.uint8, device="cuda")
    sT = torch.full((ntiles, H), fill, dtype=torch.uint8, device="cuda")
    F.fp8flow_permute_pad_dual(dev(q_tok), dev(s_tok), dev(src_p), dev(off), q_out, s_out, qT, sT)
    torch.cuda.synchronize()
    return q_out.cpu().numpy(), s_out.cpu().numpy(), qT.cpu().numpy(), sT.cpu().numpy()


def pad_ld(s_tok):
    """Scales with the row pitch rounded up to 16 bytes (the fused kernel reads 4-byte words)."""
    k, T = s_tok.shape
    out = np.zeros((k, (T + 15) // 16 * 16), np.uint8)
    out[:, :T] = s_tok
    return out


def check(F, orc, q_tok, s_tok, topk, e0, E_loc, align=16):
    s_tok = pad_ld(s_tok)
    rm, src, off = orc.permute_plan(topk, e0, E_loc, align=align)
    max_rows = (len(src) + 15) // 16 * 16
    src_p = np.full(max_rows, -1, np.int32)
    src_p[: len(src)] = src
    R = int(off[-1])
    qo, so, qT, sT = run_dual(F, q_tok, s_tok, src_p, off, max_rows)
    qo_ref, so_ref = orc.permute_pad(q_tok, s_tok, src_p, off, max_rows=max_rows)
    qT_ref, sT_ref = orc.scaling_aware_transpose(qo_ref[:R], so_ref, off)
    assert np.array_equal(qo[:R], qo_ref[:R]), np.argwhere(qo[:R] != qo_ref[:R])[:5]
    assert np.array_equal(so[:, :R], so_ref[:, :R])
    assert np.all(qo[R:] == 0xEE) and np.all(so[:, R:] == 0xEE)      # rows >= R untouched
    assert np.array_equal(qT[: qT_ref.size], qT_ref), np.argwhere(qT[: qT_ref.size] != qT_ref)[:5]
    assert np.array_equal(sT[: sT_ref.shape[0]], sT_ref)
    return R


@pytest.mark.parametrize("T,H,group,ngroups", [(1000, 1024, 0, 8), (1000, 1280, 2, 8), (3000, 2048, 5, 8),
                                               (16384, 7168, 3, 8)])
def test_permute_pad_dual_parity(F, orc, T, H, group, ngroups):
    """EP8 shards of the DeepSeek-V3 routing (ragged experts, PAD rows in every expert's last block)."""
    x = synth.activations_bf16(T, H, 700 + T)
    q, s = orc.quantize_rowwise_bf16(synth.bf16_bits(x))
    idx, _ = synth.routing(T, 701 + T)
    sh = synth.expert_shard(idx, torch.zeros(idx.shape), group, ngroups)
    q_recv = np.ascontiguousarray(q[sh.recv_tokens])
    s_recv = np.ascontiguousarray(s[:, sh.recv_tokens])
    check(F, orc, q_recv, s_recv, sh.topk_idx, sh.expert_begin, sh.num_local_experts)


def test_permute_pad_dual_whole_layer(F, orc):
    """The whole layer on one GPU: 16384 tokens, 256 local experts, ~133k padded rows."""
    T, H = 16384, 7168
    x = synth.activations_bf16(T, H, 710)
    q, s = orc.quantize_rowwise_bf16(synth.bf16_bits(x))
    idx, _ = synth.routing(T, 711)
    R = check(F, orc, q, s, idx.numpy(), 0, 256)
    assert R > 130000


def test_permute_pad_dual_constructed_codes_and_scales(F, orc):
    """Every code (NaN codes included) and row scales spread over 40 binades, so the shift hits
    every k, the subnormal re-rounding and the flush to +-0 (R7, R10, R26); tiny experts (one token:
    15 PAD rows), empty experts, and experts longer than one 128-row block."""
    rng = np.random.default_rng(9)
    T, H, E = 700, 512, 24
    q_tok = rng.integers(0, 256, (T, H), dtype=np.uint8)
    s_tok = rng.integers(90, 131, (H // 128, T), dtype=np.uint8)
    s_tok[:, ::7] = 0                                               # scale byte 0 rows
    topk = np.stack([rng.permutation(E - 4)[:3] for _ in range(T)]).astype(np.int32)
    topk[0] = [E - 1, E - 3, 0]                                     # experts E-1, E-3: one token each
    check(F, orc, q_tok, s_tok, topk, 0, E)                         # E-4, E-2: empty


def test_permute_pad_dual_equals_two_launches(F, orc):
    """Same bytes as fp8flow_permute_pad followed by fp8flow_scaling_aware_transpose (the unfused
    route the fusion replaces), including the sT rows of every expert."""
    T, H = 2048, 7168
    x = synth.activations_bf16(T, H, 720)
    q, s = orc.quantize_rowwise_bf16(synth.bf16_bits(x))
    idx, _ = synth.routing(T, 721)
    sh = synth.expert_shard(idx, torch.zeros(idx.shape), 1, 8)
    q_recv = np.ascontiguousarray(q[sh.recv_tokens])
    s_recv = pad_ld(s[:, sh.recv_tokens])
    rm, src, off = orc.permute_plan(sh.topk_idx, sh.expert_begin, sh.num_local_experts)
    max_rows = (len(src) + 15) // 16 * 16
    src_p = np.full(max_rows, -1, np.int32)
    src_p[: len(src)] = src
    qo, so, qT, sT = run_dual(F, q_recv, s_recv, src_p, off, max_rows)
    q_out = torch.full((max_rows, H), 0xEE, dtype=torch.uint8, device="cuda")
    s_out = torch.full((H // 128, max_rows), 0xEE, dtype=torch.uint8, device="cuda")
    F.fp8flow_permute_pad(dev(q_recv), dev(s_recv), dev(rm), dev(src_p), dev(off), q_out, s_out)
    nbytes, ntiles = F.transpose_out_shapes(max_rows, H, len(off) - 1)
    qT2 = torch.full((nbytes,), 0xEE, dtype=torch.uint8, device="cuda")
    sT2 = torch.full((ntiles, H), 0xEE, dtype=torch.uint8, device="cuda")
    F.fp8flow_scaling_aware_transpose(q_out, s_out, qT2, sT2, seg_offsets=dev(off))
    torch.cuda.synchronize()
    assert np.array_equal(qo, q_out.cpu().numpy()) and np.array_equal(so, s_out.cpu().numpy())
    assert np.array_equal(qT, qT2.cpu().numpy()) and np.array_equal(sT, sT2.cpu().numpy())


def test_permute_pad_dual_overflowed_plan_stays_in_bounds(F):
    """An overflowed plan (64 padded rows, capacity 32) reports its true total; the fused kernel
    clamps the expert offsets to max_rows: rows 0..31 = tokens 0..31 and nothing past any buffer."""
    T, H, mr = 64, 256, 32
    q_tok = torch.randint(0, 0x7E, (T, H), dtype=torch.uint8, device="cuda")
    s_tok = torch.randint(100, 140, (H // 128, T), dtype=torch.uint8, device="cuda")
    src = torch.arange(mr, dtype=torch.int32, device="cuda")
    off = torch.tensor([0, 64], dtype=torch.int32, device="cuda")
    guard = 4096
    bufs = [torch.full((n + guard,), 0xEE, dtype=torch.uint8, device="cuda")
            for n in (mr * H, (H // 128) * mr, mr * H, (mr // 128 + 1) * H)]
    q_out, s_out = bufs[0][: mr * H].view(mr, H), bufs[1][: (H // 128) * mr].view(H // 128, mr)
    qT, sT = bufs[2][: mr * H], bufs[3][: (mr // 128 + 1) * H].view(-1, H)
    F.fp8flow_permute_pad_dual(q_tok, s_tok, src, off, q_out, s_out, qT, sT)
    torch.cuda.synchronize()
    for b, n in zip(bufs, (mr * H, (H // 128) * mr, mr * H, (mr // 128 + 1) * H)):
        assert torch.all(b[n:] == 0xEE), "write past the capacity"
    assert torch.equal(q_out, q_tok[:mr]) and torch.equal(s_out, s_tok[:, :mr])


def test_permute_pad_dual_zero_tokens_is_noop(F):
    q_tok = torch.empty(0, 256, dtype=torch.uint8, device="cuda")
    s_tok = torch.empty(2, 0, dtype=torch.uint8, device="cuda")
    src = torch.full((16,), -1, dtype=torch.int32, device="cuda")
    off = torch.zeros(5, dtype=torch.int32, device="cuda")
    q_out = torch.full((16, 256), 0xEE, dtype=torch.uint8, device="cuda")
    s_out = torch.full((2, 16), 0xEE, dtype=torch.uint8, device="cuda")
    qT = torch.full((16 * 256,), 0xEE, dtype=torch.uint8, device="cuda")
    sT = torch.full((5, 256), 0xEE, dtype=torch.uint8, device="cuda")
    F.fp8flow_permute_pad_dual(q_tok, s_tok, src, off, q_out, s_out, qT, sT)
    torch.cuda.synchronize()
    assert torch.all(q_out == 0xEE) and torch.all(qT == 0xEE)


@pytest.mark.parametrize("T,H,E,K,align", [(50, 128, 1024, 2, 16), (300, 384, 7, 3, 32), (1, 256, 4, 1, 16),
                                           (129, 1152, 2, 2, 16)])
def test_permute_pad_dual_edge_shapes(F, orc, T, H, E, K, align):
    """One column block (H = 128), 1024 local experts (most empty: the largest segment table),
    align 32, a single token (one expert of 16 rows, 15 of them PAD), an expert of 129 + PAD rows
    (a full block and a 16-row partial one) with an odd number of column blocks."""
    rng = np.random.default_rng(T + H)
    q_tok = rng.integers(0, 256, (T, H), dtype=np.uint8)
    s_tok = rng.integers(100, 135, (H // 128, T), dtype=np.uint8)
    topk = np.stack([rng.permutation(E)[:K] for _ in range(T)]).astype(np.int32)
    check(F, orc, q_tok, s_tok, topk, 0, E, align=align)
