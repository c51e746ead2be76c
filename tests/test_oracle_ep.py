"""Pins for the oracle's NEXT-3 expert-parallel ops (R34):
dispatch + fused permute/pad across n ranks (oracle.dispatch_permute_pad) and combine
(oracle.combine / orc_combine).

What pins them, independently of their own code:
* partition: over all ranks, every routing pair (token, k) lands in exactly one rank's plan, the
  rank that owns expert topk[token][k] (P:245 dispatch -> permutation), and every dispatched row
  holds the exact bytes (codes and the 1x128 scale bytes) of its source token -- checked here by
  numpy indexing, not by the oracle;
* n = 1 reduces to A3 / A4 on one device (special case);
* combine with one-hot gates returns the selected expert's row bit for bit;
* combine(dispatch(Q)) with an identity "expert" (exact E4M3 -> BF16 decode by torch) and K a
  power of two equals K * dequant(Q) exactly (all partial sums exact in fp32), for any rank count.
"""
import numpy as np
import pytest
import torch

import synth


def _bits_f64(b):
    return torch.from_numpy(np.ascontiguousarray(b).view(np.int16)).view(torch.bfloat16).to(torch.float64).numpy()


def _f64_bits(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def _ranks(n, tpr, H, E, K, seed, groups=4, topk_groups=2):
    """n ranks' row-wise FP8 tokens: random code bytes (no NaN) and scale bytes, routing."""
    g = torch.Generator().manual_seed(seed)
    qs, ss, ts, ps = [], [], [], []
    for r in range(n):
        q = torch.randint(0, 256, (tpr, H), generator=g, dtype=torch.int32).numpy().astype(np.uint8)
        q[(q & 0x7F) == 0x7F] = 0x00                                             # no NaN codes
        s = torch.randint(100, 150, (H // 128, tpr), generator=g, dtype=torch.int32).numpy().astype(np.uint8)
        idx, p = synth.routing(tpr, seed * 31 + r, num_experts=E, top_k=K, num_groups=groups,
                               topk_groups=topk_groups)
        qs.append(q), ss.append(s), ts.append(idx.numpy()), ps.append(p.numpy())
    return qs, ss, ts, ps


@pytest.mark.parametrize("n", [1, 2, 4])
def test_dispatch_partition_and_row_bytes(orc, n):
    tpr, H, E, K = 40, 256, 16, 4
    qs, ss, ts, _ = _ranks(n, tpr, H, E, K, 11 + n)
    topk_all = np.concatenate(ts)
    q_all, s_all = np.concatenate(qs), np.concatenate(ss, axis=1)
    owner = np.full(topk_all.shape, -1)
    for g in range(n):
        qo, so, rm, src, off = orc.dispatch_permute_pad(qs, ss, ts, g, E, align=16)
        e0, e_per = g * E // n, E // n
        local = (topk_all >= e0) & (topk_all < e0 + e_per)
        assert np.array_equal(rm >= 0, local)
        assert np.all(owner[local] == -1)
        owner[local] = g
        assert np.all(np.diff(off) % 16 == 0)
        for (t, k) in zip(*np.nonzero(local)):
            r = rm[t, k]
            assert src[r] == t
            assert np.array_equal(qo[r], q_all[t])                               # codes travel as is
            assert np.array_equal(so[:, r], s_all[:, t])                         # with their scales
            assert off[topk_all[t, k] - e0] <= r < off[topk_all[t, k] - e0 + 1]
        pad = [r for r in range(off[-1]) if src[r] < 0]
        assert np.all(qo[pad] == 0) and np.all(so[:, pad] == 0)
    assert np.all(owner >= 0)                                                    # every pair exactly once


def test_dispatch_one_rank_is_a3(orc):
    qs, ss, ts, _ = _ranks(1, 64, 256, 16, 4, 3)
    qo, so, rm, src, off = orc.dispatch_permute_pad(qs, ss, ts, 0, 16)
    rm1, src1, off1 = orc.permute_plan(ts[0], 0, 16)
    qo1, so1 = orc.permute_pad(qs[0], ss[0], src1, off1)
    assert np.array_equal(rm, rm1) and np.array_equal(off, off1)
    assert np.array_equal(qo, qo1) and np.array_equal(so, so1)


def _decode_rows(q, s):
    """Exact dequantization by torch's own E4M3 cast (library routine) times 2^(s-127)."""
    v = torch.from_numpy(q).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    return v * np.exp2(np.repeat(s.T.astype(np.float64) - 127.0, 128, axis=1))


@pytest.mark.parametrize("n", [1, 2, 4])
def test_combine_of_dispatch_is_K_times_dequant(orc, n):
    tpr, H, E, K = 32, 256, 16, 4
    qs, ss, ts, _ = _ranks(n, tpr, H, E, K, 21 + n)
    xs, rms = [], []
    for g in range(n):
        qo, so, rm, src, off = orc.dispatch_permute_pad(qs, ss, ts, g, E)
        # identity expert: x = dequant(row) in BF16 (exact: 3 mantissa bits, exponent in range)
        xs.append(_f64_bits(_decode_rows(qo, so)))
        rms.append(rm)
    for g in range(n):
        y = orc.combine(xs, rms, ts[g], E // n, token_begin=g * tpr)
        assert np.array_equal(_bits_f64(y), K * _decode_rows(qs[g], ss[g]))


def test_combine_one_rank_is_a4_and_one_hot_gates(orc):
    tpr, H, E, K = 48, 256, 8, 2
    _, _, ts, ps = _ranks(1, tpr, H, E, K, 5, groups=2, topk_groups=1)
    rm, src, off = orc.permute_plan(ts[0], 0, E)
    x = synth.bf16_bits(synth.normal_bf16(len(src), H, 9))
    y = orc.combine([x], [rm], ts[0], E, probs=ps[0])
    assert np.array_equal(y, orc.unpermute(x, rm, ps[0]))
    onehot = np.zeros_like(ps[0])
    onehot[:, 1] = 1.0
    y1 = orc.combine([x], [rm], ts[0], E, probs=onehot)
    assert np.array_equal(y1, x[rm[:, 1]])


def test_combine_two_ranks_equals_a4_over_concatenation(orc):
    """Two ranks' expert outputs stacked (rank 1's rows offset by rank 0's row count) form one
    device's expert-major buffer: combine must equal A4 on it for every gate set."""
    n, tpr, H, E, K = 2, 24, 256, 16, 4
    qs, ss, ts, ps = _ranks(n, tpr, H, E, K, 33)
    plans = [orc.dispatch_permute_pad(qs, ss, ts, g, E)[2:] for g in range(n)]
    xs = [synth.bf16_bits(synth.normal_bf16(len(p[1]), H, 40 + g)) for g, p in enumerate(plans)]
    base = [0, len(plans[0][1])]
    rm_glob = np.where(plans[0][0] >= 0, plans[0][0], plans[1][0] + base[1]).astype(np.int32)
    x_cat = np.concatenate(xs)
    for g in range(n):
        y = orc.combine(xs, [p[0] for p in plans], ts[g], E // n, probs=ps[g], token_begin=g * tpr)
        ref = orc.unpermute(x_cat, rm_glob[g * tpr:(g + 1) * tpr], ps[g])
        assert np.array_equal(y, ref)


def test_combine_k_order_half_ulp_tie(orc):
    """R34 / R21: combine sums a token's K terms in fp32 in k order across the ranks that hold
    them (no per-rank partial sums).  Same hand-built terms as the A4 pin
    (test_unpermute_k_order_half_ulp_tie): 1, 2^-8, 2^-24, 2^-24 in k order -> BF16 0x3F80;
    the reversed listing -> 0x3F81.  Two ranks, two experts each; each rank holds two of the
    terms, so the order crosses ranks."""
    H = 128
    one, e8, e24 = 0x3F80, 0x3B80, 0x3380
    # rank 0 holds experts 0, 1; rank 1 holds experts 2, 3.  Rows: x_0 = [1, 2^-24], x_1 = [2^-8, 2^-24]
    x0 = np.repeat(np.array([one, e24], np.uint16)[:, None], H, axis=1)
    x1 = np.repeat(np.array([e8, e24], np.uint16)[:, None], H, axis=1)
    # token 0: experts [0, 2, 1, 3] -> terms 1, 2^-8, 2^-24, 2^-24; token 1: the reverse listing
    topk = np.array([[0, 2, 1, 3], [3, 1, 2, 0]], np.int32)
    rm0 = np.array([[0, -1, 1, -1], [-1, 1, -1, 0]], np.int32)     # rows on rank 0 (experts 0, 1)
    rm1 = np.array([[-1, 0, -1, 1], [1, -1, 0, -1]], np.int32)     # rows on rank 1 (experts 2, 3)
    for probs in (None, np.ones((2, 4), np.float32)):
        y = orc.combine([x0, x1], [rm0, rm1], topk, 2, probs=probs)
        assert np.all(y[0] == one) and np.all(y[1] == 0x3F81), (probs is None, y[:, 0])
