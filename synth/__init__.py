"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no quantization, no scales, no transpose,
no permutation plan): it only draws random numbers with ``torch.Generator`` on the CPU, so the
CUDA path and the oracle see byte-identical inputs.  Input recipe:

* activations  x[t, h] = g_t * z[t, h] * c_h,  z ~ N(0, 1),  per-token gain g_t = exp(N(0, 1)),
  1 % of the hidden channels (a fixed, seeded set) amplified by c_h = 20 (outlier channels),
  rounded to BF16.  Shape of DeepSeek-V3 MoE inputs: hidden 7168 ("tensor shapes ...
  reflect ... DeepSeek V2-Lite, V2, and V3").
* routing      per-expert bias b_e ~ N(0, 1) (skewed load), score[t, e] = b_e + Gumbel(0, 1);
  DeepSeek-V3 group-limited top-k: 8 groups of 32 experts, keep the 4 groups with the largest
  sum of their top-2 scores, then the top-8 distinct experts; gate probabilities = softmax over
  the 8 selected scores (fp32).  Gives skewed, ragged per-expert token counts.
* fc1 output   h ~ N(0, 1.5^2) in BF16, shape [rows, 2F] (F = 2048 for DeepSeek-V3).
* fc2 output   y ~ N(0, 1) in BF16, shape [rows, 7168].
"""
from __future__ import annotations

import dataclasses

import numpy as np
import torch

BASE_SEED = 2511023020

# DeepSeek-V3 MoE dimensions (BASELINE.json configs)
HIDDEN = 7168
FFN = 2048
NUM_EXPERTS = 256
TOP_K = 8
NUM_GROUPS = 8
TOPK_GROUPS = 4
ALIGN = 16


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed) & 0xFFFFFFFFFFFFFFFF)
    return g


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    """BF16 tensor -> numpy uint16 bit patterns (no arithmetic)."""
    assert t.dtype == torch.bfloat16
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


def activations_bf16(rows: int, cols: int, seed: int, outlier_frac: float = 0.01, outlier_gain: float = 20.0,
                     gain_sigma: float = 1.0) -> torch.Tensor:
    g = _gen(seed)
    z = torch.randn(rows, cols, generator=g, dtype=torch.float32)
    gain = torch.exp(torch.randn(rows, 1, generator=g, dtype=torch.float32) * gain_sigma)
    n_out = int(round(outlier_frac * cols))
    ch = torch.ones(1, cols, dtype=torch.float32)
    if n_out > 0:
        idx = torch.randperm(cols, generator=g)[:n_out]
        ch[0, idx] = outlier_gain
    return (z * gain * ch).to(torch.bfloat16)


def activations_bf16_device(rows: int, cols: int, seed: int, device, outlier_frac: float = 0.01,
                            outlier_gain: float = 20.0, gain_sigma: float = 1.0) -> torch.Tensor:
    """Same recipe as activations_bf16, drawn on the device (Philox) for the large bandwidth sweep."""
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & 0xFFFFFFFFFFFFFFFF)
    z = torch.randn(rows, cols, generator=g, device=device, dtype=torch.float32)
    gain = torch.exp(torch.randn(rows, 1, generator=g, device=device, dtype=torch.float32) * gain_sigma)
    n_out = int(round(outlier_frac * cols))
    ch = torch.ones(1, cols, dtype=torch.float32, device=device)
    if n_out > 0:
        idx = torch.randperm(cols, generator=g, device=device)[:n_out]
        ch[0, idx] = outlier_gain
    return (z.mul_(gain).mul_(ch)).to(torch.bfloat16)


def normal_bf16_device(rows: int, cols: int, seed: int, device, sigma: float = 1.0) -> torch.Tensor:
    """N(0, sigma^2) in BF16 drawn on the device (Philox) for large bench-only buffers."""
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & 0xFFFFFFFFFFFFFFFF)
    return (torch.randn(rows, cols, generator=g, device=device, dtype=torch.float32) * sigma).to(torch.bfloat16)


def normal_bf16(rows: int, cols: int, seed: int, sigma: float = 1.0) -> torch.Tensor:
    g = _gen(seed)
    return (torch.randn(rows, cols, generator=g, dtype=torch.float32) * sigma).to(torch.bfloat16)


def routing(num_tokens: int, seed: int, num_experts: int = NUM_EXPERTS, top_k: int = TOP_K,
            num_groups: int = NUM_GROUPS, topk_groups: int = TOPK_GROUPS):
    """Returns (topk_idx int32 [T, K], probs float32 [T, K]); experts distinct per token."""
    g = _gen(seed)
    bias = torch.randn(num_experts, generator=g, dtype=torch.float64)
    u = torch.rand(num_tokens, num_experts, generator=g, dtype=torch.float64).clamp_(1e-12, 1 - 1e-12)
    score = bias[None, :] - torch.log(-torch.log(u))
    per_group = num_experts // num_groups
    gs = score.view(num_tokens, num_groups, per_group).topk(min(2, per_group), dim=-1).values.sum(-1)
    keep = gs.topk(topk_groups, dim=-1).indices
    mask = torch.full((num_tokens, num_groups), float("-inf"), dtype=torch.float64)
    mask.scatter_(1, keep, 0.0)
    masked = score + mask.repeat_interleave(per_group, dim=1)
    top = masked.topk(top_k, dim=-1)
    probs = torch.softmax(top.values, dim=-1).to(torch.float32)
    return top.indices.to(torch.int32).contiguous(), probs.contiguous()


@dataclasses.dataclass
class ExpertShard:
    """What an expert-parallel rank holds after dispatch (constructed, not communicated):
    the received tokens (those with >= 1 expert in the rank's group) and their routing rows."""
    group: int
    expert_begin: int
    num_local_experts: int
    recv_tokens: np.ndarray      # int64 [T_recv] indices into the global token batch
    topk_idx: np.ndarray         # int32 [T_recv, K] (global expert ids)
    probs: np.ndarray            # float32 [T_recv, K]


def expert_shard(topk_idx: torch.Tensor, probs: torch.Tensor, group: int, num_groups: int,
                 num_experts: int = NUM_EXPERTS) -> ExpertShard:
    per = num_experts // num_groups
    return expert_range_shard(topk_idx, probs, group * per, per, group)


def expert_range_shard(topk_idx: torch.Tensor, probs: torch.Tensor, e0: int, per: int, group: int = -1) -> ExpertShard:
    """The tokens routed to >= 1 expert of [e0, e0 + per) and their routing rows (a selection)."""
    idx = topk_idx.numpy()
    local = (idx >= e0) & (idx < e0 + per)
    recv = np.nonzero(local.any(axis=1))[0]
    return ExpertShard(group, e0, per, recv.astype(np.int64), np.ascontiguousarray(idx[recv]),
                       np.ascontiguousarray(probs.numpy()[recv]))
