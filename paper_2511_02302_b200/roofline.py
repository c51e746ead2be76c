"""Algorithmic byte counts per launch of each hot-path op.

These are the bytes the method must move (inputs read once, outputs written once), not what a
particular kernel happens to move; achieved GB/s = these bytes / measured kernel time, and the
roofline fraction divides by the measured HBM copy bandwidth (MEASURED_PEAKS.json).
Scales are UE8M0: one byte per 128 elements.
"""
from __future__ import annotations

import json
import os


def quantize_bytes(rows: int, cols: int) -> int:
    """A1: BF16 read (2 B) + E4M3 write (1 B) + one scale byte per 1x128 tile."""
    return rows * cols * 3 + rows * (cols // 128)


def transpose_bytes(seg_lengths, cols: int) -> int:
    """A2: codes + row scales read for the rows inside segments, codes written once, one output
    scale byte per (128-row block, column) of each segment."""
    m = sum(seg_lengths)
    blocks = sum((x + 127) // 128 for x in seg_lengths)
    return m * cols + m * (cols // 128) + m * cols + blocks * cols


def naive_transpose_actual_bytes(seg_lengths, cols: int) -> int:
    """The comparator's own traffic: dequant (1 + 1/128 -> 2), BF16 transpose (2 -> 2),
    column-wise quantize (2 -> 1 + scales)."""
    m = sum(seg_lengths)
    blocks = sum((x + 127) // 128 for x in seg_lengths)
    return m * cols * (1 + 2) + m * (cols // 128) + m * cols * (2 + 2) + m * cols * (2 + 1) + blocks * cols


def permute_plan_bytes(num_tokens: int, top_k: int, padded_rows: int) -> int:
    """A3 plan: topk_idx read, row_map written, src_of_row written (int32 each)."""
    return num_tokens * top_k * 4 * 2 + padded_rows * 4


def permute_move_bytes(unique_src_rows: int, padded_rows: int, hidden: int) -> int:
    """A3 move: each source token's codes + scales read once, every output row (incl. PAD) written,
    src_of_row read."""
    row = hidden + hidden // 128
    return unique_src_rows * row + padded_rows * row + padded_rows * 4


def unpermute_bytes(valid_rows: int, num_tokens: int, top_k: int, hidden: int, with_probs: bool = True) -> int:
    """A4: every non-PAD BF16 row read once, every token's BF16 output written, row_map (+ probs)."""
    return valid_rows * hidden * 2 + num_tokens * hidden * 2 + num_tokens * top_k * (4 + (4 if with_probs else 0))


def swiglu_quant_bytes(rows: int, ffn: int) -> int:
    """A5: BF16 [rows, 2F] read, E4M3 [rows, F] written, one scale byte per 1x128 output tile."""
    return rows * (4 * ffn + ffn + ffn // 128)


def swiglu_bwd_quant_bytes(rows: int, ffn: int) -> int:
    """NEXT-1: BF16 h [rows, 2F] and dA [rows, F] read, E4M3 dH [rows, 2F] written, one scale byte
    per 1x128 output tile (4.008 B per output element)."""
    return rows * (4 * ffn + 2 * ffn + 2 * ffn + 2 * ffn // 128)


def quantize_dual_bytes(seg_lengths, cols: int) -> int:
    """NEXT-1 dual A1: BF16 read once, row-wise codes + scales and column-wise codes + block scales
    written once."""
    m = sum(seg_lengths)
    blocks = sum((x + 127) // 128 for x in seg_lengths)
    return m * cols * (2 + 1 + 1) + m * (cols // 128) + blocks * cols


def swiglu_quant_dual_bytes(seg_lengths, ffn: int) -> int:
    """NEXT-1 dual A5: BF16 h [m, 2F] read once, row-wise and column-wise codes + scales written."""
    m = sum(seg_lengths)
    blocks = sum((x + 127) // 128 for x in seg_lengths)
    return m * (4 * ffn + ffn + ffn) + m * (ffn // 128) + blocks * ffn


def permute_dual_bytes(unique_src_rows: int, seg_lengths, hidden: int) -> int:
    """NEXT-1 dual A3 move: each source token's codes + scales read once, every padded row written
    row-wise (codes + scales) and column-wise (codes + one scale byte per (128-row block, column)),
    src_of_row read."""
    m = sum(seg_lengths)
    blocks = sum((x + 127) // 128 for x in seg_lengths)
    row = hidden + hidden // 128
    return unique_src_rows * row + m * row + m * hidden + blocks * hidden + m * 4


def dispatch_permute_bytes(unique_recv_tokens: int, padded_rows: int, total_tokens: int, top_k: int,
                           hidden: int) -> int:
    """NEXT-3 dispatch + permute (receive side): every routed token's codes + scales read once from
    its owner (NVLink on the 8-GPU box, HBM when the ranks share a device), every local row (incl.
    PAD) written once, the global plan's row_map read."""
    row = hidden + hidden // 128
    return unique_recv_tokens * row + padded_rows * row + total_tokens * top_k * 4


def combine_bytes(num_tokens: int, top_k: int, hidden: int, with_probs: bool = True) -> int:
    """NEXT-3 combine: top_k BF16 expert rows pulled per owned token, the BF16 output written,
    topk_idx + the experts' row_map entries (+ gates) read."""
    return num_tokens * top_k * hidden * 2 + num_tokens * hidden * 2 + num_tokens * top_k * (8 + (4 if with_probs else 0))


def measured_peaks(root: str) -> dict:
    """HBM copy bandwidth to use as the roofline denominator: the driver-measured figure when
    MEASURED_PEAKS.json exists, else the profiling guide's fallback (6650 GB/s)."""
    path = os.path.join(root, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}
