"""CPU oracle for the FP8-Flow-MoE hot path (arXiv 2511.02302) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import this package.  The product path (``paper_2511_02302_b200``) never
imports it and shares no code with it; the arithmetic lives in ``fp8flow_oracle.c`` (plain C,
scalar loops, fp64), which cites the paper passage each function follows.  This module only
marshals numpy arrays into that library (ctypes) and, for large inputs, splits independent rows /
segments across host threads (ctypes releases the GIL).

Parity status per function: see the header of ``fp8flow_oracle.c`` and DESIGN.md §4.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fp8flow_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# tests/test_oracle_mutations.py points this at a deliberately broken build of the same source to
# show that the pins catch the mutation; never set otherwise.
_LIB_OVERRIDE = os.environ.get("FP8FLOW_ORACLE_LIB")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no GPU, no nvcc).  Idempotent."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if _LIB_OVERRIDE:
                L = ctypes.CDLL(_LIB_OVERRIDE)
            else:
                build()
                L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            I64 = ctypes.c_int64
            I32 = ctypes.c_int32
            sig = {
                "orc_decode_e4m3": (ctypes.c_double, [ctypes.c_uint8]),
                "orc_encode_e4m3": (ctypes.c_uint8, [ctypes.c_double]),
                "orc_scale_exponent": (ctypes.c_int, [ctypes.c_double]),
                "orc_shift_e4m3": (ctypes.c_uint8, [ctypes.c_uint8, ctypes.c_int]),
                "orc_round_bf16": (ctypes.c_uint16, [ctypes.c_double]),
                "orc_quantize_rows_f64": (None, [P, I64, I64, P, P, I64]),
                "orc_quantize_rowwise_bf16": (None, [P, I64, I64, P, P, I64]),
                "orc_dequantize_rows": (None, [P, P, I64, I64, I64, P]),
                "orc_quantize_rows_real": (None, [P, I64, I64, P, P]),
                "orc_scaling_aware_transpose": (None, [P, P, I64, I64, I64, P, I32, P, P]),
                "orc_naive_transpose": (None, [P, P, I64, I64, I64, P, I32, P, P]),
                "orc_permute_plan": (ctypes.c_int, [P, I64, I32, I32, I32, I32, P, P, I64, P]),
                "orc_permute_pad": (None, [P, P, I64, I64, I64, P, P, I32, I64, P, P]),
                "orc_unpermute": (None, [P, I64, P, P, I64, I32, P]),
                "orc_swiglu_f32": (None, [P, I64, I64, P]),
                "orc_swiglu_quant": (None, [P, I64, I64, P, P, I64]),
                "orc_checksum64": (ctypes.c_uint64, [P, I64]),
                "orc_swiglu_bwd_f32": (None, [P, P, I64, I64, P]),
                "orc_swiglu_bwd_quant": (None, [P, P, I64, I64, P, P, I64]),
                "orc_gemm_blockscaled": (None, [P, P, I64, P, P, I64, I64, I64, I64, P, I32, I64, I64, P]),
                "orc_combine": (None, [P, P, I64, P, I32, P, I64, I64, I32, P]),
            }
            for name, (res, args) in sig.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _p(a: np.ndarray | None, off: int = 0):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "oracle inputs must be C-contiguous"
    return a.ctypes.data + off


def _threads(n_items: int, threads: int | None) -> int:
    if threads is None:
        threads = len(os.sched_getaffinity(0))
    return max(1, min(threads, n_items))


def _run_split(n: int, threads: int | None, fn) -> None:
    """Run fn(lo, hi) over [0, n) split into contiguous chunks, one host thread per chunk."""
    t = _threads(n, threads)
    if t == 1:
        fn(0, n)
        return
    bounds = np.linspace(0, n, t + 1).astype(np.int64)
    ths = [threading.Thread(target=fn, args=(int(bounds[i]), int(bounds[i + 1]))) for i in range(t)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()


# --------------------------------------------------------------------------------------------
# scalar codec (C1, C2, C3, C5)
# --------------------------------------------------------------------------------------------
def decode_e4m3(c: int) -> float:
    return lib().orc_decode_e4m3(int(c))


def encode_e4m3(v: float) -> int:
    return lib().orc_encode_e4m3(float(v))


def scale_exponent(amax: float) -> int:
    return lib().orc_scale_exponent(float(amax))


def shift_e4m3(c: int, k: int) -> int:
    return lib().orc_shift_e4m3(int(c), int(k))


def round_bf16(v: float) -> int:
    return lib().orc_round_bf16(float(v))


def decode_table() -> np.ndarray:
    return np.array([decode_e4m3(c) for c in range(256)], dtype=np.float64)


# --------------------------------------------------------------------------------------------
# tensors.  BF16 tensors are passed as uint16 bit patterns.  Scales are MN-major [tiles][ld_s].
# --------------------------------------------------------------------------------------------
def quantize_rowwise_bf16(x_bits: np.ndarray, ld_s: int | None = None, threads: int | None = None):
    """A1 (C4): BF16 [rows, cols] -> (codes u8 [rows, cols], scales u8 [cols/128, ld_s])."""
    x_bits = np.ascontiguousarray(x_bits, dtype=np.uint16)
    rows, cols = x_bits.shape
    ld_s = rows if ld_s is None else ld_s
    q = np.zeros((rows, cols), np.uint8)
    s = np.zeros(((cols + 127) // 128, ld_s), np.uint8)
    L = lib()

    def work(lo, hi):
        L.orc_quantize_rowwise_bf16(_p(x_bits, lo * cols * 2), hi - lo, cols, _p(q, lo * cols), _p(s, lo), ld_s)

    _run_split(rows, threads, work)
    return q, s


def quantize_rows_f64(x: np.ndarray, ld_s: int | None = None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    rows, cols = x.shape
    ld_s = rows if ld_s is None else ld_s
    q = np.zeros((rows, cols), np.uint8)
    s = np.zeros(((cols + 127) // 128, ld_s), np.uint8)
    lib().orc_quantize_rows_f64(_p(x), rows, cols, _p(q), _p(s), ld_s)
    return q, s


def dequantize_rows(q: np.ndarray, s: np.ndarray) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.uint8)
    s = np.ascontiguousarray(s, dtype=np.uint8)
    rows, cols = q.shape
    x = np.zeros((rows, cols), np.float64)
    lib().orc_dequantize_rows(_p(q), _p(s), s.shape[1], rows, cols, _p(x))
    return x


def quantize_rows_real(x: np.ndarray):
    """Real-valued scales s = amax/448 (Eq. 2 literal), for the Eq. 1 demonstration only."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    rows, cols = x.shape
    q = np.zeros((rows, cols), np.uint8)
    s = np.zeros((cols // 128, rows), np.float64)
    lib().orc_quantize_rows_real(_p(x), rows, cols, _p(q), _p(s))
    return q, s


def transpose_out_sizes(rows: int, cols: int, seg_offsets) -> tuple[int, int]:
    """(bytes of qT, number of scale-tile rows of sT) for a segmented transpose."""
    if seg_offsets is None:
        return rows * cols, (rows + 127) // 128
    seg = np.asarray(seg_offsets, dtype=np.int64)
    m = np.diff(seg)
    return int(seg[-1]) * cols, int(np.sum((m + 127) // 128))


def _transpose(fn_name: str, q, s, seg_offsets, threads):
    q = np.ascontiguousarray(q, dtype=np.uint8)
    s = np.ascontiguousarray(s, dtype=np.uint8)
    rows, cols = q.shape
    L = lib()
    fn = getattr(L, fn_name)
    if seg_offsets is None:
        seg = np.array([0, rows], np.int32)
    else:
        seg = np.ascontiguousarray(seg_offsets, dtype=np.int32)
    nseg = len(seg) - 1
    m = np.diff(seg.astype(np.int64))
    tiles = (m + 127) // 128
    tile_base = np.concatenate([[0], np.cumsum(tiles)]).astype(np.int64)
    qT = np.zeros(int(seg[-1]) * cols, np.uint8)
    sT = np.zeros((int(tile_base[-1]), cols), np.uint8)

    def work(lo, hi):
        # segments [lo, hi): call with a sub-array of offsets; output pointers shifted so that the
        # library's placement formulas (N*o_e, N*P_e) land in the global buffers.
        for e in range(lo, hi):
            sub = np.ascontiguousarray(seg[e:e + 2])
            fn(_p(q), _p(s), s.shape[1], rows, cols, _p(sub), 1, _p(qT), _p(sT, int(tile_base[e]) * cols))

    _run_split(nseg, threads, work)
    return qT, sT


def scaling_aware_transpose(q, s, seg_offsets=None, threads: int | None = None):
    """A2 (C6, Algorithm 1).  Returns (qT flat bytes, sT [sum ceil(m_e/128), cols])."""
    return _transpose("orc_scaling_aware_transpose", q, s, seg_offsets, threads)


def naive_transpose(q, s, seg_offsets=None, threads: int | None = None):
    """C7 naive dequant(BF16) -> transpose -> column-wise requant; same layout as A2."""
    return _transpose("orc_naive_transpose", q, s, seg_offsets, threads)


def permute_plan(topk_idx: np.ndarray, e0: int, E_loc: int, align: int = 16, max_rows: int | None = None):
    """A3 plan (C8).  Returns (row_map [T,K], src_of_row [max_rows], offsets [E_loc+1])."""
    topk_idx = np.ascontiguousarray(topk_idx, dtype=np.int32)
    T, K = topk_idx.shape
    if max_rows is None:
        max_rows = T * K + E_loc * (align - 1)
    row_map = np.zeros((T, K), np.int32)
    src = np.zeros(max_rows, np.int32)
    off = np.zeros(E_loc + 1, np.int32)
    rc = lib().orc_permute_plan(_p(topk_idx), T, K, e0, E_loc, align, _p(row_map), _p(src), max_rows, _p(off))
    if rc != 0:
        raise ValueError("padded rows exceed max_rows")
    return row_map, src, off


def permute_pad(q_tok, s_tok, src_of_row, offsets, max_rows: int | None = None, threads: int | None = None):
    """A3 move (C8).  Returns (q_out [max_rows, H], s_out [H/128, max_rows]); rows >= R zero."""
    q_tok = np.ascontiguousarray(q_tok, dtype=np.uint8)
    s_tok = np.ascontiguousarray(s_tok, dtype=np.uint8)
    src_of_row = np.ascontiguousarray(src_of_row, dtype=np.int32)
    offsets = np.ascontiguousarray(offsets, dtype=np.int32)
    T, H = q_tok.shape
    max_rows = len(src_of_row) if max_rows is None else max_rows
    E_loc = len(offsets) - 1
    q_out = np.zeros((max_rows, H), np.uint8)
    s_out = np.zeros((H // 128, max_rows), np.uint8)
    L = lib()
    R = int(offsets[-1])

    def work(lo, hi):
        # rows [lo, hi): a one-"expert" offsets view [0, hi-lo] over shifted src/out pointers
        sub_off = np.array([0, hi - lo], np.int32)
        L.orc_permute_pad(_p(q_tok), _p(s_tok), s_tok.shape[1], T, H, _p(src_of_row, 4 * lo), _p(sub_off), 1,
                          max_rows, _p(q_out, lo * H), _p(s_out, lo))

    _run_split(R, threads, work)
    del E_loc
    return q_out, s_out


def unpermute(x_bits, row_map, probs=None, threads: int | None = None):
    """A4 (C9).  x_bits BF16 [R, H] -> y BF16 bits [T, H]."""
    x_bits = np.ascontiguousarray(x_bits, dtype=np.uint16)
    row_map = np.ascontiguousarray(row_map, dtype=np.int32)
    T, K = row_map.shape
    H = x_bits.shape[1]
    if probs is not None:
        probs = np.ascontiguousarray(probs, dtype=np.float32)
    y = np.zeros((T, H), np.uint16)
    L = lib()

    def work(lo, hi):
        L.orc_unpermute(_p(x_bits), H, _p(row_map, 4 * lo * K), _p(probs, 4 * lo * K) if probs is not None else None,
                        hi - lo, K, _p(y, 2 * lo * H))

    _run_split(T, threads, work)
    return y


def swiglu_f32(h_bits):
    h_bits = np.ascontiguousarray(h_bits, dtype=np.uint16)
    rows, F2 = h_bits.shape
    y = np.zeros((rows, F2 // 2), np.float32)
    lib().orc_swiglu_f32(_p(h_bits), rows, F2 // 2, _p(y))
    return y


def swiglu_quant(h_bits, ld_s: int | None = None, threads: int | None = None):
    """A5 (C10).  h BF16 [rows, 2F] -> (q [rows, F], s [F/128, ld_s])."""
    h_bits = np.ascontiguousarray(h_bits, dtype=np.uint16)
    rows, F2 = h_bits.shape
    F = F2 // 2
    ld_s = rows if ld_s is None else ld_s
    q = np.zeros((rows, F), np.uint8)
    s = np.zeros((F // 128, ld_s), np.uint8)
    L = lib()

    def work(lo, hi):
        L.orc_swiglu_quant(_p(h_bits, lo * F2 * 2), hi - lo, F, _p(q, lo * F), _p(s, lo), ld_s)

    _run_split(rows, threads, work)
    return q, s


def swiglu_bwd_f32(h_bits, dA_bits):
    """NEXT-1: fp32 [rows, 2F] = [dA*b*silu'(a) | dA*silu(a)] (fp64 evaluation, one rounding)."""
    h_bits = np.ascontiguousarray(h_bits, dtype=np.uint16)
    dA_bits = np.ascontiguousarray(dA_bits, dtype=np.uint16)
    rows, F2 = h_bits.shape
    assert dA_bits.shape == (rows, F2 // 2)
    dh = np.zeros((rows, F2), np.float32)
    lib().orc_swiglu_bwd_f32(_p(h_bits), _p(dA_bits), rows, F2 // 2, _p(dh))
    return dh


def swiglu_bwd_quant(h_bits, dA_bits, ld_s: int | None = None, threads: int | None = None):
    """NEXT-1: h BF16 [rows, 2F], dA BF16 [rows, F] -> (q [rows, 2F], s [2F/128, ld_s])."""
    h_bits = np.ascontiguousarray(h_bits, dtype=np.uint16)
    dA_bits = np.ascontiguousarray(dA_bits, dtype=np.uint16)
    rows, F2 = h_bits.shape
    F = F2 // 2
    ld_s = rows if ld_s is None else ld_s
    q = np.zeros((rows, F2), np.uint8)
    s = np.zeros((F2 // 128, ld_s), np.uint8)
    L = lib()

    def work(lo, hi):
        L.orc_swiglu_bwd_quant(_p(h_bits, lo * F2 * 2), _p(dA_bits, lo * F * 2), hi - lo, F, _p(q, lo * F2),
                               _p(s, lo), ld_s)

    _run_split(rows, threads, work)
    return q, s


def checksum64(buf: np.ndarray) -> int:
    b = np.ascontiguousarray(buf).view(np.uint8).reshape(-1)
    return int(lib().orc_checksum64(_p(b), b.size))


def gemm_blockscaled(A, sa, B, sb, seg_offsets=None, threads: int | None = None):
    """NEXT-2 (R33): D[m][n] = sum_k dequant(A)[m][k] * dequant(B_g)[n][k] in fp64.
    A u8 [M, K], sa u8 [K/128, ld_sa]; B u8 [G, N, K] (or [N, K]), sb u8 [G, K/128, ld_sb] (or 2-D).
    Rows outside every group are NaN."""
    A = np.ascontiguousarray(A, dtype=np.uint8)
    sa = np.ascontiguousarray(sa, dtype=np.uint8)
    B = np.ascontiguousarray(B, dtype=np.uint8)
    sb = np.ascontiguousarray(sb, dtype=np.uint8)
    M, K = A.shape
    N = B.shape[-2]
    D = np.full((M, N), np.nan, np.float64)
    seg = None if seg_offsets is None else np.ascontiguousarray(seg_offsets, dtype=np.int32)
    groups = 1 if seg is None else len(seg) - 1
    L = lib()

    def work(lo, hi):
        L.orc_gemm_blockscaled(_p(A), _p(sa), sa.shape[-1], _p(B), _p(sb), sb.shape[-1], M, N, K, _p(seg), groups,
                               lo, hi, _p(D))

    _run_split(M, threads, work)
    return D


# --------------------------------------------------------------------------------------------
# NEXT-3: expert-parallel dispatch + permute and combine across ranks
# --------------------------------------------------------------------------------------------
def dispatch_permute_pad(q_list, s_list, topk_list, rank: int, num_experts: int, align: int = 16,
                         max_rows: int | None = None, threads: int | None = None):
    """What rank `rank` of n = len(q_list) holds after the FP8 dispatch (the row-wise codes
    and their scales travel) and the fused permute + pad (C8) of the tokens it received: by
    definition the C8 plan and move over every rank's tokens gathered in rank order (global token
    id = r * tokens_per_rank + t) restricted to the rank's experts [rank*E/n, (rank+1)*E/n).
    q_list[r] [Tpr, H] uint8, s_list[r] [H/128, ld] uint8 (first Tpr columns used), topk_list[r]
    [Tpr, K] int32.  Returns (q_out, s_out, row_map [n*Tpr, K], src_of_row, offsets)."""
    n = len(q_list)
    e_per = num_experts // n
    q_all = np.concatenate([np.ascontiguousarray(q) for q in q_list], axis=0)
    tpr = q_list[0].shape[0]
    s_all = np.concatenate([np.ascontiguousarray(s)[:, :tpr] for s in s_list], axis=1)
    topk_all = np.concatenate([np.ascontiguousarray(t, dtype=np.int32) for t in topk_list], axis=0)
    row_map, src, off = permute_plan(topk_all, rank * e_per, e_per, align=align, max_rows=max_rows)
    q_out, s_out = permute_pad(q_all, s_all, src, off, max_rows=len(src), threads=threads)
    return q_out, s_out, row_map, src, off


def combine(x_list, row_map_list, topk_idx, experts_per_rank: int, probs=None, token_begin: int = 0,
            threads: int | None = None):
    """NEXT-3 combine (orc_combine): the owner's tokens [token_begin, token_begin + T) summed over
    their top_k expert outputs x_list[d] (BF16 bits [rows_d, H]) located by row_map_list[d]
    ([T_global, K], rank d's plan).  Returns y BF16 bits [T, H]."""
    xs = [np.ascontiguousarray(x, dtype=np.uint16) for x in x_list]
    rms = [np.ascontiguousarray(r, dtype=np.int32) for r in row_map_list]
    topk_idx = np.ascontiguousarray(topk_idx, dtype=np.int32)
    T, K = topk_idx.shape
    H = xs[0].shape[1]
    if probs is not None:
        probs = np.ascontiguousarray(probs, dtype=np.float32)
    xp = (ctypes.c_void_p * len(xs))(*[x.ctypes.data for x in xs])
    rp = (ctypes.c_void_p * len(rms))(*[r.ctypes.data for r in rms])
    y = np.zeros((T, H), np.uint16)
    L = lib()

    def work(lo, hi):
        L.orc_combine(ctypes.cast(xp, ctypes.c_void_p), ctypes.cast(rp, ctypes.c_void_p), H, _p(topk_idx, 4 * lo * K),
                      experts_per_rank, _p(probs, 4 * lo * K) if probs is not None else None, token_begin + lo,
                      hi - lo, K, _p(y, 2 * lo * H))

    _run_split(T, threads, work)
    return y
