"""Thin Python binding of libfp8flow (include/fp8flow.h).

Argument marshalling only: every function has the name of the C entry point it calls, takes
torch CUDA tensors (device memory owned by the caller) and passes their pointers, sizes and the
current CUDA stream to the library.  No compute happens here and there is no fallback: if the
shared library is missing or the device is not sm_100, calls raise.

Layouts (see include/fp8flow.h): BF16 tensors are torch.bfloat16; E4M3 codes and UE8M0 scale
bytes are torch.uint8; scales are MN-major [cols/128, ld_s].
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libfp8flow.so")
_lib = None

STATUS = {
    0: "FP8FLOW_OK", 1: "FP8FLOW_ERR_NULL", 2: "FP8FLOW_ERR_SHAPE", 3: "FP8FLOW_ERR_ALIGN",
    4: "FP8FLOW_ERR_ARG", 5: "FP8FLOW_ERR_WORKSPACE", 6: "FP8FLOW_ERR_ARCH", 7: "FP8FLOW_ERR_CUDA",
}

# exported symbols and their C signatures (restype, argtypes)
_P, _I64, _I32, _SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
SIGNATURES = {
    "fp8flow_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "fp8flow_last_cuda_error": (ctypes.c_int, []),
    "fp8flow_version": (ctypes.c_int, []),
    "fp8flow_build_target": (ctypes.c_char_p, []),
    "fp8flow_source_hash": (ctypes.c_char_p, []),
    "fp8flow_device_check": (ctypes.c_int, []),
    "fp8flow_quantize_rowwise": (ctypes.c_int, [_P, _I64, _I64, _P, _P, _I64, _P]),
    "fp8flow_scaling_aware_transpose": (ctypes.c_int, [_P, _P, _I64, _I64, _I64, _P, _I32, _P, _P, _P]),
    "fp8flow_naive_workspace_bytes": (_SZ, [_I64, _I64, _I32]),
    "fp8flow_naive_transpose": (ctypes.c_int, [_P, _P, _I64, _I64, _I64, _P, _I32, _P, _P, _P, _SZ, _P]),
    "fp8flow_permute_workspace_bytes": (_SZ, [_I64, _I32, _I32]),
    "fp8flow_permute_plan": (ctypes.c_int, [_P, _I64, _I32, _I32, _I32, _I32, _P, _P, _I64, _P, _P, _SZ, _P]),
    "fp8flow_permute_pad": (ctypes.c_int, [_P, _P, _I64, _I64, _I64, _P, _I32, _P, _P, _I32, _I64, _P, _P, _P]),
    "fp8flow_unpermute_unpad": (ctypes.c_int, [_P, _I64, _P, _P, _I64, _I32, _P, _P]),
    "fp8flow_swiglu_quant": (ctypes.c_int, [_P, _I64, _P, _I64, _P, _P, _I64, _P]),
    "fp8flow_checksum64": (ctypes.c_int, [_P, _I64, _P, _P]),
    "fp8flow_swiglu_bwd_quant": (ctypes.c_int, [_P, _P, _I64, _P, _I64, _P, _P, _I64, _P]),
    "fp8flow_quantize_dual": (ctypes.c_int, [_P, _I64, _I64, _P, _I32, _P, _P, _I64, _P, _P, _P]),
    "fp8flow_swiglu_quant_dual": (ctypes.c_int, [_P, _I64, _P, _I64, _P, _I32, _P, _P, _I64, _P, _P, _P]),
    "fp8flow_permute_pad_dual": (ctypes.c_int, [_P, _P, _I64, _I64, _I64, _P, _P, _I32, _I64, _P, _P, _P, _P, _P]),
    "fp8flow_gemm_blockscaled": (ctypes.c_int, [_P, _P, _I64, _P, _P, _I64, _I64, _I64, _I64, _P, _I32, _P, _I32, _P]),
    "fp8flow_gemm_wgrad_workspace_bytes": (_I64, [_I32]),
    "fp8flow_gemm_wgrad": (ctypes.c_int, [_P, _P, _I64, _P, _P, _I64, _P, _I32, _P, _I32, _P, _I64, _P]),
    "fp8flow_ipc_get_handle": (ctypes.c_int, [_P, _P, ctypes.POINTER(_I64)]),
    "fp8flow_ipc_open": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    "fp8flow_ipc_close": (ctypes.c_int, [_P]),
    "fp8flow_peer_barrier": (ctypes.c_int, [_P, _I32, _I32, _P, ctypes.c_uint32, _P]),
    "fp8flow_peer_gather": (ctypes.c_int, [_P, _I32, _I64, _P, _P, _P]),
    "fp8flow_dispatch_permute_pad": (ctypes.c_int, [_P, _P, _I64, _I32, _I64, _I64, _P, _I32, _P, _P, _I32, _I64,
                                                    _P, _P, _I32, _P, _P]),
    "fp8flow_combine_unpermute": (ctypes.c_int, [_P, _P, _I32, _I64, _P, _I32, _P, _I64, _I64, _I32, _P, _P, _P]),
}

IPC_HANDLE_BYTES = 64
MAX_RANKS = 64


class Fp8FlowError(RuntimeError):
    pass


def lib() -> ctypes.CDLL:
    """Loads libfp8flow.so (built in-tree by __graft_entry__.build()).  Raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise Fp8FlowError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        from . import build as _build

        built, current = L.fp8flow_source_hash().decode(), _build.source_hash()
        if built != current:
            raise Fp8FlowError(f"{LIB_PATH} was built from other sources (hash {built}, sources {current}): "
                               "rebuild with `python -c 'import __graft_entry__ as g; g.build()'`")
        _lib = L
    return _lib


def _check(status: int, what: str) -> None:
    if status != 0:
        msg = f"{what} failed: {STATUS.get(status, status)}"
        if status == 7:
            msg += f" (cudaError {lib().fp8flow_last_cuda_error()})"
        raise Fp8FlowError(msg)


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise Fp8FlowError("libfp8flow takes device tensors only (no CPU fallback)")
    if not t.is_contiguous():
        raise Fp8FlowError("tensors must be contiguous")
    return t.data_ptr()


def _ptr_rows(t: torch.Tensor):
    """A 2-D matrix whose rows are contiguous (its row pitch is passed separately)."""
    if not t.is_cuda:
        raise Fp8FlowError("libfp8flow takes device tensors only (no CPU fallback)")
    if t.dim() != 2 or t.stride(1) != 1:
        raise Fp8FlowError("matrix rows must be contiguous")
    return t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _u8(t):
    assert t.dtype == torch.uint8, t.dtype
    return t


# ----------------------------------------------------------------------------------- misc
def fp8flow_device_check() -> None:
    _check(lib().fp8flow_device_check(), "fp8flow_device_check")


def fp8flow_version() -> int:
    return lib().fp8flow_version()


def fp8flow_build_target() -> str:
    return lib().fp8flow_build_target().decode()


def fp8flow_source_hash() -> str:
    return lib().fp8flow_source_hash().decode()


# ----------------------------------------------------------------------------------- A1
def fp8flow_quantize_rowwise(x: torch.Tensor, q: torch.Tensor, s: torch.Tensor, stream=None) -> None:
    """x bf16 [rows, cols] -> q uint8 [rows, cols], s uint8 [cols/128, ld_s] (ld_s = s.stride(0): a
    column slice of a wider scale matrix is accepted)."""
    assert x.dtype == torch.bfloat16 and x.dim() == 2 and s.stride(1) == 1
    rows, cols = x.shape
    _check(lib().fp8flow_quantize_rowwise(_ptr(x), rows, cols, _ptr(_u8(q)), _ptr_rows(_u8(s)), s.stride(0),
                                          _stream(stream)), "fp8flow_quantize_rowwise")


# ----------------------------------------------------------------------------------- A2
def fp8flow_scaling_aware_transpose(q: torch.Tensor, s: torch.Tensor, qT: torch.Tensor, sT: torch.Tensor,
                                    seg_offsets: torch.Tensor | None = None, stream=None) -> None:
    """q uint8 [rows, cols] + s [cols/128, ld_s] -> qT (flat, segment-major), sT [tiles, cols]."""
    rows, cols = q.shape
    nseg = 0 if seg_offsets is None else seg_offsets.numel() - 1
    if seg_offsets is not None:
        assert seg_offsets.dtype == torch.int32
    _check(lib().fp8flow_scaling_aware_transpose(_ptr(_u8(q)), _ptr(_u8(s)), s.shape[1], rows, cols,
                                                 _ptr(seg_offsets), nseg, _ptr(_u8(qT)), _ptr(_u8(sT)),
                                                 _stream(stream)), "fp8flow_scaling_aware_transpose")


def fp8flow_naive_workspace_bytes(rows: int, cols: int, num_segs: int) -> int:
    return lib().fp8flow_naive_workspace_bytes(rows, cols, num_segs)


def fp8flow_naive_transpose(q, s, qT, sT, ws: torch.Tensor, seg_offsets=None, stream=None) -> None:
    rows, cols = q.shape
    nseg = 0 if seg_offsets is None else seg_offsets.numel() - 1
    _check(lib().fp8flow_naive_transpose(_ptr(_u8(q)), _ptr(_u8(s)), s.shape[1], rows, cols, _ptr(seg_offsets), nseg,
                                         _ptr(_u8(qT)), _ptr(_u8(sT)), _ptr(ws), ws.numel() * ws.element_size(),
                                         _stream(stream)), "fp8flow_naive_transpose")


# ----------------------------------------------------------------------------------- A3
def fp8flow_permute_workspace_bytes(num_tokens: int, top_k: int, num_local_experts: int) -> int:
    return lib().fp8flow_permute_workspace_bytes(num_tokens, top_k, num_local_experts)


def fp8flow_permute_plan(topk_idx: torch.Tensor, expert_begin: int, num_local_experts: int, align: int,
                         row_map: torch.Tensor, src_of_row: torch.Tensor, expert_offsets: torch.Tensor,
                         ws: torch.Tensor, stream=None) -> None:
    assert topk_idx.dtype == torch.int32 and topk_idx.dim() == 2
    T, K = topk_idx.shape
    _check(lib().fp8flow_permute_plan(_ptr(topk_idx), T, K, expert_begin, num_local_experts, align, _ptr(row_map),
                                      _ptr(src_of_row), src_of_row.numel(), _ptr(expert_offsets), _ptr(ws),
                                      ws.numel() * ws.element_size(), _stream(stream)), "fp8flow_permute_plan")


def fp8flow_permute_pad(q_tok, s_tok, row_map, src_of_row, expert_offsets, q_out, s_out, stream=None) -> None:
    """A3 move with the plan's (row_map, src_of_row, expert_offsets): q_tok [T, H] + s_tok [H/128, ld]."""
    T, H = q_tok.shape
    _check(lib().fp8flow_permute_pad(_ptr(_u8(q_tok)), _ptr(_u8(s_tok)), s_tok.shape[1], T, H, _ptr(row_map),
                                     row_map.shape[1], _ptr(src_of_row), _ptr(expert_offsets),
                                     expert_offsets.numel() - 1, q_out.shape[0], _ptr(_u8(q_out)), _ptr(_u8(s_out)),
                                     _stream(stream)), "fp8flow_permute_pad")


# ----------------------------------------------------------------------------------- A4
def fp8flow_unpermute_unpad(x: torch.Tensor, row_map: torch.Tensor, probs: torch.Tensor | None, y: torch.Tensor,
                            stream=None) -> None:
    assert x.dtype == torch.bfloat16 and y.dtype == torch.bfloat16
    T, K = row_map.shape
    _check(lib().fp8flow_unpermute_unpad(_ptr(x), x.shape[1], _ptr(row_map), _ptr(probs), T, K, _ptr(y),
                                         _stream(stream)), "fp8flow_unpermute_unpad")


# ----------------------------------------------------------------------------------- A5
def fp8flow_swiglu_quant(h: torch.Tensor, q: torch.Tensor, s: torch.Tensor, rows_dev: torch.Tensor | None = None,
                         stream=None) -> None:
    assert h.dtype == torch.bfloat16 and h.dim() == 2
    rows_max, F2 = h.shape
    _check(lib().fp8flow_swiglu_quant(_ptr(h), rows_max, _ptr(rows_dev), F2 // 2, _ptr(_u8(q)), _ptr(_u8(s)),
                                      s.shape[1], _stream(stream)), "fp8flow_swiglu_quant")


def fp8flow_swiglu_bwd_quant(h: torch.Tensor, dA: torch.Tensor, q: torch.Tensor, s: torch.Tensor,
                             rows_dev: torch.Tensor | None = None, stream=None) -> None:
    """NEXT-1: h bf16 [rows, 2F], dA bf16 [rows, F] -> q uint8 [rows, 2F], s uint8 [2F/128, ld_s]."""
    assert h.dtype == torch.bfloat16 and dA.dtype == torch.bfloat16
    rows_max, F2 = h.shape
    assert dA.shape == (rows_max, F2 // 2)
    _check(lib().fp8flow_swiglu_bwd_quant(_ptr(h), _ptr(dA), rows_max, _ptr(rows_dev), F2 // 2, _ptr(_u8(q)),
                                          _ptr(_u8(s)), s.shape[1], _stream(stream)), "fp8flow_swiglu_bwd_quant")


def fp8flow_quantize_dual(x: torch.Tensor, q: torch.Tensor, s: torch.Tensor, qT: torch.Tensor, sT: torch.Tensor,
                          seg_offsets: torch.Tensor | None = None, stream=None) -> None:
    """NEXT-1 dual output: x bf16 [rows, cols] -> q, s (as A1) and qT, sT (as A2 of q, s)."""
    assert x.dtype == torch.bfloat16 and x.dim() == 2
    rows, cols = x.shape
    nseg = 0 if seg_offsets is None else seg_offsets.numel() - 1
    _check(lib().fp8flow_quantize_dual(_ptr(x), rows, cols, _ptr(seg_offsets), nseg, _ptr(_u8(q)), _ptr(_u8(s)),
                                       s.shape[1], _ptr(_u8(qT)), _ptr(_u8(sT)), _stream(stream)),
           "fp8flow_quantize_dual")


def fp8flow_swiglu_quant_dual(h: torch.Tensor, q: torch.Tensor, s: torch.Tensor, qT: torch.Tensor, sT: torch.Tensor,
                              seg_offsets: torch.Tensor | None = None, rows_dev: torch.Tensor | None = None,
                              stream=None) -> None:
    """NEXT-1 dual output: h bf16 [rows, 2F] -> q, s (as A5) and qT, sT (as A2 of q, s)."""
    assert h.dtype == torch.bfloat16 and h.dim() == 2
    rows_max, F2 = h.shape
    nseg = 0 if seg_offsets is None else seg_offsets.numel() - 1
    _check(lib().fp8flow_swiglu_quant_dual(_ptr(h), rows_max, _ptr(rows_dev), F2 // 2, _ptr(seg_offsets), nseg,
                                           _ptr(_u8(q)), _ptr(_u8(s)), s.shape[1], _ptr(_u8(qT)), _ptr(_u8(sT)),
                                           _stream(stream)), "fp8flow_swiglu_quant_dual")


def fp8flow_permute_pad_dual(q_tok, s_tok, src_of_row, expert_offsets, q_out, s_out, qT, sT, stream=None) -> None:
    """NEXT-1 dual output of the A3 move: (q_out, s_out) as fp8flow_permute_pad and (qT, sT) as A2 of them
    with the plan's expert offsets as segments."""
    T, H = q_tok.shape
    _check(lib().fp8flow_permute_pad_dual(_ptr(_u8(q_tok)), _ptr(_u8(s_tok)), s_tok.shape[1], T, H, _ptr(src_of_row),
                                          _ptr(expert_offsets), expert_offsets.numel() - 1, q_out.shape[0],
                                          _ptr(_u8(q_out)), _ptr(_u8(s_out)), _ptr(_u8(qT)), _ptr(_u8(sT)),
                                          _stream(stream)), "fp8flow_permute_pad_dual")


def fp8flow_gemm_blockscaled(A: torch.Tensor, sa: torch.Tensor, B: torch.Tensor, sb: torch.Tensor, D: torch.Tensor,
                             seg_offsets: torch.Tensor | None = None, stream=None) -> None:
    """NEXT-2: A uint8 [M, K] + sa [K/128, ld_sa]; B uint8 [G, N, K] (or [N, K]) + sb [G, K/128, ld_sb]
    (or [K/128, ld_sb]); D float32 or bfloat16 [M, N]."""
    M, K = A.shape
    N = B.shape[-2]
    G = 1 if B.dim() == 2 else B.shape[0]
    assert D.shape == (M, N) and D.dtype in (torch.float32, torch.bfloat16)
    ngroups = 0 if seg_offsets is None else seg_offsets.numel() - 1
    assert seg_offsets is None or ngroups == G
    _check(lib().fp8flow_gemm_blockscaled(_ptr(_u8(A)), _ptr(_u8(sa)), sa.shape[-1], _ptr(_u8(B)), _ptr(_u8(sb)),
                                          sb.shape[-1], M, N, K, _ptr(seg_offsets), ngroups, _ptr(D),
                                          1 if D.dtype == torch.float32 else 0, _stream(stream)),
           "fp8flow_gemm_blockscaled")


def fp8flow_gemm_wgrad(AT: torch.Tensor, saT: torch.Tensor, BT: torch.Tensor, sbT: torch.Tensor, D: torch.Tensor,
                       seg_offsets: torch.Tensor, workspace: torch.Tensor | None = None, stream=None) -> None:
    """NEXT-2 Wgrad: AT/BT flat uint8 (A2 outputs of [rows, Ma] / [rows, Nb]) + their sT [tiles, Ma/Nb];
    D float32 or bfloat16 [G, Ma, Nb]; groups = the A2 segments.  workspace: uint8 CUDA tensor of
    >= fp8flow_gemm_wgrad_workspace_bytes(G) bytes (allocated here when None)."""
    G, Ma, Nb = D.shape
    assert seg_offsets.numel() == G + 1 and saT.shape[1] == Ma and sbT.shape[1] == Nb
    if workspace is None:
        workspace = torch.empty(fp8flow_gemm_wgrad_workspace_bytes(G), dtype=torch.uint8, device=D.device)
    _check(lib().fp8flow_gemm_wgrad(_ptr(_u8(AT)), _ptr(_u8(saT)), Ma, _ptr(_u8(BT)), _ptr(_u8(sbT)), Nb,
                                    _ptr(seg_offsets), G, _ptr(D), 1 if D.dtype == torch.float32 else 0,
                                    _ptr(workspace), workspace.numel(), _stream(stream)), "fp8flow_gemm_wgrad")


def fp8flow_gemm_wgrad_workspace_bytes(num_groups: int) -> int:
    return int(lib().fp8flow_gemm_wgrad_workspace_bytes(num_groups))


def fp8flow_checksum64(buf: torch.Tensor, out: torch.Tensor, stream=None) -> None:
    """out: int64 CUDA tensor of one element (holds the uint64 bit pattern)."""
    _check(lib().fp8flow_checksum64(_ptr(buf), buf.numel() * buf.element_size(), _ptr(out), _stream(stream)),
           "fp8flow_checksum64")


# ----------------------------------------------------------------------------------- NEXT-3
def _table(ptrs) -> ctypes.Array:
    """Host array of device pointers (ints, or CUDA tensors whose data_ptr is taken)."""
    vals = [p.data_ptr() if isinstance(p, torch.Tensor) else int(p) for p in ptrs]
    return (ctypes.c_void_p * len(vals))(*vals)


def fp8flow_ipc_get_handle(t: torch.Tensor) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding t, byte offset of t inside it)."""
    h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    off = ctypes.c_int64(0)
    _check(lib().fp8flow_ipc_get_handle(_ptr(t), h, ctypes.byref(off)), "fp8flow_ipc_get_handle")
    return h.raw, off.value


def fp8flow_ipc_open(handle: bytes) -> int:
    """Maps another process's allocation; returns its base device address in this process."""
    base = ctypes.c_void_p(0)
    buf = ctypes.create_string_buffer(bytes(handle), IPC_HANDLE_BYTES)
    _check(lib().fp8flow_ipc_open(buf, ctypes.byref(base)), "fp8flow_ipc_open")
    return int(base.value)


def fp8flow_ipc_close(base: int) -> None:
    _check(lib().fp8flow_ipc_close(ctypes.c_void_p(base)), "fp8flow_ipc_close")


def fp8flow_peer_barrier(peer_signal, rank: int, status: torch.Tensor | None = None, timeout_ms: int = 10000,
                         stream=None) -> None:
    """peer_signal: n device pointers to the ranks' uint32 [n+1] signal buffers (zeroed once)."""
    n = len(peer_signal)
    _check(lib().fp8flow_peer_barrier(_table(peer_signal), rank, n, _ptr(status), timeout_ms, _stream(stream)),
           "fp8flow_peer_barrier")


def fp8flow_peer_gather(peer_src, bytes_per_rank: int, dst: torch.Tensor, status: torch.Tensor | None = None,
                        stream=None) -> None:
    """status: the barrier's device int32 (the kernel writes nothing if it is nonzero) or None."""
    n = len(peer_src)
    _check(lib().fp8flow_peer_gather(_table(peer_src), n, bytes_per_rank, _ptr(dst), _ptr(status), _stream(stream)),
           "fp8flow_peer_gather")


DISPATCH_AUTO, DISPATCH_ENGINE, DISPATCH_REGISTER = 0, 1, 2


def fp8flow_dispatch_permute_pad(peer_q, peer_s, ld_s_tok: int, tokens_per_rank: int, hidden: int,
                                 row_map: torch.Tensor, src_of_row: torch.Tensor, expert_offsets: torch.Tensor,
                                 q_out: torch.Tensor, s_out: torch.Tensor, kernel: int = DISPATCH_AUTO,
                                 status: torch.Tensor | None = None, stream=None) -> None:
    """peer_q / peer_s: n device pointers (or tensors) of the ranks' A1 outputs; row_map etc. from
    fp8flow_permute_plan over the gathered topk_idx [n*tokens_per_rank, K].  kernel: DISPATCH_*
    (identical results); status: the barrier gate or None."""
    n = len(peer_q)
    assert len(peer_s) == n
    _check(lib().fp8flow_dispatch_permute_pad(_table(peer_q), _table(peer_s), ld_s_tok, n, tokens_per_rank, hidden,
                                              _ptr(row_map), row_map.shape[1], _ptr(src_of_row),
                                              _ptr(expert_offsets), expert_offsets.numel() - 1, q_out.shape[0],
                                              _ptr(_u8(q_out)), _ptr(_u8(s_out)), kernel, _ptr(status),
                                              _stream(stream)),
           "fp8flow_dispatch_permute_pad")


def fp8flow_combine_unpermute(peer_x, peer_row_map, hidden: int, topk_idx: torch.Tensor, experts_per_rank: int,
                              probs: torch.Tensor | None, token_begin: int, y: torch.Tensor,
                              status: torch.Tensor | None = None, stream=None) -> None:
    """peer_x: n device pointers to BF16 expert outputs; peer_row_map: n device pointers to the
    ranks' plan row_maps; topk_idx/probs [T, K] of the caller's tokens; y bf16 [T, hidden]."""
    n = len(peer_x)
    assert y.dtype == torch.bfloat16
    T, K = topk_idx.shape
    _check(lib().fp8flow_combine_unpermute(_table(peer_x), _table(peer_row_map), n, hidden, _ptr(topk_idx),
                                           experts_per_rank, _ptr(probs), token_begin, T, K, _ptr(y), _ptr(status),
                                           _stream(stream)), "fp8flow_combine_unpermute")

# ----------------------------------------------------------------------------------- sizes
def transpose_out_shapes(rows: int, cols: int, num_segs: int = 1):
    """Capacity of qT (bytes) and sT (tile rows) for fp8flow_scaling_aware_transpose."""
    return rows * cols, rows // 128 + num_segs


def permute_max_rows(num_tokens: int, top_k: int, num_local_experts: int, align: int = 16) -> int:
    r = num_tokens * top_k + num_local_experts * (align - 1)
    return (r + 15) // 16 * 16
