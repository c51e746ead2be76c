"""CPU checks of the C-ABI library: it builds, loads, exports exactly what include/fp8flow.h declares,
and validates arguments synchronously (these paths return before any CUDA call, so they run
without a GPU).  No compute is launched here."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fp8flow.h")


@pytest.fixture(scope="module")
def L():
    from paper_2511_02302_b200 import build, fp8flow

    build.build_library()
    return fp8flow.lib()


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"FP8FLOW_API\s+[\w\s\*]+?\b(fp8flow_\w+)\s*\(", txt)))


def test_exports_match_header(L):
    from paper_2511_02302_b200 import fp8flow

    declared = header_symbols()
    assert len(declared) >= 14
    out = subprocess.check_output(["nm", "-D", "--defined-only", fp8flow.LIB_PATH]).decode()
    exported = sorted(set(re.findall(r"\b(fp8flow_\w+)\b", out)))
    assert exported == declared
    assert sorted(fp8flow.SIGNATURES) == declared          # the binding covers every entry point
    for name in declared:
        assert hasattr(L, name)


def test_build_target_is_sm100a(L):
    from paper_2511_02302_b200 import fp8flow

    assert L.fp8flow_build_target() == b"sm_100a"
    sass = subprocess.run(["cuobjdump", "--list-elf", fp8flow.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in sass


def test_tma_and_no_legacy_tensor_path_in_sass():
    """The transpose kernel issues TMA (UTMALDG); none of the kernels uses tensor-core MMA (HBM-bound ops)."""
    from paper_2511_02302_b200 import fp8flow

    sass = subprocess.run(["cuobjdump", "-sass", fp8flow.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass
    assert "HMMA" not in sass


def test_status_strings(L):
    assert L.fp8flow_status_string(0) == b"FP8FLOW_OK"
    assert L.fp8flow_status_string(6) == b"FP8FLOW_ERR_ARCH"


def test_validation_before_any_cuda_call(L):
    # bad shapes / args are rejected synchronously (no device needed)
    assert L.fp8flow_quantize_rowwise(None, 4, 100, None, None, 16, None) == 2            # cols % 128
    assert L.fp8flow_quantize_rowwise(None, 4, 128, None, None, 2, None) == 2              # ld_s < rows
    assert L.fp8flow_quantize_rowwise(None, 0, 128, None, None, 16, None) == 0             # empty: no-op
    assert L.fp8flow_quantize_rowwise(None, 4, 128, None, None, 16, None) == 1             # NULL
    assert L.fp8flow_quantize_rowwise(ctypes.c_void_p(8), 4, 128, ctypes.c_void_p(16), ctypes.c_void_p(16), 16,
                                      None) == 3                                            # alignment
    assert L.fp8flow_scaling_aware_transpose(None, None, 32, 24, 128, None, 0, None, None, None) == 2  # rows % 16
    assert L.fp8flow_scaling_aware_transpose(ctypes.c_void_p(16), ctypes.c_void_p(16), 32, 32, 128,
                                             ctypes.c_void_p(16), 2000, ctypes.c_void_p(16), ctypes.c_void_p(16),
                                             None) == 4                                     # num_segs
    assert L.fp8flow_permute_plan(None, 10, 0, 0, 8, 16, None, None, 100, None, None, 0, None) == 4   # top_k
    assert L.fp8flow_permute_plan(None, 10, 8, 0, 0, 16, None, None, 100, None, None, 0, None) == 4   # E_loc
    ws_need = L.fp8flow_permute_workspace_bytes(10, 8, 4)
    assert ws_need > 0
    assert L.fp8flow_permute_plan(ctypes.c_void_p(16), 10, 8, 0, 4, 16, ctypes.c_void_p(16), ctypes.c_void_p(16),
                                  100, ctypes.c_void_p(16), ctypes.c_void_p(16), ws_need - 1, None) == 5
    assert L.fp8flow_unpermute_unpad(None, 7168, None, None, 4, 17, None, None) == 4       # top_k > 16
    assert L.fp8flow_swiglu_quant(None, 4, None, 100, None, None, 16, None) == 2            # ffn % 128
    assert L.fp8flow_naive_transpose(ctypes.c_void_p(16), ctypes.c_void_p(16), 32, 32, 128, None, 0,
                                     ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(16), 10, None) == 5


def test_validation_of_next_row_entry_points(L):
    """NEXT-1 / NEXT-2 entry points reject bad arguments synchronously, with the documented codes."""
    P = ctypes.c_void_p
    a16 = P(16)
    # SwiGLU backward: ffn % 128, ld_s < rows, NULL, alignment
    assert L.fp8flow_swiglu_bwd_quant(None, None, 4, None, 100, None, None, 16, None) == 2
    assert L.fp8flow_swiglu_bwd_quant(None, None, 32, None, 128, None, None, 16, None) == 2
    assert L.fp8flow_swiglu_bwd_quant(None, None, 4, None, 128, None, None, 16, None) == 1
    assert L.fp8flow_swiglu_bwd_quant(P(8), a16, 4, None, 128, a16, a16, 16, None) == 3
    # dual outputs: transpose-style shape rules (rows % 16, cols % 128), NULL input, segment count
    assert L.fp8flow_quantize_dual(a16, 24, 128, None, 0, a16, a16, 32, a16, a16, None) == 2
    assert L.fp8flow_quantize_dual(None, 32, 128, None, 0, a16, a16, 32, a16, a16, None) == 1
    assert L.fp8flow_quantize_dual(a16, 32, 128, a16, 2000, a16, a16, 32, a16, a16, None) == 4
    assert L.fp8flow_swiglu_quant_dual(a16, 32, None, 100, None, 0, a16, a16, 32, a16, a16, None) == 2
    assert L.fp8flow_swiglu_quant_dual(P(8), 32, None, 128, None, 0, a16, a16, 32, a16, a16, None) == 3
    # GEMM: M % 16, N % 256, K % 128, ld_sa < M, groups out of range, NULL, alignment
    assert L.fp8flow_gemm_blockscaled(a16, a16, 32, a16, a16, 256, 24, 256, 128, None, 0, a16, 1, None) == 2
    assert L.fp8flow_gemm_blockscaled(a16, a16, 32, a16, a16, 256, 32, 128, 128, None, 0, a16, 1, None) == 2
    assert L.fp8flow_gemm_blockscaled(a16, a16, 32, a16, a16, 256, 32, 256, 100, None, 0, a16, 1, None) == 2
    assert L.fp8flow_gemm_blockscaled(a16, a16, 16, a16, a16, 256, 32, 256, 128, None, 0, a16, 1, None) == 2
    assert L.fp8flow_gemm_blockscaled(a16, a16, 32, a16, a16, 256, 32, 256, 128, a16, 600, a16, 1, None) == 4
    assert L.fp8flow_gemm_blockscaled(None, a16, 32, a16, a16, 256, 32, 256, 128, None, 0, a16, 1, None) == 1
    assert L.fp8flow_gemm_blockscaled(P(8), a16, 32, a16, a16, 256, 32, 256, 128, None, 0, a16, 1, None) == 3
    assert L.fp8flow_gemm_blockscaled(None, None, 0, None, None, 256, 0, 256, 128, None, 0, None, 1, None) == 0
    # fused move + A2: hidden % 128, max_rows % 16, scale pitch (>= tokens, % 4), expert count, NULL,
    # alignment; no tokens = no-op
    pd = L.fp8flow_permute_pad_dual
    assert pd(a16, a16, 64, 64, 100, a16, a16, 4, 64, a16, a16, a16, a16, None) == 2
    assert pd(a16, a16, 64, 64, 128, a16, a16, 4, 60, a16, a16, a16, a16, None) == 2
    assert pd(a16, a16, 32, 64, 128, a16, a16, 4, 64, a16, a16, a16, a16, None) == 2
    assert pd(a16, a16, 66, 64, 128, a16, a16, 4, 64, a16, a16, a16, a16, None) == 2
    assert pd(a16, a16, 64, 64, 128, a16, a16, 0, 64, a16, a16, a16, a16, None) == 4
    assert pd(a16, a16, 64, 64, 128, a16, a16, 2000, 64, a16, a16, a16, a16, None) == 4
    assert pd(a16, a16, 64, 64, 128, a16, a16, 4, 64, a16, a16, None, a16, None) == 1
    assert pd(P(8), a16, 64, 64, 128, a16, a16, 4, 64, a16, a16, a16, a16, None) == 3
    assert pd(a16, P(8), 64, 64, 128, a16, a16, 4, 64, a16, a16, a16, a16, None) == 3
    assert pd(None, None, 0, 0, 128, None, None, 4, 64, None, None, None, None, None) == 0
    # Wgrad: Ma % 128, Nb % 256, groups required, NULL, workspace size and alignment
    a128 = P(128)
    assert L.fp8flow_gemm_wgrad_workspace_bytes(4) == 1024
    assert L.fp8flow_gemm_wgrad(a16, a16, 100, a16, a16, 256, a16, 4, a16, 1, a128, 1024, None) == 2
    assert L.fp8flow_gemm_wgrad(a16, a16, 128, a16, a16, 200, a16, 4, a16, 1, a128, 1024, None) == 2
    assert L.fp8flow_gemm_wgrad(a16, a16, 128, a16, a16, 256, a16, 0, a16, 1, a128, 1024, None) == 4
    assert L.fp8flow_gemm_wgrad(a16, a16, 128, a16, a16, 256, None, 4, a16, 1, a128, 1024, None) == 1
    assert L.fp8flow_gemm_wgrad(a16, a16, 128, a16, a16, 256, a16, 4, a16, 1, None, 1024, None) == 1
    assert L.fp8flow_gemm_wgrad(a16, a16, 128, a16, a16, 256, a16, 4, a16, 1, a128, 1023, None) == 5
    assert L.fp8flow_gemm_wgrad(a16, a16, 128, a16, a16, 256, a16, 4, a16, 1, a16, 1024, None) == 3


def test_validation_of_next3_entry_points(L):
    """NEXT-3 peer-memory entry points reject bad arguments synchronously (no device touched)."""
    P = ctypes.c_void_p
    a16 = P(16)
    tab2 = (P * 2)(16, 32)
    tab_null = (P * 2)(16, None)
    tab_mis = (P * 2)(16, 40)
    # IPC helpers: NULL arguments
    assert L.fp8flow_ipc_get_handle(None, None, None) == 1
    assert L.fp8flow_ipc_open(None, None) == 1
    assert L.fp8flow_ipc_close(None) == 1
    # barrier: rank outside [0, n), n outside [1, 64], NULL table / entry
    assert L.fp8flow_peer_barrier(tab2, 2, 2, None, 100, None) == 4
    assert L.fp8flow_peer_barrier(tab2, 0, 65, None, 100, None) == 4
    assert L.fp8flow_peer_barrier(None, 0, 2, None, 100, None) == 1
    assert L.fp8flow_peer_barrier(tab_null, 0, 2, None, 100, None) == 1
    # gather: bytes % 4, empty no-op, misaligned peer
    assert L.fp8flow_peer_gather(tab2, 2, 22, a16, None, None) == 2
    assert L.fp8flow_peer_gather(tab2, 2, 0, None, None, None) == 0
    assert L.fp8flow_peer_gather(tab_mis, 2, 32, a16, None, None) == 3
    # dispatch: top_k, hidden % 128, ld_s < tokens, NULL plan, unknown kernel choice
    assert L.fp8flow_dispatch_permute_pad(tab2, tab2, 64, 2, 64, 7168, a16, 17, a16, a16, 32, 1024, a16, a16,
                                          0, None, None) == 4
    assert L.fp8flow_dispatch_permute_pad(tab2, tab2, 64, 2, 64, 100, a16, 8, a16, a16, 32, 1024, a16, a16,
                                          0, None, None) == 2
    assert L.fp8flow_dispatch_permute_pad(tab2, tab2, 32, 2, 64, 7168, a16, 8, a16, a16, 32, 1024, a16, a16,
                                          0, None, None) == 2
    assert L.fp8flow_dispatch_permute_pad(tab2, tab2, 64, 2, 64, 7168, None, 8, a16, a16, 32, 1024, a16, a16,
                                          0, None, None) == 1
    assert L.fp8flow_dispatch_permute_pad(tab2, tab2, 64, 2, 64, 7168, a16, 8, a16, a16, 32, 1024, a16, a16,
                                          3, None, None) == 4
    # combine: experts_per_rank, hidden % 8, empty no-op, NULL peer entry
    assert L.fp8flow_combine_unpermute(tab2, tab2, 2, 7168, a16, 0, None, 0, 4, 8, a16, None, None) == 4
    assert L.fp8flow_combine_unpermute(tab2, tab2, 2, 7164, a16, 32, None, 0, 4, 8, a16, None, None) == 2
    assert L.fp8flow_combine_unpermute(tab2, tab2, 2, 7168, a16, 32, None, 0, 0, 8, a16, None, None) == 0
    assert L.fp8flow_combine_unpermute(tab_null, tab2, 2, 7168, a16, 32, None, 0, 4, 8, a16, None, None) == 1


def test_no_device_means_error_not_fallback(L):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    # valid arguments, but no usable device: a CUDA/arch error, never a silent CPU path
    st = L.fp8flow_quantize_rowwise(ctypes.c_void_p(16), 4, 128, ctypes.c_void_p(16), ctypes.c_void_p(16), 16, None)
    assert st in (6, 7)


def test_binding_refuses_cpu_tensors(L):
    import torch

    from paper_2511_02302_b200 import fp8flow

    x = torch.zeros(4, 128, dtype=torch.bfloat16)
    q = torch.zeros(4, 128, dtype=torch.uint8)
    s = torch.zeros(1, 16, dtype=torch.uint8)
    with pytest.raises(fp8flow.Fp8FlowError):
        fp8flow.fp8flow_quantize_rowwise(x, q, s)


def test_product_package_never_imports_oracle():
    """The product path (package + CUDA sources) neither imports, links nor calls the oracle."""
    pkg = os.path.join(ROOT, "paper_2511_02302_b200")
    bad = re.compile(r"^\s*(import\s+oracle|from\s+oracle\b)|liboracle|\borc_\w+\(|fp8flow_oracle", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                assert not bad.search(open(os.path.join(dirpath, f)).read()), f


def test_oracle_loaded_only_by_tests_smoke_and_bench_cpu_leg():
    """oracle/ is test infrastructure: tools/ never load it, and in bench.py only cpu_baseline_leg
    (and the --impl reference arm, which IS the oracle) import it."""
    bad = re.compile(r"^\s*(import\s+oracle|from\s+oracle\b)", re.M)
    for f in os.listdir(os.path.join(ROOT, "tools")):
        if f.endswith(".py"):
            assert not bad.search(open(os.path.join(ROOT, "tools", f)).read()), f
    src = open(os.path.join(ROOT, "bench.py")).read()
    owners = []
    for m in bad.finditer(src):
        head = src[:m.start()]
        owners.append(re.findall(r"^def (\w+)", head, re.M)[-1])
    assert sorted(owners) == ["cpu_baseline_leg", "run_reference"], owners



def test_product_library_has_no_environment_knobs():
    """The library reads no environment variables (no tuning or results-changing switches): every
    launch configuration is a constant of the source; kernel choices that a caller may need are
    explicit arguments (fp8flow_dispatch_permute_pad's `kernel`)."""
    csrc = os.path.join(ROOT, "paper_2511_02302_b200", "csrc")
    for f in os.listdir(csrc):
        txt = open(os.path.join(csrc, f)).read()
        assert "getenv" not in txt and "FP8FLOW_" not in txt.replace("FP8FLOW_OK", "").replace(
            "FP8FLOW_ERR_", "").replace("FP8FLOW_DISPATCH_", "").replace("FP8FLOW_MAX_RANKS", "").replace(
            "FP8FLOW_IPC_HANDLE_BYTES", "").replace("FP8FLOW_UNKNOWN_STATUS", "").replace(
            "FP8FLOW_SOURCE_HASH", ""), f


def test_stale_library_is_refused(monkeypatch):
    """Build provenance: the library carries the hash of the sources it was compiled from; the
    binding refuses to load a library whose hash differs from the sources next to it."""
    from paper_2511_02302_b200 import build as B
    from paper_2511_02302_b200 import fp8flow

    assert fp8flow.lib().fp8flow_source_hash().decode() == B.source_hash()
    monkeypatch.setattr(fp8flow, "_lib", None)
    monkeypatch.setattr(B, "source_hash", lambda: "0000000000000000")
    with pytest.raises(fp8flow.Fp8FlowError, match="built from other sources"):
        fp8flow.lib()
