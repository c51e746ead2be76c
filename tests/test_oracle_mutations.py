"""Mutation checks of the oracle's pins: each case compiles a deliberately broken copy of
``oracle/fp8flow_oracle.c`` (one plausible mistake: a dropped term, a wrong index, another
grouping or order) and asserts that the pin tests named for it FAIL against that build, while the
unmodified source passes the same tests.  The oracle module loads the mutated library through
``FP8FLOW_ORACLE_LIB`` (set only here).

Each mutation cites the passage / DESIGN.md reading the mutated line implements.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "fp8flow_oracle.c")

sys.path.insert(0, ROOT)
import oracle  # noqa: E402

# A whole-column amax instead of one per 128-row block (R29): the helper is inserted
# before orc_naive_transpose and replaces its per-tile quantization of a column.
_WHOLE_COLUMN = """
static void quantize_row_whole_column(const double* x, int64_t n, uint8_t* q, uint8_t* s_col, int64_t ld_s,
                                      int64_t row)
{
    double amax = 0.0;
    for (int64_t j = 0; j < n; j++) if (fabs(x[j]) > amax) amax = fabs(x[j]);
    int t = orc_scale_exponent(amax);
    for (int64_t tile = 0; tile * 128 < n; tile++) s_col[tile * ld_s + row] = (uint8_t)(t + 127);
    for (int64_t j = 0; j < n; j++) q[j] = orc_encode_e4m3(x[j] * ldexp(1.0, -t));
}

void orc_naive_transpose("""

MUTATIONS = {
    # P:224 / R29 -- the verdict's first mutation
    "naive_whole_column_scale": (
        [("void orc_naive_transpose(", _WHOLE_COLUMN),
         ("quantize_row_f64(col, m, qTe + j * m, sTe, cols, j);",
          "quantize_row_whole_column(col, m, qTe + j * m, sTe, cols, j);")],
        "tests/test_oracle_tensor.py", "naive"),
    # dequantize with the first tile's row scale for every column
    "naive_wrong_row_tile": (
        [("ldexp(1.0, (int)s[(j / 128) * ld_s + (o + i)] - 127);", "ldexp(1.0, (int)s[0 * ld_s + (o + i)] - 127);")],
        "tests/test_oracle_tensor.py", "naive"),
    # P:322-324 / R21 -- the verdict's second mutation: k summed in reverse order
    "unpermute_reverse_k": (
        [("for (int32_t k = 0; k < K; k++) {\n                int32_t r = row_map[t * K + k];",
          "for (int32_t k = K - 1; k >= 0; k--) {\n                int32_t r = row_map[t * K + k];")],
        "tests/test_oracle_moe.py", "unpermute"),
    # R34 -- combine in reverse k order
    "combine_reverse_k": (
        [("for (int32_t k = 0; k < K; k++) {\n                int32_t d = topk_idx",
          "for (int32_t k = K - 1; k >= 0; k--) {\n                int32_t d = topk_idx")],
        "tests/test_oracle_ep.py", "combine"),
    # R21 -- an fp64 accumulator (one rounding at the end) instead of fp32 FMA steps
    "unpermute_fp64_accumulator": (
        [("            float acc = 0.0f;\n            for (int32_t k = 0; k < K; k++) {\n                int32_t r =",
          "            double acc = 0.0;\n            for (int32_t k = 0; k < K; k++) {\n                int32_t r =")],
        "tests/test_oracle_moe.py", "unpermute"),
    # Alg. 1 line "S_max = max": the block minimum instead
    "transpose_min_scale": (
        [("int tmax = -1000;", "int tmax = 1000;"), ("if (t > tmax) tmax = t;", "if (t < tmax) tmax = t;")],
        "tests/test_oracle_tensor.py", "transpose"),
    # Alg. 1 / R5 -- k with the wrong sign (shift up instead of down)
    "transpose_k_sign": (
        [("int k = tmax - ((int)s[jb * ld_s + i] - 127);", "int k = ((int)s[jb * ld_s + i] - 127) - tmax;")],
        "tests/test_oracle_tensor.py", "transpose"),
    # R3 -- pow2 scale rounded down (floor) instead of the least covering T
    "scale_floor": (
        [("while (amax > 448.0 * ldexp(1.0, t)) t++;", "while (amax > 448.0 * ldexp(1.0, t)) t++;\n    t--;")],
        "tests/test_oracle_codec.py", "scale"),
    # R16 -- tokens placed in descending order inside an expert
    "plan_descending_tokens": (
        [("        int64_t next = offsets[le];\n        for (int64_t t = 0; t < T; t++)",
          "        int64_t next = offsets[le];\n        for (int64_t t = T - 1; t >= 0; t--)")],
        "tests/test_oracle_moe.py", "permute or plan"),
    # R18 -- SwiGLU gate on the second half
    "swiglu_halves_swapped": (
        [("y[i * F + j] = (float)(a * b / (1.0 + exp(-a)));", "y[i * F + j] = (float)(a * b / (1.0 + exp(-b)));")],
        "tests/test_oracle_moe.py", "swiglu"),
    # Eq. 4 / R33 -- GEMM drops B's block scale
    "gemm_drops_b_scale": (
        [("double b = orc_decode_e4m3(Bg[n * K + k]) * ldexp(1.0, (int)sbg[(k / 128) * ld_sb + n] - 127);",
          "double b = orc_decode_e4m3(Bg[n * K + k]);")],
        "tests/test_oracle_tensor.py tests/test_oracle_codec.py tests/test_oracle_moe.py", "gemm"),
}


def _build(tmp_path, name, edits):
    src = open(SRC).read()
    for old, new in edits:
        assert src.count(old) >= 1, f"{name}: pattern not found: {old!r}"
        src = src.replace(old, new, 1)
    cpath = tmp_path / f"{name}.c"
    cpath.write_text(src)
    so = tmp_path / f"lib{name}.so"
    subprocess.check_call(["gcc", *oracle.CFLAGS, "-o", str(so), str(cpath), "-lm"])
    return str(so)


def _run(files, kexpr, lib):
    env = dict(os.environ)
    if lib:
        env["FP8FLOW_ORACLE_LIB"] = lib
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-k", kexpr, *files.split()]
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)


def test_pins_catch_every_mutation(tmp_path):
    """Every mutation fails its pins; the unmodified source (compiled the same way) passes the same
    pin sets.  The pytest subprocesses run concurrently (they are independent)."""
    from concurrent.futures import ThreadPoolExecutor

    control = _build(tmp_path, "control", [])
    jobs = {name: (files, kexpr, _build(tmp_path, name, edits)) for name, (edits, files, kexpr) in MUTATIONS.items()}
    for files, kexpr in {(f, k) for _, f, k in MUTATIONS.values()}:
        jobs[f"control:{files}:{kexpr}"] = (files, kexpr, control)
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), len(os.sched_getaffinity(0))))) as ex:
        res = dict(zip(jobs, ex.map(lambda j: _run(*j), jobs.values())))
    bad = []
    for name, r in res.items():
        if name.startswith("control:"):
            if r.returncode != 0 or " passed" not in r.stdout:      # also: the selection is not empty
                bad.append(f"{name} fails on the unmodified oracle:\n{r.stdout[-1500:]}")
        elif not (r.returncode == 1 and " failed" in r.stdout):
            bad.append(f"mutation {name} survived its pins:\n{r.stdout[-1500:]}{r.stderr[-1500:]}")
    assert not bad, "\n".join(bad)
