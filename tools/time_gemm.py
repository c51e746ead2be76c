"""Times the NEXT-2 block-scaled FP8 GEMM (TFLOP/s vs the FP8 dense peak = 2 x measured bf16) on
the MoE shapes of bench.py's expert group and a square shape, next to torch._scaled_mm (cuBLAS
FP8, per-tensor scales -- a library ceiling, not the same math) where available.
Usage: python tools/time_gemm.py"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02302_b200 import fp8flow as F  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
dev = torch.device("cuda:0")
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1673.3}
fp8_peak = 2 * peaks["bf16_tflops"]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def med(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda._sleep(500_000)
        ev[0].record()
        fn()
        ev[1].record()
        ev[1].synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    return statistics.median(ts)


def case(name, M, N, K, G, seg=None):
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    A = torch.randint(0, 120, (M, K), dtype=torch.uint8, device=dev, generator=g)
    B = torch.randint(0, 120, (G, N, K), dtype=torch.uint8, device=dev, generator=g)
    sa = torch.full((K // 128, M), 120, dtype=torch.uint8, device=dev)
    sb = torch.full((G, K // 128, N), 127, dtype=torch.uint8, device=dev)
    D = torch.empty(M, N, dtype=torch.bfloat16, device=dev)
    segt = None if seg is None else torch.tensor(seg, dtype=torch.int32, device=dev)
    ms = med(lambda: F.fp8flow_gemm_blockscaled(A, sa, B if G > 1 else B[0], sb if G > 1 else sb[0], D, seg_offsets=segt))
    rows = M if seg is None else seg[-1]
    flops = 2.0 * rows * N * K
    tf = flops / ms / 1e9
    line = f"{name:34s} {ms * 1e3:9.1f} us  {tf:7.1f} TFLOP/s  frac {tf / fp8_peak:.3f}"
    if G == 1 and hasattr(torch, "_scaled_mm"):
        try:
            a8 = A.view(torch.float8_e4m3fn)
            b8 = B[0].view(torch.float8_e4m3fn)
            one = torch.ones((), device=dev)
            ms2 = med(lambda: torch._scaled_mm(a8, b8.t(), scale_a=one, scale_b=one, out_dtype=torch.bfloat16))
            line += f"   | cuBLAS FP8 (per-tensor) {ms2 * 1e3:8.1f} us {flops / ms2 / 1e9:7.1f} TFLOP/s"
        except Exception as e:  # noqa: BLE001
            line += f"   | cuBLAS FP8 unavailable: {type(e).__name__}"
    print(line, flush=True)


print(f"FP8 dense peak used: {fp8_peak:.1f} TFLOP/s (2 x measured bf16)")
case("square 8192^3", 8192, 8192, 8192, 1)
case("fprop-like 16384x4096x7168", 16384, 4096, 7168, 1)
rng = np.random.default_rng(0)
m = (rng.integers(20, 40, 32) * 16)
m = (m * (15872 / m.sum())).astype(np.int64) // 16 * 16
m[-1] += 15872 - m.sum()
seg = [0] + list(np.cumsum(m).astype(int))
case("grouped fc1 fprop 32 experts N=4096", 15872, 4096, 7168, 32, seg)
case("grouped fc2 fprop 32 experts N=7168", 15872, 7168, 2048, 32, seg)


def wgrad_case(name, Ma, Nb, m):
    seg = torch.tensor([0] + list(np.cumsum(m).astype(int)), dtype=torch.int32, device=dev)
    R = int(sum(m))
    G = len(m)
    P = int(sum((x + 127) // 128 for x in m))
    AT = torch.randint(0, 120, (R * Ma,), dtype=torch.uint8, device=dev)
    BT = torch.randint(0, 120, (R * Nb,), dtype=torch.uint8, device=dev)
    saT = torch.full((P, Ma), 120, dtype=torch.uint8, device=dev)
    sbT = torch.full((P, Nb), 120, dtype=torch.uint8, device=dev)
    D = torch.empty(G, Ma, Nb, dtype=torch.bfloat16, device=dev)
    ms = med(lambda: F.fp8flow_gemm_wgrad(AT, saT, BT, sbT, D, seg), reps=5)
    flops = 2.0 * R * Ma * Nb
    tf = flops / ms / 1e9
    out_gbs = D.numel() * 2 / ms / 1e6
    print(f"{name:34s} {ms * 1e3:9.1f} us  {tf:7.1f} TFLOP/s  frac {tf / fp8_peak:.3f}  (BF16 dW written at "
          f"{out_gbs:.0f} GB/s)", flush=True)


wgrad_case("grouped fc1 wgrad 32 experts", 4096, 7168, list(m))
