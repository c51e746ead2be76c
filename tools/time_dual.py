"""Times the NEXT-1 dual-output kernels against the two-launch composition they replace, L2
flushed before each measurement: A1 + A2 vs fp8flow_quantize_dual (cfg-2 shape 4096x7168, one
segment) and A5 + A2 vs fp8flow_swiglu_quant_dual (bench.py's A shape, 32 expert segments).
Usage: python tools/time_dual.py"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_02302_b200 import fp8flow as F, roofline as RL  # noqa: E402

dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
clean = torch.ones(64 << 20, dtype=torch.float32, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
peak = RL.measured_peaks(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))["hbm_gbs"]


def timed(fn):
    fn()
    ts = []
    for _ in range(30):
        flush.fill_(1)
        clean.sum()
        torch.cuda._sleep(1_000_000)
        ev[0].record()
        fn()
        ev[1].record()
        ev[1].synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    return statistics.median(ts) * 1e3


def report(name, us, nbytes):
    print(f"  {name:34s} {us:8.2f} us  {nbytes / us / 1e3:8.1f} GB/s  frac {nbytes / us / 1e3 / peak:.3f}")


# ---- A1 + A2 vs quantize_dual, 4096 x 7168 ---------------------------------------------------
rows, cols = 4096, 7168
x = synth.activations_bf16(rows, cols, synth.BASE_SEED + 9).to(dev)
q = torch.empty(rows, cols, dtype=torch.uint8, device=dev)
s = torch.empty(cols // 128, rows, dtype=torch.uint8, device=dev)
qT = torch.empty(rows * cols, dtype=torch.uint8, device=dev)
sT = torch.empty(rows // 128 + 1, cols, dtype=torch.uint8, device=dev)
b_dual = RL.quantize_dual_bytes([rows], cols)
print(f"quantize {rows}x{cols}")
t_a1 = timed(lambda: F.fp8flow_quantize_rowwise(x, q, s))
t_a2 = timed(lambda: F.fp8flow_scaling_aware_transpose(q, s, qT, sT))
t_two = timed(lambda: (F.fp8flow_quantize_rowwise(x, q, s), F.fp8flow_scaling_aware_transpose(q, s, qT, sT)))
t_dual = timed(lambda: F.fp8flow_quantize_dual(x, q, s, qT, sT))
report("A1", t_a1, RL.quantize_bytes(rows, cols))
report("A2", t_a2, RL.transpose_bytes([rows], cols))
report("A1 -> A2 (two launches)", t_two, b_dual)
report("quantize_dual", t_dual, b_dual)

# ---- A5 + A2 vs swiglu_quant_dual, bench shape ------------------------------------------------
R, FFN = 15872, 2048
rng = np.random.default_rng(3)
m = rng.integers(20, 40, 32) * 16
m = (m * (R / m.sum())).astype(np.int64) // 16 * 16
m[-1] += R - m.sum()
seg = torch.from_numpy(np.concatenate([[0], np.cumsum(m)]).astype(np.int32)).to(dev)
h = synth.normal_bf16(R, 2 * FFN, synth.BASE_SEED + 3, sigma=1.5).to(dev)
qa = torch.empty(R, FFN, dtype=torch.uint8, device=dev)
sa = torch.empty(FFN // 128, R, dtype=torch.uint8, device=dev)
aT = torch.empty(R * FFN, dtype=torch.uint8, device=dev)
saT = torch.empty(R // 128 + 32, FFN, dtype=torch.uint8, device=dev)
segs = [int(v) for v in m]
b_dual = RL.swiglu_quant_dual_bytes(segs, FFN)
print(f"swiglu {R}x{2 * FFN} -> {FFN}, 32 segments")
t_a5 = timed(lambda: F.fp8flow_swiglu_quant(h, qa, sa))
t_a2 = timed(lambda: F.fp8flow_scaling_aware_transpose(qa, sa, aT, saT, seg_offsets=seg))
t_two = timed(lambda: (F.fp8flow_swiglu_quant(h, qa, sa),
                       F.fp8flow_scaling_aware_transpose(qa, sa, aT, saT, seg_offsets=seg)))
t_dual = timed(lambda: F.fp8flow_swiglu_quant_dual(h, qa, sa, aT, saT, seg_offsets=seg))
report("A5", t_a5, RL.swiglu_quant_bytes(R, FFN))
report("A2", t_a2, RL.transpose_bytes(segs, FFN))
report("A5 -> A2 (two launches)", t_two, b_dual)
report("swiglu_quant_dual", t_dual, b_dual)
