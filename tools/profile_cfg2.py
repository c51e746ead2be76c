"""Profiling driver (not product): config 2 (one expert's activations, 4096x7168) -- A1, A2 and the
naive dequant -> transpose -> requant comparator, one launch each between cudaProfilerStart/Stop:
    ncu --set full --profile-from-start off ... python tools/profile_cfg2.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_02302_b200 import fp8flow as F  # noqa: E402

dev = torch.device("cuda:0")
rows, cols = 4096, 7168
x = synth.activations_bf16_device(rows, cols, synth.BASE_SEED + 1, dev)
q = torch.empty(rows, cols, dtype=torch.uint8, device=dev)
s = torch.empty(cols // 128, rows, dtype=torch.uint8, device=dev)
qT = torch.empty(rows * cols, dtype=torch.uint8, device=dev)
sT = torch.empty(rows // 128 + 1, cols, dtype=torch.uint8, device=dev)
ws = torch.empty(F.fp8flow_naive_workspace_bytes(rows, cols, 1), dtype=torch.uint8, device=dev)


def ops():
    F.fp8flow_quantize_rowwise(x, q, s)
    F.fp8flow_scaling_aware_transpose(q, s, qT, sT)
    F.fp8flow_naive_transpose(q, s, qT, sT, ws)


for _ in range(3):
    ops()
torch.cuda.synchronize()
torch.cuda.profiler.start()
ops()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled: A1, A2, naive comparator (its launches) at 4096x7168")
