"""ncu driver (not product): one A2 launch on the whole-layer X_perm (133056 x 7168, 256 experts)
and one on the dense 65536 x 7168, between cudaProfilerStart/Stop (L2 flushed before each)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth
from paper_2511_02302_b200 import fp8flow as F
dev = torch.device("cuda:0")
idx, _ = synth.routing(16384, synth.BASE_SEED)
cnt = np.bincount(idx.numpy().ravel(), minlength=256)
layer = np.concatenate([[0], np.cumsum((cnt + 15) // 16 * 16)]).astype(np.int32)
fw = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
fr = torch.ones(64 << 20, dtype=torch.float32, device=dev)
runs = []
for rows, cols, seg in [(int(layer[-1]), 7168, layer), (65536, 7168, None)]:
    q = torch.empty(rows, cols, dtype=torch.uint8, device=dev)
    s = torch.empty(cols // 128, rows, dtype=torch.uint8, device=dev)
    for r0 in range(0, rows, 16384):
        r1 = min(rows, r0 + 16384)
        x = synth.activations_bf16_device(r1 - r0, cols, 7 + r0, dev)
        F.fp8flow_quantize_rowwise(x, q[r0:r1], s[:, r0:r1])
    nseg = 1 if seg is None else len(seg) - 1
    qT = torch.empty(rows * cols, dtype=torch.uint8, device=dev)
    sT = torch.empty(rows // 128 + nseg, cols, dtype=torch.uint8, device=dev)
    seg_t = None if seg is None else torch.from_numpy(seg).to(dev)
    runs.append((q, s, qT, sT, seg_t))
for q, s, qT, sT, seg_t in runs:
    F.fp8flow_scaling_aware_transpose(q, s, qT, sT, seg_offsets=seg_t)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for q, s, qT, sT, seg_t in runs:
    fw.zero_(); fr.sum()
    F.fp8flow_scaling_aware_transpose(q, s, qT, sT, seg_offsets=seg_t)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
