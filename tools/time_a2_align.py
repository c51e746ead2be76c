"""Experiment: A2 on a 15872x7168 FP8 input with 32 expert segments padded to 16 rows (the paper's
P:319, bench.py) vs the same row count in segments padded to 128 rows, vs one segment -- does the
16-byte-only alignment of the column-wise output rows cost bandwidth?  L2 flushed, median of 30."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02302_b200 import fp8flow as F, roofline as RL  # noqa: E402

dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
clean = torch.ones(64 << 20, dtype=torch.float32, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
R, H = 15872, 7168
q = torch.randint(0, 0x7E, (R, H), dtype=torch.uint8, device=dev)
s = torch.randint(115, 125, (H // 128, R), dtype=torch.uint8, device=dev)
qT = torch.empty(R * H, dtype=torch.uint8, device=dev)
sT = torch.empty(R // 128 + 32, H, dtype=torch.uint8, device=dev)
rng = np.random.default_rng(0)
m16 = rng.integers(300, 700, 32) // 16 * 16
m16[-1] += R - m16.sum()
m128 = np.full(32, R // 32 // 128 * 128)
m128[-1] += R - m128.sum()
for name, m in [("32 segments, pad 16", m16), ("32 segments, pad 128", m128), ("one segment", None)]:
    seg = None if m is None else torch.tensor(np.concatenate([[0], np.cumsum(m)]), dtype=torch.int32, device=dev)
    fn = lambda: F.fp8flow_scaling_aware_transpose(q, s, qT, sT, seg_offsets=seg)  # noqa: E731
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
    ms = statistics.median(ts)
    nb = RL.transpose_bytes([R] if m is None else list(m), H)
    print(f"{name:24s} {ms * 1e3:7.2f} us  {nb / ms / 1e6:7.1f} GB/s", flush=True)
