"""A2 experiment driver (not product): marginal cold-L2 us of A2 under experiment-build env knobs.
    python tools/probe/a2_env.py VAR v1 v2 ...   (e.g. A2GATE 0 1)"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench, synth
from paper_2511_02302_b200 import fp8flow as F
from paper_2511_02302_b200 import roofline as RL
dev = torch.device("cuda:0")
fw = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
fr = torch.ones(64 << 20, dtype=torch.float32, device=dev)
flush = lambda: (fw.fill_(1), fr.sum())
peak = 6551.7
var, vals = sys.argv[1], sys.argv[2:]
idx, _ = synth.routing(16384, synth.BASE_SEED)
cnt = np.bincount(idx.numpy().ravel(), minlength=256)
layer = np.concatenate([[0], np.cumsum((cnt + 15) // 16 * 16)]).astype(np.int32)
g0 = np.concatenate([[0], np.cumsum(((cnt + 15) // 16 * 16)[:32])]).astype(np.int32)
shapes = [(2048, 7168, None), (4096, 7168, None), (8192, 7168, None), (int(g0[-1]), 7168, g0),
          (65536, 7168, None), (int(layer[-1]), 2048, layer), (int(layer[-1]), 7168, layer)]
for rows, cols, seg in shapes:
    q = torch.empty(rows, cols, dtype=torch.uint8, device=dev)
    s = torch.empty(cols // 128, rows, dtype=torch.uint8, device=dev)
    for r0 in range(0, rows, 16384):
        r1 = min(rows, r0 + 16384)
        x = synth.activations_bf16_device(r1 - r0, cols, 7 + r0, dev)
        F.fp8flow_quantize_rowwise(x, q[r0:r1], s[:, r0:r1])
        del x
    nseg = 1 if seg is None else len(seg) - 1
    seg_t = torch.from_numpy(seg).to(dev) if seg is not None else None
    qT = torch.empty(rows * cols, dtype=torch.uint8, device=dev)
    sT = torch.empty(rows // 128 + nseg, cols, dtype=torch.uint8, device=dev)
    nb = RL.transpose_bytes(np.diff(seg) if seg is not None else [rows], cols)
    line, ref = [], None
    for v in vals:
        os.environ[var] = v
        fn = lambda: F.fp8flow_scaling_aware_transpose(q, s, qT, sT, seg_offsets=seg_t)
        ts = [bench.marginal_us(fn, flush, K=20 if rows < 60000 else 6) for _ in range(3)]
        fn(); torch.cuda.synchronize()
        h = (qT.sum().item(), sT.sum().item())
        ref = ref or h
        line.append(f"{v}: {min(ts):.2f}/{np.median(ts):.2f}us {nb / min(ts) * 1e-3 / peak:.3f}{'' if h == ref else ' MISMATCH'}")
    print(f"{rows}x{cols} nseg={nseg}", " | ".join(line), flush=True)
    del q, s, qT, sT
