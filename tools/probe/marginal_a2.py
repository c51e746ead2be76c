import os, statistics, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth
from paper_2511_02302_b200 import fp8flow as F
from paper_2511_02302_b200 import roofline as RL
dev = torch.device("cuda:0")
fw = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
fr = torch.ones(64 << 20, dtype=torch.float32, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
def flush():
    fw.fill_(1); fr.sum()
def marginal(fn, K=20, reps=5):
    fn(); res = []
    for _ in range(reps):
        tt = []
        for with_op in (True, False):
            torch.cuda.synchronize(); torch.cuda._sleep(30_000_000)
            ev[0].record()
            for _ in range(K):
                flush()
                if with_op: fn()
            ev[1].record(); ev[1].synchronize()
            tt.append(ev[0].elapsed_time(ev[1]) * 1e3)
        res.append((tt[0] - tt[1]) / K)
    return statistics.median(res)
peak = 6551.7
rng = np.random.default_rng(1)
def segs(rows, n):
    w = rng.gamma(1.0, 1.0, n); m = np.floor(w / w.sum() * rows / 16).astype(int) * 16
    m[-1] += rows - m.sum(); return np.concatenate([[0], np.cumsum(m)]).astype(np.int32)
idx, _ = synth.routing(16384, synth.BASE_SEED)
cnt = np.bincount(idx.numpy().ravel(), minlength=256)
layer = np.concatenate([[0], np.cumsum((cnt + 15) // 16 * 16)]).astype(np.int32)   # whole-layer experts
g0 = np.concatenate([[0], np.cumsum(((cnt + 15) // 16 * 16)[:32])]).astype(np.int32)
shapes = [(2048, 7168, 1), (4096, 7168, 1), (16384, 7168, 1), (int(g0[-1]), 2048, g0), (int(g0[-1]), 7168, g0),
          (65536, 7168, 1), (int(layer[-1]), 2048, layer), (int(layer[-1]), 7168, layer)]
if len(sys.argv) > 1 and sys.argv[1] == "big":
    shapes = shapes[-3:]
    sys.argv.pop(1)
for rows, cols, nseg in shapes:
    q = torch.empty(rows, cols, dtype=torch.uint8, device=dev)
    s = torch.empty(cols // 128, rows, dtype=torch.uint8, device=dev)
    for r0 in range(0, rows, 16384):
        r1 = min(rows, r0 + 16384)
        x = synth.activations_bf16_device(r1 - r0, cols, 7 + r0, dev)
        F.fp8flow_quantize_rowwise(x, q[r0:r1], s[:, r0:r1])
        del x
    seg = nseg if isinstance(nseg, np.ndarray) else (segs(rows, nseg) if nseg > 1 else None)
    nseg = 1 if seg is None else len(seg) - 1
    seg_t = torch.from_numpy(seg).to(dev) if seg is not None else None
    qT = torch.empty(rows * cols, dtype=torch.uint8, device=dev)
    sT = torch.empty(rows // 128 + nseg, cols, dtype=torch.uint8, device=dev)
    nb = RL.transpose_bytes(np.diff(seg) if seg is not None else [rows], cols)
    line = []
    ref = None
    for v in sys.argv[1:]:
        os.environ["A2R"] = v
        fn = lambda: F.fp8flow_scaling_aware_transpose(q, s, qT, sT, seg_offsets=seg_t)
        t = marginal(fn, K=20 if rows < 60000 else 6)
        fn(); torch.cuda.synchronize()
        h = (qT.sum().item(), sT.sum().item())
        ref = ref or h
        line.append(f"v{v} {t:.2f}us {nb/t*1e-3/peak:.3f}{'' if h == ref else ' MISMATCH'}")
    print(rows, cols, nseg, " | ".join(line), flush=True)
    del q, s, qT, sT
