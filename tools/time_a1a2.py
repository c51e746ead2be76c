"""Timing driver (not product): A1 quantize, A2 scaling-aware transpose and the naive comparator
alone at several shapes, each launch after a clean L2 flush (256 MiB write + 256 MiB read, as
bench.py), median of N CUDA-event-timed launches; plus hot-L2 times (no flush, back to back).
    python tools/time_a1a2.py [reps]"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_02302_b200 import fp8flow as F  # noqa: E402
from paper_2511_02302_b200 import roofline as RL  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 6650.0
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
clean = torch.ones(64 << 20, dtype=torch.float32, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def med(fn, hot=False):
    fn()
    ts = []
    for _ in range(reps):
        if not hot:
            flush.fill_(1)
            clean.sum()
        torch.cuda._sleep(200_000)
        ev[0].record()
        fn()
        ev[1].record()
        ev[1].synchronize()
        ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
    return statistics.median(ts)


out = []
for rows, cols in [(2048, 7168), (4096, 7168), (16384, 7168), (15872, 2048), (65536, 7168)]:
    x = synth.activations_bf16_device(rows, cols, synth.BASE_SEED + 1, dev)
    q = torch.empty(rows, cols, dtype=torch.uint8, device=dev)
    s = torch.empty(cols // 128, rows, dtype=torch.uint8, device=dev)
    qT = torch.empty(rows * cols, dtype=torch.uint8, device=dev)
    sT = torch.empty(rows // 128 + 1, cols, dtype=torch.uint8, device=dev)
    ws = torch.empty(F.fp8flow_naive_workspace_bytes(rows, cols, 1), dtype=torch.uint8, device=dev)
    b1 = RL.quantize_bytes(rows, cols)
    b2 = RL.transpose_bytes([rows], cols)
    r = dict(shape=[rows, cols])
    for name, fn, nb in (("A1", lambda: F.fp8flow_quantize_rowwise(x, q, s), b1),
                         ("A2", lambda: F.fp8flow_scaling_aware_transpose(q, s, qT, sT), b2),
                         ("naive", lambda: F.fp8flow_naive_transpose(q, s, qT, sT, ws), b2)):
        us = med(fn)
        hot = med(fn, hot=True)
        r[name] = dict(us=round(us, 2), frac=round(nb / us * 1e-3 / peak, 3), hot_us=round(hot, 2))
    out.append(r)
    print(json.dumps(r), flush=True)
    del x, q, s, qT, sT, ws
