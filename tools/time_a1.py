"""Times A1 (quantize) variants on bench.py's x shard and the cfg-2 shape, L2 flushed, and checks
that the variants agree bit for bit.  Usage: python tools/time_a1.py"""
import os
import statistics
import sys

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
    return statistics.median(ts)


for rows, cols in [(2048, 7168), (4096, 7168), (16384, 7168)]:
    x = synth.activations_bf16_device(rows, cols, 5, dev)
    outs = {}
    for var, sched in [("0", "0"), ("5", "0"), ("1", "0")]:
        os.environ["FP8FLOW_A1_VARIANT"] = var
        os.environ["FP8FLOW_SCHED_A1"] = sched
        q = torch.empty(rows, cols, dtype=torch.uint8, device=dev)
        s = torch.empty(cols // 128, rows, dtype=torch.uint8, device=dev)
        ms = timed(lambda: F.fp8flow_quantize_rowwise(x, q, s))
        nb = RL.quantize_bytes(rows, cols)
        outs[(var, sched)] = (q.clone(), s.clone())
        print(f"A1 {rows}x{cols} variant {var} sched {sched}: {ms * 1e3:7.2f} us  {nb / ms / 1e6:7.1f} GB/s  "
              f"frac {nb / ms / 1e6 / peak:.3f}", flush=True)
    ref = outs[("0", "0")]
    for k, (q, s) in outs.items():
        assert torch.equal(q, ref[0]) and torch.equal(s, ref[1]), f"variant {k} differs"
print("variants bit-identical")
