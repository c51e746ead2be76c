"""A2 tile order experiment: row-block-major (default) vs column-block-major (the FP8FLOW_A2_COLMAJOR
knob existed only for this experiment; results in profiles/r01_a2_order_experiment.txt, the knob
was removed), on the sweep's large shapes and on the step's ragged X_perm (32 experts), L2
flushed; outputs must be bit-identical.  Usage: python tools/time_a2_order.py"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_02302_b200 import fp8flow as F, roofline as RL  # noqa: E402

KNOB = os.environ.get("A2_KNOB", "FP8FLOW_A2_VARIANT")      # FP8FLOW_A2_COLMAJOR for the order experiment
VARIANTS = os.environ.get("A2_VALUES", "0,1,2,3").split(",")
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
clean = torch.ones(64 << 20, dtype=torch.float32, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
peak = RL.measured_peaks(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))["hbm_gbs"]


def timed(fn, reps=15):
    fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        clean.sum()
        torch.cuda._sleep(1_000_000)
        ev[0].record()
        fn()
        ev[1].record()
        ev[1].synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    return statistics.median(ts)


idx, _ = synth.routing(16384, synth.BASE_SEED)
counts = np.bincount(idx.numpy().ravel(), minlength=256)[:32]
segs = (counts + 15) // 16 * 16
cases = [("4096x7168", 4096, 7168, None), ("16384x7168", 16384, 7168, None), ("32768x7168", 32768, 7168, None),
         ("65536x7168", 65536, 7168, None), ("X_perm 32 experts", int(segs.sum()), 7168, segs),
         ("A 32 experts", int(segs.sum()), 2048, segs)]
for name, rows, cols, sg in cases:
    x = synth.activations_bf16_device(rows, cols, 3, dev)
    q = torch.empty(rows, cols, dtype=torch.uint8, device=dev)
    s = torch.empty(cols // 128, rows, dtype=torch.uint8, device=dev)
    F.fp8flow_quantize_rowwise(x, q, s)
    del x
    off = None if sg is None else torch.from_numpy(np.concatenate([[0], np.cumsum(sg)]).astype(np.int32)).to(dev)
    nseg = 1 if sg is None else len(sg)
    nb = RL.transpose_bytes([rows] if sg is None else [int(v) for v in sg], cols)
    outs = {}
    for order in VARIANTS:
        os.environ[KNOB] = order
        qT = torch.zeros(rows * cols, dtype=torch.uint8, device=dev)
        sT = torch.zeros(rows // 128 + nseg, cols, dtype=torch.uint8, device=dev)
        ms = timed(lambda: F.fp8flow_scaling_aware_transpose(q, s, qT, sT, seg_offsets=off))
        outs[order] = (qT, sT)
        print(f"A2 {name}: {KNOB}={order} {ms * 1e3:8.2f} us  {nb / ms / 1e6:7.1f} GB/s  frac {nb / ms / 1e6 / peak:.3f}",
              flush=True)
    for k in outs:
        assert torch.equal(outs["0"][0], outs[k][0]) and torch.equal(outs["0"][1], outs[k][1]), (name, k)
    del q, s, outs
print("variants bit-identical")
