"""Times A5 (fused SwiGLU + quant) and NEXT-1 (fused SwiGLU backward + quant) alone on bench.py's
shape, L2 flushed before each launch.
Usage: python tools/time_swiglu.py [KNOB=V,KNOB=V ...]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_02302_b200 import fp8flow as F, roofline as RL  # noqa: E402

R, FFN = 15872, 2048
dev = torch.device("cuda:0")
h = synth.normal_bf16(R, 2 * FFN, synth.BASE_SEED + 3, sigma=1.5).to(dev)
dA = synth.normal_bf16(R, FFN, synth.BASE_SEED + 5, sigma=0.5).to(dev)
q = torch.empty(R, 2 * FFN, dtype=torch.uint8, device=dev)
s = torch.empty(2 * FFN // 128, R, dtype=torch.uint8, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
clean = torch.ones(64 << 20, dtype=torch.float32, device=dev)
qf = torch.empty(R, FFN, dtype=torch.uint8, device=dev)
sf = torch.empty(FFN // 128, R, dtype=torch.uint8, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
peak = RL.measured_peaks(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))["hbm_gbs"]


def timed(fn, nb, name):
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
    print(f"{name} {R}x{FFN}: {ms*1e3:.2f} us  {nb/ms/1e6:.1f} GB/s  frac {nb/ms/1e6/peak:.3f}")


for setting in [a for a in sys.argv[1:] if not a.startswith("--")] or [""]:
    for kv in filter(None, setting.split(",")):  # FP8FLOW_* knobs, e.g. A5_SLEEP_NS=0,CTAS_PER_SM_A5=2
        k, v = kv.split("=")
        os.environ["FP8FLOW_" + k] = v
    print(f"[{setting}]")
    timed(lambda: F.fp8flow_swiglu_quant(h, qf, sf), RL.swiglu_quant_bytes(R, FFN), "A5 swiglu_quant")
    timed(lambda: F.fp8flow_swiglu_bwd_quant(h, dA, q, s), RL.swiglu_bwd_quant_bytes(R, FFN), "NEXT1 swiglu_bwd_quant")
# (code/scale parity against the oracle lives in tests/test_gpu_parity.py; tools/ never load oracle/)
