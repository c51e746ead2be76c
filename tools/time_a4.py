"""Times A4 (unpermute + unpad) on the bench's expert-group-0 workload (16384 tokens, top-8 of 256,
hidden 7168), L2 flushed.  (The register-variant comparison it once ran is recorded in
profiles/r01_a4_lsu_experiment.txt.)  Usage: python tools/time_a4.py"""
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


idx, probs = synth.routing(16384, synth.BASE_SEED)
for group in (0,):
    sh = synth.expert_shard(idx, probs, group, 8)
    topk = torch.from_numpy(sh.topk_idx).to(dev)
    p = torch.from_numpy(sh.probs).to(dev)
    T, K, E = topk.shape[0], topk.shape[1], sh.num_local_experts
    max_rows = F.permute_max_rows(T, K, E)
    rm = torch.empty(T, K, dtype=torch.int32, device=dev)
    src = torch.empty(max_rows, dtype=torch.int32, device=dev)
    off = torch.empty(E + 1, dtype=torch.int32, device=dev)
    ws = torch.empty(F.fp8flow_permute_workspace_bytes(T, K, E), dtype=torch.uint8, device=dev)
    F.fp8flow_permute_plan(topk, sh.expert_begin, E, 16, rm, src, off, ws)
    x = synth.normal_bf16_device(max_rows, 7168, 5, dev)
    valid = int((rm >= 0).sum().item())
    nb = RL.unpermute_bytes(valid, T, K, 7168, True)
    outs = {}
    for var in ["0"]:
        os.environ["FP8FLOW_A4_LSU"] = var
        y = torch.empty(T, 7168, dtype=torch.bfloat16, device=dev)
        ms = timed(lambda: F.fp8flow_unpermute_unpad(x, rm, p, y))
        outs[var] = y.clone()
        print(f"A4 group {group} T={T} valid={valid} LSU={var}: {ms * 1e3:7.2f} us  {nb / ms / 1e6:7.1f} GB/s  "
              f"frac {nb / ms / 1e6 / peak:.3f}", flush=True)
    for k, y in outs.items():
        assert torch.equal(y.view(torch.int16), outs["0"].view(torch.int16)), f"variant {k} differs"
print("variants bit-identical")
