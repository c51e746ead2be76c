"""Times the A3 plan (cooperative single launch vs the 2-kernel path) on the step's routing
(expert group 0: 7939 received tokens) and on NEXT-3's global plan (16384 tokens, 32 local
experts), L2 flushed.  Usage: python tools/time_plan.py"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_02302_b200 import fp8flow as F  # noqa: E402

dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
clean = torch.ones(64 << 20, dtype=torch.float32, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(fn, reps=30):
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


idx, probs = synth.routing(16384, synth.BASE_SEED)
sh = synth.expert_shard(idx, probs, 0, 8)
for name, topk in [("step group 0 (received tokens)", torch.from_numpy(sh.topk_idx)), ("NEXT-3 global", idx)]:
    topk = topk.to(dev).contiguous()
    T, K = topk.shape
    E = 32
    mr = F.permute_max_rows(T, K, E)
    rm = torch.empty(T, K, dtype=torch.int32, device=dev)
    src = torch.empty(mr, dtype=torch.int32, device=dev)
    off = torch.empty(E + 1, dtype=torch.int32, device=dev)
    ws = torch.empty(F.fp8flow_permute_workspace_bytes(T, K, E), dtype=torch.uint8, device=dev)
    res = {}
    for fused in ("1", "0"):
        os.environ["FP8FLOW_PLAN_FUSED"] = fused
        ms = timed(lambda: F.fp8flow_permute_plan(topk, 0, E, 16, rm, src, off, ws))
        res[fused] = (rm.clone(), off.clone())
        print(f"plan {name} T={T}: fused={fused} {ms * 1e3:7.2f} us", flush=True)
    assert torch.equal(res["1"][0], res["0"][0]) and torch.equal(res["1"][1], res["0"][1])
    os.environ["FP8FLOW_PLAN_FUSED"] = "1"
    for stop in ("1", "2", "3"):
        os.environ["FP8FLOW_PLAN_STOP"] = stop
        ms = timed(lambda: F.fp8flow_permute_plan(topk, 0, E, 16, rm, src, off, ws))
        print(f"plan {name}: fused, ends after stage {stop}: {ms * 1e3:7.2f} us", flush=True)
    os.environ["FP8FLOW_PLAN_STOP"] = "0"
print("paths agree")
