"""Tuning experiment (not part of the product): time each hot-path op of bench.py's workload in
isolation (L2 flushed, CUDA events, median of reps) under every work-item schedule
(FP8FLOW_SCHED_<OP> = 0 one item per warp, 1 blocked, 2 interleaved)."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    reps = int(os.environ.get("REPS", "15"))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    hw = bench.HostWorkload(0)
    ds = bench.DeviceStep(hw, dev)
    F, E = ds.F, hw.E_loc
    ops = {
        "A1": lambda: F.fp8flow_quantize_rowwise(ds.x_shard, ds.q_x, ds.s_x),
        "A3": lambda: F.fp8flow_permute_pad(ds.q_recv, ds.s_recv, ds.src, ds.off, ds.x_perm, ds.s_perm),
        "A5": lambda: F.fp8flow_swiglu_quant(ds.h, ds.q_a, ds.s_a, rows_dev=ds.off[E:]),
        "A4": lambda: F.fp8flow_unpermute_unpad(ds.y, ds.row_map, ds.probs, ds.y_tok),
    }
    nbytes = hw.op_bytes()
    bkey = {"A1": "A1_quantize_x", "A3": "A3_move", "A5": "A5_swiglu_quant", "A4": "A4_unpermute"}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    res = {}
    for op, fn in ops.items():
        for sched in (0, 1, 2):
            os.environ[f"FP8FLOW_SCHED_{op}"] = str(sched)
            fn()
            ts = []
            for _ in range(reps):
                ds.flush_l2()
                torch.cuda._sleep(1_000_000)
                ev[0].record()
                fn()
                ev[1].record()
                ev[1].synchronize()
                ts.append(ev[0].elapsed_time(ev[1]))
            ms = statistics.median(ts)
            res[f"{op}/sched{sched}"] = {"us": round(ms * 1e3, 2), "gbs": round(nbytes[bkey[op]] / ms / 1e6, 1)}
            print(op, sched, res[f"{op}/sched{sched}"], flush=True)
        del os.environ[f"FP8FLOW_SCHED_{op}"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
