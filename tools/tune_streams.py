"""Tuning experiment (not product): bench.py's concurrent step under different stream layouts and
stream priorities -- which kernels of the DAG share a stream, and whether the longest chain
(plan -> move -> A2(X_perm)) gets a high-priority stream.  Median of 15 L2-flushed steps each."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    hw = bench.HostWorkload(0)
    ds = bench.DeviceStep(hw, dev)
    F = ds.F
    lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
    print(f"stream priority range (low, high) = ({lo}, {hi})")
    ev_start, ev_end, ev_plan = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                                 torch.cuda.Event())
    done = [torch.cuda.Event() for _ in range(5)]

    def make(p_crit, p_a1, p_a5, p_a4, split_a1):
        crit = torch.cuda.Stream(dev, priority=p_crit)
        s_a1x = torch.cuda.Stream(dev, priority=p_a1)
        s_a1d = torch.cuda.Stream(dev, priority=p_a1) if split_a1 else s_a1x
        s_a5 = torch.cuda.Stream(dev, priority=p_a5)
        s_a4 = torch.cuda.Stream(dev, priority=p_a4)

        def step():
            main = torch.cuda.current_stream()
            ev_start.record(main)
            for s in (crit, s_a1x, s_a1d, s_a5, s_a4):
                s.wait_event(ev_start)
            F.fp8flow_permute_plan(ds.topk, hw.e0, hw.E_loc, bench.ALIGN, ds.row_map, ds.src, ds.off, ds.ws, stream=crit)
            ev_plan.record(crit)
            F.fp8flow_quantize_rowwise(ds.x_shard, ds.q_x, ds.s_x, stream=s_a1x)
            F.fp8flow_quantize_rowwise(ds.dy_shard, ds.q_dy, ds.s_dy, stream=s_a1d)
            s_a5.wait_event(ev_plan)
            s_a4.wait_event(ev_plan)
            F.fp8flow_swiglu_quant(ds.h, ds.q_a, ds.s_a, rows_dev=ds.off[hw.E_loc:], stream=s_a5)
            F.fp8flow_scaling_aware_transpose(ds.q_a, ds.s_a, ds.aT, ds.saT, seg_offsets=ds.off, stream=s_a5)
            F.fp8flow_unpermute_unpad(ds.y, ds.row_map, ds.probs, ds.y_tok, stream=s_a4)
            F.fp8flow_permute_pad(ds.q_recv, ds.s_recv, ds.src, ds.off, ds.x_perm, ds.s_perm, stream=crit)
            F.fp8flow_scaling_aware_transpose(ds.x_perm, ds.s_perm, ds.xT, ds.sxT, seg_offsets=ds.off, stream=crit)
            for e, s in zip(done, (crit, s_a1x, s_a1d, s_a5, s_a4)):
                e.record(s)
                main.wait_event(e)
            ev_end.record(main)

        return step

    variants = {
        "baseline-like (A1s shared, no prio)": (0, 0, 0, 0, False),
        "A1s split": (0, 0, 0, 0, True),
        "A1s split, crit high": (hi, 0, 0, 0, True),
        "A1s split, crit+A5 high": (hi, 0, hi, 0, True),
        "A1s shared, crit high": (hi, 0, 0, 0, False),
        "A1s split, A4 low (crit, A5 high)": (hi, 0, hi, 0, True),
    }
    for name, cfg in variants.items():
        step = make(*cfg)
        ts = []
        for i in range(20):
            ds.flush_l2()
            torch.cuda._sleep(2_000_000)
            step()
            ev_end.synchronize()
            if i >= 5:
                ts.append(ev_start.elapsed_time(ev_end))
        ms = statistics.median(ts)
        print(f"{name:40s} {ms * 1e3:7.1f} us  {sum(hw.op_bytes().values()) / ms / 1e6:7.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
