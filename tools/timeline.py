"""Tuning experiment (not product): per-kernel start/end times (CUDA events on each kernel's own
stream) inside bench.py's concurrent step, to see how the DAG's kernels overlap."""
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
    F, E = ds.F, hw.E_loc
    main_s = torch.cuda.current_stream()
    s1, s2, s3 = ds.side
    names = ["A1_x", "A1_dy", "plan", "A5", "A2_a", "A4", "move", "A2_x"]
    evs = {n: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for n in names}

    def run(name, stream, fn):
        evs[name][0].record(stream)
        fn()
        evs[name][1].record(stream)

    res = {n: [] for n in names}
    tot = []
    for it in range(12):
        ds.flush_l2()
        torch.cuda._sleep(2_000_000)
        ds.ev_start.record(main_s)
        s1.wait_event(ds.ev_start)
        run("A1_x", s1, lambda: F.fp8flow_quantize_rowwise(ds.x_shard, ds.q_x, ds.s_x, stream=s1))
        run("A1_dy", s1, lambda: F.fp8flow_quantize_rowwise(ds.dy_shard, ds.q_dy, ds.s_dy, stream=s1))
        ds.ev_side[0].record(s1)
        run("plan", main_s, lambda: F.fp8flow_permute_plan(ds.topk, hw.e0, E, bench.ALIGN, ds.row_map, ds.src, ds.off,
                                                          ds.ws, stream=main_s))
        ds.ev_plan.record(main_s)
        s2.wait_event(ds.ev_plan)
        s3.wait_event(ds.ev_plan)
        run("A5", s2, lambda: F.fp8flow_swiglu_quant(ds.h, ds.q_a, ds.s_a, rows_dev=ds.off[E:], stream=s2))
        run("A2_a", s2, lambda: F.fp8flow_scaling_aware_transpose(ds.q_a, ds.s_a, ds.aT, ds.saT, seg_offsets=ds.off,
                                                                 stream=s2))
        ds.ev_side[1].record(s2)
        run("A4", s3, lambda: F.fp8flow_unpermute_unpad(ds.y, ds.row_map, ds.probs, ds.y_tok, stream=s3))
        ds.ev_side[2].record(s3)
        run("move", main_s, lambda: F.fp8flow_permute_pad(ds.q_recv, ds.s_recv, ds.src, ds.off, ds.x_perm, ds.s_perm,
                                                         stream=main_s))
        run("A2_x", main_s, lambda: F.fp8flow_scaling_aware_transpose(ds.x_perm, ds.s_perm, ds.xT, ds.sxT,
                                                                     seg_offsets=ds.off, stream=main_s))
        for e in ds.ev_side:
            main_s.wait_event(e)
        ds.ev_end.record(main_s)
        ds.ev_end.synchronize()
        if it >= 2:
            for n in names:
                res[n].append((ds.ev_start.elapsed_time(evs[n][0]) * 1e3, ds.ev_start.elapsed_time(evs[n][1]) * 1e3))
            tot.append(ds.ev_start.elapsed_time(ds.ev_end) * 1e3)
    print(f"step {statistics.median(tot):.1f} us")
    for n in names:
        s = statistics.median(a for a, _ in res[n])
        e = statistics.median(b for _, b in res[n])
        print(f"  {n:6s} start {s:7.1f}  end {e:7.1f}  span {e - s:6.1f}  " + " " * int(s / 4) + "#" * max(1, int((e - s) / 4)))


if __name__ == "__main__":
    main()
