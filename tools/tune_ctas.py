"""Tuning experiment (not product): CTAs per SM (shared-memory budget split) of the bulk-copy /
TMA kernels A3-move, A4, A5 -- isolated op time and the concurrent step time."""
import itertools
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
    for a3, a4, a5 in [(2, 2, 1), (3, 3, 1), (4, 4, 1), (2, 3, 1), (3, 2, 1), (4, 2, 1), (2, 4, 1)]:
        os.environ["FP8FLOW_CTAS_PER_SM_A3"] = str(a3)
        os.environ["FP8FLOW_CTAS_PER_SM_A4"] = str(a4)
        os.environ["FP8FLOW_CTAS_PER_SM_A5"] = str(a5)
        for _ in range(3):
            ds.timed_step_concurrent()
            ds.timed_step()
        conc = statistics.median(ds.timed_step_concurrent() for _ in range(15))
        ser = [ds.timed_step() for _ in range(15)]
        ops = {op: statistics.median(p[i] for p in ser) * 1e3 for i, op in enumerate(bench.OPS)}
        print(f"A3={a3} A4={a4} A5={a5}: concurrent {conc*1e3:7.1f} us  serial {statistics.median(sum(p) for p in ser)*1e3:7.1f} us"
              f"  move {ops['A3_move']:.1f}  A5 {ops['A5_swiglu_quant']:.1f}  A4 {ops['A4_unpermute']:.1f}", flush=True)


if __name__ == "__main__":
    main()
