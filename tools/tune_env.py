"""Tuning experiment (not product): for each FP8FLOW_* environment setting given on the command
line (e.g. "A2_VARIANT=1,CTAS_PER_SM_A4=2"), the isolated op times (serial pass) and the
concurrent step time of bench.py's workload."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402


def main(settings):
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    hw = bench.HostWorkload(0)
    ds = bench.DeviceStep(hw, dev)
    nb = hw.op_bytes()
    for setting in settings:
        env = dict(kv.split("=") for kv in setting.split(",") if kv)
        for k, v in env.items():
            os.environ["FP8FLOW_" + k] = v
        for _ in range(3):
            ds.timed_step_concurrent()
            ds.timed_step()
        conc = statistics.median(ds.timed_step_concurrent() for _ in range(15))
        ser = [ds.timed_step() for _ in range(15)]
        ops = {op: statistics.median(p[i] for p in ser) for i, op in enumerate(bench.OPS)}
        txt = "  ".join(f"{op.split('_', 1)[1]} {ops[op]*1e3:.1f}" for op in bench.OPS)
        print(f"{setting or 'default':40s} concurrent {conc*1e3:7.1f} us ({sum(nb.values())/conc/1e6:.0f} GB/s) "
              f"serial {statistics.median(sum(p) for p in ser)*1e3:7.1f} us | {txt}", flush=True)
        for k in env:
            del os.environ["FP8FLOW_" + k]


if __name__ == "__main__":
    main(sys.argv[1:] or [""])
