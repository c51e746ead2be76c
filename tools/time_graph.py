"""Experiment: the concurrent step launched stream by stream vs replayed from a CUDA graph
(median of 20 L2-flushed steps each), and a parity check of the graph's outputs."""
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
    nb = sum(hw.op_bytes().values())
    for _ in range(3):
        ds.timed_step_concurrent()
    ds.capture_graph()
    for _ in range(3):
        ds.timed_step_graph()
    for name, fn in (("streams", ds.timed_step_concurrent), ("graph", ds.timed_step_graph),
                     ("streams", ds.timed_step_concurrent), ("graph", ds.timed_step_graph)):
        ts = [fn() for _ in range(20)]
        ms = statistics.median(ts)
        print(f"{name:8s} {ms * 1e3:7.1f} us  {nb / ms / 1e6:7.1f} GB/s", flush=True)
    # the replayed outputs must equal a fresh eager launch of the same step (device checksums;
    # oracle parity of these outputs is the job of tests/ and bench.py's cpu_baseline leg)
    after_graph = ds.checksums()
    ds.launch_ops(record=False)
    torch.cuda.synchronize()
    print("graph replay == eager step:", after_graph == ds.checksums())


if __name__ == "__main__":
    main()
