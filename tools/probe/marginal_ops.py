"""Marginal cold-L2 cost of each step op of bench.py's workload (not product):
    python tools/probe/marginal_ops.py [strong|weak] [op ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
mode = sys.argv[1] if len(sys.argv) > 1 else "strong"
want = sys.argv[2:]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
wl = bench.Workload(0, 1, mode, dev)
ds = bench.DeviceStep(wl)
ds.launch_ops(record=False)
torch.cuda.synchronize()
nb = wl.op_bytes()
peak = bench.RL.measured_peaks(bench.ROOT)["hbm_gbs"]
for op, fn in ds.op_fns().items():
    if want and op not in want:
        continue
    us = bench.marginal_us(fn, ds.flush_l2)
    print(f"{op:20s} {us:8.2f} us  {nb[op] / us / 1e3 / peak:.3f}", flush=True)
