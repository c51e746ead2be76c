"""Profiling driver (not product): one launch of the fused permute + transpose (and the unfused move and
A2 beside it) on bench.py's whole-layer workload, between cudaProfilerStart/Stop."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
mode = sys.argv[1] if len(sys.argv) > 1 else "balanced"
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
wl = bench.Workload(0, 1, mode, dev)
ds = bench.DeviceStep(wl)
ds.launch_ops(record=False)
F = ds.F
pd = lambda: F.fp8flow_permute_pad_dual(wl.q_recv, wl.s_recv, ds.src, ds.off, ds.x_perm, ds.s_perm, ds.xT, ds.sxT)
pd()
torch.cuda.synchronize()
torch.cuda.profiler.start()
pd()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled permute_pad_dual", mode)
