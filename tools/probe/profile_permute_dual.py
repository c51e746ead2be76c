"""Profiling driver (not product): one launch of a dual-output kernel on bench.py's workload, between
cudaProfilerStart/Stop:  python tools/probe/profile_permute_dual.py [balanced|weak] [permute|swiglu]"""
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
which = sys.argv[2] if len(sys.argv) > 2 else "permute"
if which == "permute":
    pd = lambda: F.fp8flow_permute_pad_dual(wl.q_recv, wl.s_recv, ds.src, ds.off, ds.x_perm, ds.s_perm, ds.xT, ds.sxT)
else:
    pd = lambda: F.fp8flow_swiglu_quant_dual(wl.h, ds.q_a, ds.s_a, ds.aT, ds.saT, seg_offsets=ds.off,
                                             rows_dev=ds.off[wl.E_loc:])
pd()
torch.cuda.synchronize()
torch.cuda.profiler.start()
pd()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled", which, mode)
