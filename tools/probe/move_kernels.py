"""A3 move at bench.py's workload sizes with each dispatch kernel (n = 1 peer = the rank itself):
marginal cold-L2 us.  Not product.   python tools/probe/move_kernels.py [balanced|weak]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
mode = sys.argv[1] if len(sys.argv) > 1 else "balanced"
dev = torch.device("cuda", 0)
wl = bench.Workload(0, 1, mode, dev)
ds = bench.DeviceStep(wl)
ds.launch_ops(record=False)
torch.cuda.synchronize()
F = ds.F
nb = wl.op_bytes()["A3_move"]
peak = bench.RL.measured_peaks(bench.ROOT)["hbm_gbs"]
ref = ds.x_perm.clone(), ds.s_perm.clone()
for name, k in (("auto", F.DISPATCH_AUTO), ("engine", F.DISPATCH_ENGINE), ("register", F.DISPATCH_REGISTER)):
    fn = lambda: F.fp8flow_dispatch_permute_pad([wl.q_recv.data_ptr()], [wl.s_recv.data_ptr()], wl.s_recv.shape[1],
                                                wl.T_recv, bench.HIDDEN, ds.row_map, ds.src, ds.off, ds.x_perm,
                                                ds.s_perm, kernel=k)
    us = bench.marginal_us(fn, ds.flush_l2)
    torch.cuda.synchronize()
    same = torch.equal(ds.x_perm, ref[0]) and torch.equal(ds.s_perm, ref[1])
    print(f"{mode} {name:9s} {us:8.2f} us  {nb / us / 1e3 / peak:.3f}  same={same}", flush=True)
