"""DRAM write ceiling of the A3 move's pattern (not product): the permute plan's output rows
(bench.py whole-layer balanced workload, 131072 rows x 7168 B) written in the plan's row_map order
(token-major: each token's 8 rows spread over its experts), warp per row, vs the same rows in
ascending order; marginal cold-L2 us.   python tools/probe/scatter_probe.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstreamprobe.so"))
dev = torch.device("cuda", 0)
ds = bench.DeviceStep(bench.Workload(0, 1, "balanced", dev))
ds.launch_ops(record=False)
torch.cuda.synchronize()
H = bench.HIDDEN
order = ds.row_map.flatten().contiguous()
valid = order[order >= 0]
srt = torch.sort(valid).values.to(torch.int32).contiguous()
out = ds.x_perm
nb = valid.numel() * H
for name, o in (("plan order", order), ("ascending", srt)):
    for grid in (592, 1184, 2368, 4736):
        fn = lambda: L.probe_scatter_rows(ctypes.c_void_p(o.data_ptr()), ctypes.c_int64(o.numel()), ctypes.c_int64(H),
                                          ctypes.c_void_p(out.data_ptr()), grid, None)
        us = bench.marginal_us(fn, ds.flush_l2)
        print(f"{name:11s} grid {grid:5d}: {us:7.1f} us  {nb / us / 1e3:7.0f} GB/s", flush=True)
