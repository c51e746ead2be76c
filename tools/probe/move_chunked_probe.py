"""Compares the A3 move (dispatch engine, fp8flow_permute_pad) with a column-chunked row-gather move
(tools/probe/move_chunked_probe.cu) on bench.py's whole-layer workload: marginal cold-L2 us and
byte equality of X_perm and its scales.  Not product."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmoveprobe.so"))
dev = torch.device("cuda", 0)
mode = sys.argv[1] if len(sys.argv) > 1 else "balanced"
wl = bench.Workload(0, 1, mode, dev)
ds = bench.DeviceStep(wl)
ds.launch_ops(record=False)
torch.cuda.synchronize()
fns = ds.op_fns()
ref_q, ref_s = ds.x_perm.clone(), ds.s_perm.clone()
R = int(ds.off[-1].item())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
t_eng = bench.marginal_us(fns["A3_move"], ds.flush_l2)
print(f"{mode}: engine {t_eng:.1f} us", flush=True)
for ch in (512, 1024, 3584, 7168):
    for grid in (148 * 8, 148 * 16, 148 * 32):
        fn = lambda: L.probe_move_chunked(P(wl.q_recv), P(wl.s_recv), ctypes.c_int64(wl.s_recv.shape[1]),
                                          ctypes.c_int64(bench.HIDDEN), P(ds.src), ctypes.c_int64(R),
                                          ctypes.c_int64(ds.x_perm.shape[0]), P(ds.x_perm), P(ds.s_perm), ch, grid, st)
        ds.x_perm.fill_(0xEE); ds.s_perm.fill_(0xEE)
        fn(); torch.cuda.synchronize()
        ok = torch.equal(ds.x_perm[:R], ref_q[:R]) and torch.equal(ds.s_perm[:, :R], ref_s[:, :R])
        t = bench.marginal_us(fn, ds.flush_l2)
        print(f"  chunk {ch} grid {grid}: {t:.1f} us  identical={ok}", flush=True)
