"""Floor of a streaming kernel for the byte volumes of A1 / A2 launches, timed like bench.py's
marginal cold-L2 cost (K x [flush, op] - K x [flush]).  Not product."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstreamprobe.so"))
dev = torch.device("cuda:0")
fw = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
fr = torch.ones(64 << 20, dtype=torch.float32, device=dev)
flush = lambda: (fw.zero_(), fr.sum())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
peak = 6551.7
for rows, cols in [(2048, 7168), (4096, 7168), (16384, 7168)]:
    n = rows * cols
    a = torch.ones(2 * n // 4, dtype=torch.int32, device=dev)
    o = torch.empty(n // 4, dtype=torch.int32, device=dev)
    out = {}
    for grid in (592, 1184, 2368):
        t_rw = bench.marginal_us(lambda: L.probe_rw(ctypes.c_void_p(a.data_ptr()), ctypes.c_int64(n), ctypes.c_void_p(o.data_ptr()), grid, 2, st), flush)
        t_cp = bench.marginal_us(lambda: L.probe_copy(ctypes.c_void_p(a.data_ptr()), ctypes.c_int64(n), ctypes.c_void_p(o.data_ptr()), grid, st), flush)
        out[grid] = (round(t_rw, 2), round(t_cp, 2))
    best_rw = min(v[0] for v in out.values()); best_cp = min(v[1] for v in out.values())
    print(f"{rows}x{cols}: A1-shaped (2n read, n write) best {best_rw} us = {3 * n / best_rw / 1e3 / peak:.3f}; "
          f"A2-shaped copy (n read, n write) best {best_cp} us = {2 * n / best_cp / 1e3 / peak:.3f}  {out}", flush=True)
