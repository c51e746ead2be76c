"""Runs tile_read_probe.cu (not product): marginal cold-L2 us of reading a u8 matrix in A2's 128x128
tile order by TMA boxes (stages x CTAs/SM) vs coalesced LDG (U tiles in flight x CTAs/SM), beside
the plain streaming read of the same bytes (stream_probe.cu)."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
here = os.path.dirname(os.path.abspath(__file__))
T = ctypes.CDLL(os.path.join(here, "libtilereadprobe.so"))
S = ctypes.CDLL(os.path.join(here, "libstreamprobe.so"))
dev = torch.device("cuda:0")
fw = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
fr = torch.ones(64 << 20, dtype=torch.float32, device=dev)
flush = lambda: (fw.fill_(1), fr.sum())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
out = torch.zeros(4, dtype=torch.int32, device=dev)
op = ctypes.c_void_p(out.data_ptr())
for rows, cols in [(4096, 7168), (16384, 7168), (65536, 7168)]:
    q = torch.ones(rows * cols, dtype=torch.uint8, device=dev)
    qp = ctypes.c_void_p(q.data_ptr())
    n = rows * cols
    res = {}
    res["stream"] = min(bench.marginal_us(lambda: S.probe_read(qp, ctypes.c_int64(n), op, g, 4, st), flush, K=20) for g in (592, 1184))
    for stages, cps in ((2, 3), (3, 3), (4, 3), (6, 2), (12, 1), (4, 2), (3, 4)):
        res[f"tma{stages}x{cps}"] = bench.marginal_us(lambda: T.probe_tma_read(qp, rows, cols, op, stages, cps, st), flush, K=20)
    for u, cps in ((1, 4), (2, 4), (4, 4), (2, 8), (1, 8), (4, 2)):
        res[f"ldg{u}x{cps}"] = bench.marginal_us(lambda: T.probe_ldg_read(qp, rows, cols, op, u, cps, st), flush, K=20)
    print(f"{rows}x{cols} {n/1e6:.1f} MB: " + " ".join(f"{k}={v:.2f}us({n/v*1e-3/6551.7:.2f})" for k, v in res.items()), flush=True)
    del q
