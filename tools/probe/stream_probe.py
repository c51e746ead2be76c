"""Runs the bandwidth probe (stream_probe.cu): cold-L2 (write+read flush) event-timed mean of N
launches, for read-only and A1-shaped (2:1) read/write volumes, over grid sizes.  Not product."""
import ctypes, os, statistics, sys
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstreamprobe.so"))
dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
clean = torch.ones(64 << 20, dtype=torch.float32, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
out = torch.zeros(4, dtype=torch.int32, device=dev)
def meas(fn, reps=50):
    fn(); ts = []
    for _ in range(reps):
        flush.fill_(1); clean.sum(); torch.cuda._sleep(200_000)
        ev[0].record(); fn(); ev[1].record(); ev[1].synchronize()
        ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
    return statistics.mean(ts)
st = torch.cuda.current_stream().cuda_stream
for mb in (29.5, 59, 88.3, 118, 236, 472):
    nb = int(mb * 1e6) // 4096 * 4096
    a = torch.ones(nb // 4, dtype=torch.int32, device=dev)
    o = torch.empty(nb // 8, dtype=torch.int32, device=dev)
    res = []
    for grid in (148 * 4, 148 * 8, 148 * 16):
        for u in (4, 8):
            t = meas(lambda: L.probe_read(ctypes.c_void_p(a.data_ptr()), ctypes.c_int64(nb), ctypes.c_void_p(out.data_ptr()), grid, u, ctypes.c_void_p(st)))
            res.append(f"read g{grid}u{u} {t:.2f}us {nb/t*1e-3:.0f}GB/s")
    for grid in (148 * 4, 148 * 8):
        for u in (2, 4):
            t = meas(lambda: L.probe_rw(ctypes.c_void_p(a.data_ptr()), ctypes.c_int64(nb // 2), ctypes.c_void_p(o.data_ptr()), grid, u, ctypes.c_void_p(st)))
            res.append(f"rw2:1 g{grid}u{u} {t:.2f}us {1.5*nb/t*1e-3:.0f}GB/s")
    print(mb, "MB read:", " | ".join(res), flush=True)
    del a, o
