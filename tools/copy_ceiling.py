"""Calibration (not product): achievable HBM GB/s of torch's device copy (read+write bytes) at the
byte volumes of the hot-path ops, L2 flushed before each copy (write flush vs write+read flush),
CUDA events, median of 15."""
import statistics
import torch

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush2 = torch.ones(64 << 20, dtype=torch.float32, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def do_flush(mode):
    flush.zero_()
    if mode == "write+read":
        flush2.sum()


for mode in ("write", "write+read"):
    for total_mb in (44, 88, 172, 338, 1000):
        n = total_mb * (1 << 20) // 2
        a = torch.empty(n, dtype=torch.uint8, device=dev)
        b = torch.empty(n, dtype=torch.uint8, device=dev)
        b.copy_(a)
        ts = []
        for _ in range(15):
            do_flush(mode)
            torch.cuda._sleep(1_000_000)
            ev[0].record()
            b.copy_(a)
            ev[1].record()
            ev[1].synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
        ms = statistics.median(ts)
        print(f"{mode:11s} copy {total_mb:5d} MB moved: {ms*1e3:8.2f} us  {2*n/ms/1e6:8.1f} GB/s", flush=True)
