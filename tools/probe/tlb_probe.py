"""Is the ~7.7 us fixed cost of a cold single launch the TLB?  Probe read of 29.5/59/118 MB after
(a) the bench flush, (b) the flush + a touch of one word per 2 MB page of the input (TLB warm, L2
still cold: 4 bytes per page), (c) a smaller flush (160 MB write + 160 MB read); plus a tiny
kernel under each."""
import ctypes, os, statistics
import torch
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstreamprobe.so"))
dev = torch.device("cuda:0")
big_w = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
big_r = torch.ones(64 << 20, dtype=torch.float32, device=dev)
sm_w = torch.empty(160 << 20, dtype=torch.uint8, device=dev)
sm_r = torch.ones(40 << 20, dtype=torch.float32, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
out = torch.zeros(4, dtype=torch.int32, device=dev)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
def meas(fn, prep, reps=50):
    fn(); ts = []
    for _ in range(reps):
        prep(); torch.cuda._sleep(200_000)
        ev[0].record(); fn(); ev[1].record(); ev[1].synchronize()
        ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
    return statistics.mean(ts)
tiny = torch.zeros(1, device=dev)
for mb in (29.5, 59, 118):
    nb = int(mb * 1e6) // 4096 * 4096
    a = torch.ones(nb // 4, dtype=torch.int32, device=dev)
    rd = lambda: L.probe_read(ctypes.c_void_p(a.data_ptr()), ctypes.c_int64(nb), ctypes.c_void_p(out.data_ptr()), 1184, 4, st)
    touch = lambda: L.probe_touch(ctypes.c_void_p(a.data_ptr()), ctypes.c_int64(nb), ctypes.c_int64(2 << 20), ctypes.c_void_p(out.data_ptr()), st)
    touch_tiny = lambda: L.probe_touch(ctypes.c_void_p(tiny.data_ptr()), ctypes.c_int64(4), ctypes.c_int64(2 << 20), ctypes.c_void_p(out.data_ptr()), st)
    fl_big = lambda: (big_w.fill_(1), big_r.sum())
    fl_sm = lambda: (sm_w.fill_(1), sm_r.sum())
    r = dict(
        bigflush=meas(rd, fl_big), bigflush_touch=meas(rd, lambda: (fl_big(), touch())),
        smallflush=meas(rd, fl_sm), noflush=meas(rd, lambda: None),
        tiny_bigflush=meas(lambda: tiny.add_(1), fl_big), tiny_bigflush_touch=meas(lambda: tiny.add_(1), lambda: (fl_big(), touch_tiny())),
        tiny_noflush=meas(lambda: tiny.add_(1), lambda: None))
    print(mb, {k: round(v, 2) for k, v in r.items()}, flush=True)
    del a
