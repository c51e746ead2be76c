"""Marginal cold-L2 time of an op: K x [flush, op] vs K x [flush] enqueued behind a long sleep (so
the host never limits), events around the whole sequence; (T_with - T_without) / K.  Compared
with the single-launch method (flush, sleep, event, op, event).  Not product."""
import ctypes, os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth
from paper_2511_02302_b200 import fp8flow as F
from paper_2511_02302_b200 import roofline as RL
L = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libstreamprobe.so"))
dev = torch.device("cuda:0")
fw = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
fr = torch.ones(64 << 20, dtype=torch.float32, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
out = torch.zeros(4, dtype=torch.int32, device=dev)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
def flush():
    fw.fill_(1); fr.sum()
def single(fn, reps=40):
    fn(); ts = []
    for _ in range(reps):
        flush(); torch.cuda._sleep(200_000)
        ev[0].record(); fn(); ev[1].record(); ev[1].synchronize()
        ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
    return statistics.mean(ts)
def marginal(fn, K=20, reps=5):
    fn(); res = []
    for _ in range(reps):
        tt = []
        for with_op in (True, False):
            torch.cuda.synchronize(); torch.cuda._sleep(20_000_000)
            ev[0].record()
            for _ in range(K):
                flush()
                if with_op: fn()
            ev[1].record(); ev[1].synchronize()
            tt.append(ev[0].elapsed_time(ev[1]) * 1e3)
        res.append((tt[0] - tt[1]) / K)
    return statistics.median(res)
peak = 6551.7
for rows, cols in [(2048, 7168), (4096, 7168), (16384, 7168)]:
    x = synth.activations_bf16_device(rows, cols, 7, dev)
    q = torch.empty(rows, cols, dtype=torch.uint8, device=dev)
    s = torch.empty(cols // 128, rows, dtype=torch.uint8, device=dev)
    qT = torch.empty(rows * cols, dtype=torch.uint8, device=dev)
    sT = torch.empty(rows // 128 + 1, cols, dtype=torch.uint8, device=dev)
    F.fp8flow_quantize_rowwise(x, q, s)
    nb1, nb2 = RL.quantize_bytes(rows, cols), RL.transpose_bytes([rows], cols)
    a1 = lambda: F.fp8flow_quantize_rowwise(x, q, s)
    a2 = lambda: F.fp8flow_scaling_aware_transpose(q, s, qT, sT)
    xb = x.view(torch.uint8)
    rw = lambda: L.probe_rw(ctypes.c_void_p(xb.data_ptr()), ctypes.c_int64(rows * cols), ctypes.c_void_p(qT.data_ptr()), 1184, 2, st)
    for name, fn, nb in (("A1", a1, nb1), ("A2", a2, nb2), ("probe_rw_A1bytes", rw, nb1)):
        t1, t2 = single(fn), marginal(fn)
        print(rows, cols, name, f"single {t1:.2f} us ({nb/t1*1e-3/peak:.3f})  marginal {t2:.2f} us ({nb/t2*1e-3/peak:.3f})", flush=True)
