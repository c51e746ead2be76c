import ctypes, os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth
from paper_2511_02302_b200 import fp8flow as F
from paper_2511_02302_b200 import roofline as RL
dev = torch.device("cuda:0")
fw = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
fr = torch.ones(64 << 20, dtype=torch.float32, device=dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
def flush():
    fw.fill_(1); fr.sum()
def marginal(fn, K=20, reps=5):
    fn(); res = []
    for _ in range(reps):
        tt = []
        for with_op in (True, False):
            torch.cuda.synchronize(); torch.cuda._sleep(30_000_000)
            ev[0].record()
            for _ in range(K):
                flush()
                if with_op: fn()
            ev[1].record(); ev[1].synchronize()
            tt.append(ev[0].elapsed_time(ev[1]) * 1e3)
        res.append((tt[0] - tt[1]) / K)
    return statistics.median(res)
peak = 6551.7
for rows, cols in [(2048, 7168), (4096, 7168), (16384, 7168), (65536, 7168)]:
    x = synth.activations_bf16_device(rows, cols, 7, dev)
    q = torch.empty(rows, cols, dtype=torch.uint8, device=dev)
    s = torch.empty(cols // 128, rows, dtype=torch.uint8, device=dev)
    nb = RL.quantize_bytes(rows, cols)
    line = []
    for v in sys.argv[1:]:
        os.environ["A1H"] = v
        t = marginal(lambda: F.fp8flow_quantize_rowwise(x, q, s), K=20 if rows < 60000 else 6)
        line.append(f"v{v} {t:.2f}us {nb/t*1e-3/peak:.3f}")
    print(rows, cols, " | ".join(line), flush=True)
    del x, q, s
