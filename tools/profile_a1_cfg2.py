import os, sys, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2511_02302_b200 import fp8flow as F
dev = torch.device("cuda:0")
x = synth.activations_bf16_device(4096, 7168, 5, dev)
q = torch.empty(4096, 7168, dtype=torch.uint8, device=dev)
s = torch.empty(56, 4096, dtype=torch.uint8, device=dev)
for _ in range(3): F.fp8flow_quantize_rowwise(x, q, s)
torch.cuda.synchronize()
torch.cuda.profiler.start()
F.fp8flow_quantize_rowwise(x, q, s)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
