"""NEXT-1 dual-output kernels vs the two launches they replace, marginal cold-L2 us (not product):
A1 / A2 / A1->A2 / quantize_dual at 4096x7168 and 16384x7168 (one segment); A5 / A2 / A5->A2 /
swiglu_quant_dual at bench.py's EP8 group-0 shape (15872 rows, F = 2048, 32 experts).
    python tools/probe/marginal_dual.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import synth
from paper_2511_02302_b200 import roofline as RL
dev = torch.device("cuda", 0)
ds = bench.DeviceStep(bench.Workload(0, 1, "weak", dev))
ds.launch_ops(record=False)
F, hw = ds.F, ds.wl
peak = RL.measured_peaks(bench.ROOT)["hbm_gbs"]
M = lambda fn: bench.marginal_us(fn, ds.flush_l2, K=10)
def line(name, us, nb):
    print(f"  {name:24s} {us:8.2f} us  frac {nb / us / 1e3 / peak:.3f}", flush=True)
for rows in (4096, 16384):
    cols = bench.HIDDEN
    x = synth.activations_bf16_device(rows, cols, synth.BASE_SEED + 9, dev)
    q = torch.empty(rows, cols, dtype=torch.uint8, device=dev)
    s = torch.empty(cols // 128, rows, dtype=torch.uint8, device=dev)
    qT = torch.empty(rows * cols, dtype=torch.uint8, device=dev)
    sT = torch.empty(rows // 128 + 1, cols, dtype=torch.uint8, device=dev)
    nb = RL.quantize_dual_bytes([rows], cols)
    print(f"quantize {rows}x{cols}")
    line("A1", M(lambda: F.fp8flow_quantize_rowwise(x, q, s)), RL.quantize_bytes(rows, cols))
    line("A2", M(lambda: F.fp8flow_scaling_aware_transpose(q, s, qT, sT)), RL.transpose_bytes([rows], cols))
    line("A1->A2", M(lambda: (F.fp8flow_quantize_rowwise(x, q, s), F.fp8flow_scaling_aware_transpose(q, s, qT, sT))), nb)
    ref = (q.clone(), s.clone(), qT.clone(), sT.clone())
    line("quantize_dual", M(lambda: F.fp8flow_quantize_dual(x, q, s, qT, sT)), nb)
    print("  bit-exact:", all(torch.equal(a, b) for a, b in zip(ref, (q, s, qT, sT))))
    del x, q, s, qT, sT
E = hw.E_loc
print(f"swiglu {hw.R}x{bench.FFN} ({E} experts)")
rows_dev = ds.off[E:]
line("A5", M(lambda: F.fp8flow_swiglu_quant(hw.h, ds.q_a, ds.s_a, rows_dev=rows_dev)), hw.op_bytes()["A5_swiglu_quant"])
line("A2(A)", M(lambda: F.fp8flow_scaling_aware_transpose(ds.q_a, ds.s_a, ds.aT, ds.saT, seg_offsets=ds.off)),
     hw.op_bytes()["A2_transpose_a"])
two = lambda: (F.fp8flow_swiglu_quant(hw.h, ds.q_a, ds.s_a, rows_dev=rows_dev),
               F.fp8flow_scaling_aware_transpose(ds.q_a, ds.s_a, ds.aT, ds.saT, seg_offsets=ds.off))
nb2 = hw.op_bytes()["A5_swiglu_quant"] + hw.op_bytes()["A2_transpose_a"]
line("A5->A2", M(two), nb2)
ref = (ds.q_a.clone(), ds.s_a.clone(), ds.aT.clone(), ds.saT.clone())
line("swiglu_quant_dual (vs 2-launch bytes)", M(lambda: F.fp8flow_swiglu_quant_dual(hw.h, ds.q_a, ds.s_a, ds.aT, ds.saT,
                                                                                   seg_offsets=ds.off)), nb2)
print("  bit-exact:", all(torch.equal(a, b) for a, b in zip(ref, (ds.q_a, ds.s_a, ds.aT, ds.saT))))
