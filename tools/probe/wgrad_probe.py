"""NEXT-2 Wgrad alone at bench.py's EP8 group-0 shape (32 experts, 15872 padded rows, dW1 =
dH^T X_perm, BF16 [32][4096][7168]): marginal cold-L2 us and TFLOP/s; --once runs one launch
(for ncu).  Not product.   python tools/probe/wgrad_probe.py [--once]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import synth
dev = torch.device("cuda", 0)
ds = bench.DeviceStep(bench.Workload(0, 1, "weak", dev))
ds.launch_ops(record=False)
F, hw, E, FFN, H = ds.F, ds.wl, ds.wl.E_loc, bench.FFN, bench.HIDDEN
dA = synth.normal_bf16_device(hw.R, FFN, synth.BASE_SEED + 5, dev, sigma=0.5)
qh = torch.empty(hw.R, 2 * FFN, dtype=torch.uint8, device=dev)
sh = torch.empty(2 * FFN // 128, hw.R, dtype=torch.uint8, device=dev)
F.fp8flow_swiglu_bwd_quant(hw.h, dA, qh, sh, rows_dev=ds.off[E:])
hT = torch.empty(hw.R * 2 * FFN, dtype=torch.uint8, device=dev)
shT = torch.empty(hw.R // 128 + E, 2 * FFN, dtype=torch.uint8, device=dev)
F.fp8flow_scaling_aware_transpose(qh, sh, hT, shT, seg_offsets=ds.off)
dW = torch.empty(E, 2 * FFN, H, dtype=torch.bfloat16, device=dev)
fn = lambda: F.fp8flow_gemm_wgrad(hT, shT, ds.xT, ds.sxT, dW, ds.off)
torch.cuda.synchronize()
if "--once" in sys.argv:
    fn(); torch.cuda.synchronize(); ds.flush_l2(); torch.cuda.synchronize()
    torch.cuda.profiler.start(); fn(); torch.cuda.synchronize(); torch.cuda.profiler.stop()
else:
    us = bench.marginal_us(fn, ds.flush_l2, K=5)
    fl = 2.0 * hw.R * 2 * FFN * H
    print(f"wgrad {us:.1f} us  {fl / us / 1e6:.0f} TF/s  frac {fl / us / 1e6 / 3305:.3f}  m_e={torch.diff(ds.off).tolist()}")
fn(); torch.cuda.synchronize()
v = dW.view(torch.int16).view(-1).to(torch.int64)
ck = (int(v.sum()), int((v * (torch.arange(v.numel(), device=dev) % 65521)).sum()))
print("checksum", ck)
