"""NEXT-2 grouped Fprop alone at bench.py's EP8 group-0 shapes (fc1: X_perm [15872][7168] x
W1_e^T, N = 4096; fc2: A [15872][2048] x W2_e^T, N = 7168; 32 experts), marginal cold-L2 us,
TF/s, output checksum.  Not product.   python tools/probe/fprop_probe.py [--once]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import synth
dev = torch.device("cuda", 0)
ds = bench.DeviceStep(bench.Workload(0, 1, "weak", dev))
ds.launch_ops(record=False)
F, hw, E = ds.F, ds.wl, ds.wl.E_loc
g = torch.Generator(device=dev)
g.manual_seed(synth.BASE_SEED + 11)
for name, (A, sA, N, K) in {"fc1": (ds.x_perm, ds.s_perm, 2 * bench.FFN, bench.HIDDEN),
                            "fc2": (ds.q_a, ds.s_a, bench.HIDDEN, bench.FFN)}.items():
    W = torch.randint(0, 0x7E, (E, N, K), dtype=torch.uint8, device=dev, generator=g)
    W |= torch.randint(0, 2, (E, N, K), dtype=torch.uint8, device=dev, generator=g) << 7
    sW = torch.randint(112, 118, (E, K // 128, N), dtype=torch.uint8, device=dev, generator=g)
    Dout = torch.empty(hw.R, N, dtype=torch.bfloat16, device=dev)
    fn = lambda: F.fp8flow_gemm_blockscaled(A, sA, W, sW, Dout, seg_offsets=ds.off)
    torch.cuda.synchronize()
    if "--once" in sys.argv:
        fn(); torch.cuda.synchronize(); ds.flush_l2(); torch.cuda.synchronize()
        torch.cuda.profiler.start(); fn(); torch.cuda.synchronize(); torch.cuda.profiler.stop()
        continue
    us = bench.marginal_us(fn, ds.flush_l2, K=5)
    fl = 2.0 * hw.R * N * K
    fn(); torch.cuda.synchronize()
    v = Dout.view(torch.int16).view(-1).to(torch.int64)
    ck = (int(v.sum()), int((v * (torch.arange(v.numel(), device=dev) % 65521)).sum()))
    print(f"{name} {us:.1f} us  {fl / us / 1e6:.0f} TF/s  frac {fl / us / 1e6 / 3305:.3f}  checksum {ck}", flush=True)
    del W, sW, Dout
