"""Marginal cold-L2 cost of the dual-output fusions on bench.py's workload (not product): the A3 move
fused with A2 (fp8flow_permute_pad_dual) against move then A2(X_perm), and the SwiGLU dual kernel
against A5 then A2(A); outputs compared byte for byte with the unfused launches.
    python tools/probe/marginal_dual_step.py [balanced|weak]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
mode = sys.argv[1] if len(sys.argv) > 1 else "balanced"
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
wl = bench.Workload(0, 1, mode, dev)
ds = bench.DeviceStep(wl)
ds.launch_ops(record=False)
torch.cuda.synchronize()
F = ds.F
KEYS = ("x_perm", "s_perm", "xT", "sxT", "q_a", "s_a", "aT", "saT")
fns = ds.op_fns()
for k in KEYS:
    getattr(ds, k).fill_(0xEE)
for op in ("A3_move", "A2_transpose_xperm", "A5_swiglu_quant", "A2_transpose_a"):
    fns[op]()
torch.cuda.synchronize()
ref = {k: getattr(ds, k).clone() for k in KEYS}
for k in KEYS:
    getattr(ds, k).fill_(0xEE)
pd = lambda: F.fp8flow_permute_pad_dual(wl.q_recv, wl.s_recv, ds.src, ds.off, ds.x_perm, ds.s_perm, ds.xT, ds.sxT)
sd = lambda: F.fp8flow_swiglu_quant_dual(wl.h, ds.q_a, ds.s_a, ds.aT, ds.saT, seg_offsets=ds.off,
                                         rows_dev=ds.off[wl.E_loc:])
pd(); sd(); torch.cuda.synchronize()
same = {k: bool(torch.equal(ref[k], getattr(ds, k))) for k in ref}
t = {}
t["move"] = bench.marginal_us(fns["A3_move"], ds.flush_l2)
t["A2_xperm"] = bench.marginal_us(fns["A2_transpose_xperm"], ds.flush_l2)
t["permute_dual"] = bench.marginal_us(pd, ds.flush_l2)
t["A5"] = bench.marginal_us(fns["A5_swiglu_quant"], ds.flush_l2)
t["A2_a"] = bench.marginal_us(fns["A2_transpose_a"], ds.flush_l2)
t["swiglu_dual"] = bench.marginal_us(sd, ds.flush_l2)
print(mode, {k: round(v, 2) for k, v in t.items()}, "identical:", same, flush=True)
print(f"move+A2 {t['move'] + t['A2_xperm']:.1f} us -> dual {t['permute_dual']:.1f};"
      f" A5+A2 {t['A5'] + t['A2_a']:.1f} -> dual {t['swiglu_dual']:.1f}", flush=True)
