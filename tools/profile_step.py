"""Profiling driver (not product): warms up bench.py's step, then runs ONE serial pass of the
step's 8 launches (whole DeepSeek-V3 layer on one GPU, bench.py's default partition) plus
the NEXT-row kernels on expert group 0 (SwiGLU backward, dual-output SwiGLU, dual-output move, grouped fc1 GEMM,
fc1 Wgrad, dual-output quantize at 4096x7168, NEXT-3 dispatch and combine of rank 0 of 8 virtual EP ranks) between cudaProfilerStart/Stop, so
    ncu --set full --profile-from-start off ... python tools/profile_step.py [--partition weak]
captures exactly one launch of each kernel, in this order."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402

ORDER = ["A1_quantize_x", "A3_plan", "A3_move", "A5_swiglu_quant", "A4_unpermute", "A1_quantize_dy",
         "A2_transpose_xperm", "A2_transpose_a", "NEXT1_swiglu_bwd_quant", "NEXT1_swiglu_quant_dual",
         "NEXT1_permute_pad_dual",
         "NEXT2_gemm_fc1_fprop", "A2_transpose_dH", "NEXT2_wgrad_maps", "NEXT2_gemm_fc1_wgrad", "NEXT1_quantize_dual",
         "NEXT3_dispatch_permute_pad", "NEXT3_combine_unpermute"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--partition", choices=["strong", "balanced", "weak"], default="balanced")
    ap.add_argument("--no-next", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    ds = bench.DeviceStep(bench.Workload(0, 1, args.partition, dev))
    extra = None
    if not args.no_next:
        g0 = bench.DeviceStep(bench.Workload(0, 1, "weak", dev))
        wl, F = g0.wl, g0.F
        dA = synth.normal_bf16_device(wl.R, bench.FFN, synth.BASE_SEED + 5, dev, sigma=0.5)
        qb = torch.empty(wl.R, 2 * bench.FFN, dtype=torch.uint8, device=dev)
        sbw = torch.empty(2 * bench.FFN // 128, wl.R, dtype=torch.uint8, device=dev)
        E = wl.E_loc
        W = torch.randint(0, 0x7E, (E, 2 * bench.FFN, bench.HIDDEN), dtype=torch.uint8, device=dev)
        sW = torch.full((E, bench.HIDDEN // 128, 2 * bench.FFN), 115, dtype=torch.uint8, device=dev)
        Dg = torch.empty(wl.R, 2 * bench.FFN, dtype=torch.bfloat16, device=dev)
        rows_dev = g0.off[E:]
        g0.launch_ops(record=False)
        hT = torch.empty(wl.R * 2 * bench.FFN, dtype=torch.uint8, device=dev)
        shT = torch.empty(wl.R // 128 + E, 2 * bench.FFN, dtype=torch.uint8, device=dev)
        dW = torch.empty(E, 2 * bench.FFN, bench.HIDDEN, dtype=torch.bfloat16, device=dev)
        wsw = torch.empty(F.fp8flow_gemm_wgrad_workspace_bytes(E), dtype=torch.uint8, device=dev)
        xq = synth.activations_bf16_device(4096, bench.HIDDEN, synth.BASE_SEED + 9, dev)
        qq = torch.empty(4096, bench.HIDDEN, dtype=torch.uint8, device=dev)
        sq = torch.empty(bench.HIDDEN // 128, 4096, dtype=torch.uint8, device=dev)
        qqT = torch.empty(4096 * bench.HIDDEN, dtype=torch.uint8, device=dev)
        sqT = torch.empty(4096 // 128 + 1, bench.HIDDEN, dtype=torch.uint8, device=dev)
        st = bench.ep_setup(dev)  # NEXT-3: 8 virtual EP ranks on this device

        def extra():
            F.fp8flow_swiglu_bwd_quant(wl.h, dA, qb, sbw, rows_dev=rows_dev)
            F.fp8flow_swiglu_quant_dual(wl.h, g0.q_a, g0.s_a, g0.aT, g0.saT, seg_offsets=g0.off)
            F.fp8flow_permute_pad_dual(wl.q_recv, wl.s_recv, g0.src, g0.off, g0.x_perm, g0.s_perm, g0.xT, g0.sxT)
            F.fp8flow_gemm_blockscaled(g0.x_perm, g0.s_perm, W, sW, Dg, seg_offsets=g0.off)
            F.fp8flow_scaling_aware_transpose(qb, sbw, hT, shT, seg_offsets=g0.off)
            F.fp8flow_gemm_wgrad(hT, shT, g0.xT, g0.sxT, dW, g0.off, workspace=wsw)
            F.fp8flow_quantize_dual(xq, qq, sq, qqT, sqT)
            st["receive"](0, kernel_only=True)
            st["ep"].combine(st["peers"], 0, st["tpr"], bench.HIDDEN, st["E"], st["ranks"][0]["topk"],
                             st["ranks"][0]["probs"], st["y"])

    for _ in range(3):
        ds.launch_ops(record=False)
        if extra:
            extra()
    torch.cuda.synchronize()
    ds.flush_l2()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    ds.launch_ops(record=False)
    if extra:
        extra()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled:", ", ".join(ORDER if extra else ORDER[:8]))


if __name__ == "__main__":
    main()
