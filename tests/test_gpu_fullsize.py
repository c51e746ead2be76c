"""Full-size parity in the launch configuration bench.py times: bench.py's own
Workload + DeviceStep for the whole DeepSeek-V3 layer on one GPU (256 experts, 16384 tokens,
133,056 padded rows) and for one EP8 expert group, the step replayed from its CUDA graph, then
bench.py's verification leg: every output element against the oracle on the same input bytes
(A5: <= 1 ULP on <= 1e-4, identical scales) and the device C11 checksums against the oracle's."""
import os
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


@pytest.mark.parametrize("mode", ["strong", "weak"])
def test_bench_step_matches_oracle_at_full_size(mode):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import bench

    dev = torch.device("cuda", 0)
    wl = bench.Workload(0, 1, mode, dev)
    ds = bench.DeviceStep(wl)
    trial = ds.choose_schedule(trials=2)          # both graphs captured; the faster one replays
    assert set(trial) >= {"dag", "serial"}
    ds.timed_step_graph()
    torch.cuda.synchronize()
    rep = bench.cpu_baseline_leg(wl, ds, time_it=False, verify=True, checks=[], threads=None)
    assert all(rep["parity"].values()), rep["parity"]
    assert rep["checksums_match"] is True
    if mode == "strong":
        assert wl.E_loc == 256 and wl.R == 133056 and wl.T_recv == 16384


def test_config5_largest_shape_matches_oracle(orc):
    """Config 5's largest shape, 65536 x 7168 (470 M codes, 947 MB moved by A2): A1 then A2 on the
    device, every code and scale byte against the oracle's A1 and A2 on the same BF16 input."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import numpy as np

    import synth
    from paper_2511_02302_b200 import fp8flow as F

    dev = torch.device("cuda", 0)
    rows, cols = 65536, 7168
    x = synth.activations_bf16_device(rows, cols, synth.BASE_SEED + 65, dev)
    q = torch.empty(rows, cols, dtype=torch.uint8, device=dev)
    s = torch.empty(cols // 128, rows, dtype=torch.uint8, device=dev)
    F.fp8flow_quantize_rowwise(x, q, s)
    qT = torch.empty(rows * cols, dtype=torch.uint8, device=dev)
    sT = torch.empty(rows // 128 + 1, cols, dtype=torch.uint8, device=dev)
    F.fp8flow_scaling_aware_transpose(q, s, qT, sT)
    torch.cuda.synchronize()
    x_bits = synth.bf16_bits(x.cpu())
    del x
    q_ref, s_ref = orc.quantize_rowwise_bf16(x_bits)
    assert np.array_equal(q.cpu().numpy(), q_ref) and np.array_equal(s.cpu().numpy(), s_ref)
    del x_bits
    qT_ref, sT_ref = orc.scaling_aware_transpose(q_ref, s_ref)
    assert np.array_equal(qT.cpu().numpy(), qT_ref)
    assert np.array_equal(sT[: sT_ref.shape[0]].cpu().numpy(), sT_ref)
