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
