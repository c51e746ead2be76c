"""The N > 1 path of bench.py on one GPU: two ranks (gloo for the host collectives, CUDA IPC between
the two processes for NEXT-3), a reduced token count.  Guards what the driver's multi-GPU run
executes: the strong split of the layer, the per-rank step, max-over-ranks timing, every rank's
whole-step verification against the oracle (elementwise + C11 checksums) merged on rank 0 with
the CPU-oracle baseline of all ranks, the NEXT-3 dispatch/combine across ranks and the NCCL-style
all-to-all baseline, each checked bit-exact."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_one_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, FP8FLOW_DIST_BACKEND="gloo", FP8FLOW_BENCH_TOKENS="2048")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--no-e2e"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["tokens"] == 2048
    # the strong split: each rank owns 128 of the 256 experts; every rank verified its whole step
    assert line["scaling"] == "strong" and line["config"]["local_experts"] == 128
    assert set(line["parity"]) == {"rank0", "rank1"}, line["parity"]
    assert all(all(p.values()) for p in line["parity"].values()), line["parity"]
    assert line["parity_all_ranks"] is True and line["checksums_match"] is True
    cb = line["cpu_baseline"]
    assert cb is not None and cb["kind"] == "oracle" and cb["value"] > 0 and "x2 ranks" in cb["sample"], cb
    ep = line["next3_multi_rank"]
    assert ep.get("parity") is True, ep
    assert ep["baseline_all_to_all_then_permute"].get("same_output") is True, ep
    assert line["load_imbalance"] >= 1.0
