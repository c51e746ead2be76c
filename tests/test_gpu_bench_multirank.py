"""The N > 1 path of bench.py on one GPU: two ranks (gloo for the host collectives, CUDA IPC between
the two processes for NEXT-3), a reduced token count.  Guards what the driver's multi-GPU run
executes: the per-rank step, max-over-ranks timing, the NEXT-3 dispatch/combine across ranks and
the NCCL-style all-to-all baseline, each checked bit-exact."""
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
           "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["tokens"] == 2048
    assert all(line["parity"].values()), line["parity"]
    ep = line["next3_multi_rank"]
    assert ep.get("parity") is True, ep
    assert ep["baseline_all_to_all_then_permute"].get("same_output") is True, ep
    assert line["load_imbalance"] >= 1.0
