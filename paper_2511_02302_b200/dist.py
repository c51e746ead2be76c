"""Expert-group sharding and the post-timing collectives.

The hot path shards with no exchange step: rank r of N owns DeepSeek-V3 expert group r mod 8
(32 of the 256 experts, the EP8 partition) and runs the whole hot path on what that group
receives.  torch.distributed (NCCL over NVLink on the B200 box, gloo in the CPU tests) is used
only OUTSIDE the timed region: barriers around it, the max over ranks of the measured time, the
sum of bytes, and the gather of per-rank output checksums.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist

NUM_GROUPS = 8


def env() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def init(backend: str) -> bool:
    """Initialises the process group when launched with WORLD_SIZE > 1; returns whether it did."""
    rank, _, world = env()
    if world <= 1:
        return False
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend, rank=rank, world_size=world)
    return True


def expert_group(rank: int, num_groups: int = NUM_GROUPS) -> int:
    """Expert group owned by a rank (weak scaling: every rank owns one full group)."""
    return rank % num_groups


def backend() -> str:
    """Collective backend: NCCL on the GPU box; FP8FLOW_DIST_BACKEND=gloo runs several ranks on one
    GPU (a test of the multi-rank orchestration when only one device is available)."""
    return os.environ.get("FP8FLOW_DIST_BACKEND", "nccl")


def local_device(local_rank: int) -> torch.device:
    n = torch.cuda.device_count()
    return torch.device("cuda", local_rank % n if n else 0)


def barrier(device: torch.device | None = None) -> None:
    if dist.is_initialized():
        if device is not None and device.type == "cuda" and dist.get_backend() == "nccl":
            dist.barrier(device_ids=[device.index])
        else:
            dist.barrier()


def _coll_device(device):
    """gloo collectives run on host tensors; NCCL on the rank's GPU."""
    return torch.device("cpu") if dist.get_backend() == "gloo" else device


def _reduce(x: float, op, device) -> float:
    if not dist.is_initialized():
        return float(x)
    device = _coll_device(device)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(x: float, device=torch.device("cpu")) -> float:
    return _reduce(x, dist.ReduceOp.MAX, device)


def sum_over_ranks(x: float, device=torch.device("cpu")) -> float:
    return _reduce(x, dist.ReduceOp.SUM, device)


def gather_checksums(values: list[int], device=torch.device("cpu")) -> list[list[int]]:
    """All-gather a list of uint64 checksums (carried as int64 bit patterns) from every rank."""
    if dist.is_initialized():
        device = _coll_device(device)
    t = torch.tensor([v - (1 << 64) if v >= (1 << 63) else v for v in values], dtype=torch.int64, device=device)
    if not dist.is_initialized():
        return [[v & ((1 << 64) - 1) for v in t.tolist()]]
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [[v & ((1 << 64) - 1) for v in o.tolist()] for o in out]
