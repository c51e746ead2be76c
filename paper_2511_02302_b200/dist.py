"""Expert-parallel sharding and the post-timing collectives.

The hot path shards with no exchange step.  Two partitions of the DeepSeek-V3
layer (256 experts, 16384 tokens):

* strong: rank g of n owns experts [g*256/n, (g+1)*256/n) and the token shard
  [g*T/n, (g+1)*T/n) of the two entry casts; n = 1 is the whole layer on one GPU.  Total work is
  fixed; the per-rank load follows the routing skew (reported as load_imbalance).
* weak: rank r owns DeepSeek-V3 expert group r mod 8 (32 experts, the EP8 partition) and 1/8 of
  the tokens, so per-GPU work is one expert group at every n.
* balanced (bench.py's default): like strong (256/n experts and 1/n of the tokens per GPU), but WHICH experts a GPU
  owns is chosen by load, longest-processing-time first over the routed row counts (the expert
  placement an expert-parallel load balancer makes); the experts are relabelled so that GPU g's
  set is the id range [g*256/n, (g+1)*256/n) (balanced_relabel).

torch.distributed (NCCL over NVLink on the B200 box, gloo in the CPU tests) is used only OUTSIDE
the timed region: barriers around it, the max over ranks of the measured time, the sum of bytes,
the gather of per-rank output checksums and verification reports.
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


def shard(rank: int, world: int, mode: str, num_experts: int = 256, num_tokens: int = 16384,
          num_groups: int = NUM_GROUPS) -> dict:
    """The rank's part of the layer: experts [expert_begin, expert_begin + num_local_experts) and
    entry-cast tokens [token_begin, token_end).  mode 'strong' splits the whole layer over the
    world (world must divide the expert count); 'weak' gives every rank one expert group."""
    if mode == "strong":
        if world < 1 or num_experts % world:
            raise ValueError(f"{num_experts} experts do not split over {world} ranks")
        per = num_experts // world
        t0, t1 = rank * num_tokens // world, (rank + 1) * num_tokens // world
        return {"mode": mode, "expert_begin": rank * per, "num_local_experts": per, "token_begin": t0,
                "token_end": t1}
    if mode == "balanced":
        sh = shard(rank, world, "strong", num_experts, num_tokens, num_groups)
        sh["mode"] = mode
        return sh
    if mode == "weak":
        g = expert_group(rank, num_groups)
        per = num_experts // num_groups
        t0, t1 = g * num_tokens // num_groups, (g + 1) * num_tokens // num_groups
        return {"mode": mode, "expert_begin": g * per, "num_local_experts": per, "token_begin": t0,
                "token_end": t1, "group": g}
    raise ValueError(f"unknown partition {mode!r}")


def balanced_placement(counts, world: int) -> list[list[int]]:
    """Expert sets of `world` GPUs with equal expert counts and near-equal padded rows: experts
    sorted by padded row count (descending, ties by id), each to the least-loaded GPU that still
    has room (ties by GPU index) -- the LPT rule.  Deterministic."""
    n = len(counts)
    if world < 1 or n % world:
        raise ValueError(f"{n} experts do not split over {world} ranks")
    per = n // world
    padded = [(int(c) + 15) // 16 * 16 for c in counts]
    order = sorted(range(n), key=lambda e: (-padded[e], e))
    load, sets = [0] * world, [[] for _ in range(world)]
    for e in order:
        g = min((g for g in range(world) if len(sets[g]) < per), key=lambda g: (load[g], g))
        sets[g].append(e)
        load[g] += padded[e]
    return [sorted(x) for x in sets]


def balanced_relabel(counts, world: int):
    """new_id[e] for every expert id e: GPU g's LPT set becomes [g*E/n, (g+1)*E/n), in id order."""
    sets = balanced_placement(counts, world)
    new_id = [0] * len(counts)
    for g, experts in enumerate(sets):
        for i, e in enumerate(experts):
            new_id[e] = g * (len(counts) // world) + i
    return new_id


def gather_objects(obj, device=torch.device("cpu")) -> list:
    """All-gather a picklable object from every rank (verification reports; outside timing)."""
    if not dist.is_initialized():
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def merge_rank_reports(reports: list[dict]) -> dict:
    """Rank 0's view of the per-rank verification reports: every rank's parity flags, whether
    every rank's GPU checksums equal the oracle's C11 checksums of its shard, and the CPU-oracle
    baseline as one job (bytes of all ranks / the slowest rank's seconds, cores of all ranks)."""
    out = {"parity": {f"rank{i}": r.get("parity") for i, r in enumerate(reports)}}
    flags = [v for r in reports for v in (r.get("parity") or {}).values()]
    out["parity_all_ranks"] = bool(flags) and all(flags)
    cs = [r.get("checksums_match") for r in reports]
    out["checksums_match"] = all(c is True for c in cs) if cs else None
    cpu = [r.get("cpu") for r in reports if r.get("cpu")]
    if cpu and len(cpu) == len(reports):
        secs = max(c["seconds"] for c in cpu)
        nbytes = sum(c["bytes"] for c in cpu)
        out["cpu_baseline"] = {"value": round(nbytes / secs / 1e9, 4), "unit": "GB/s",
                               "cores": sum(c["cores"] for c in cpu), "kind": "oracle",
                               "sample": cpu[0]["sample"] + (f" (x{len(cpu)} ranks, each on its own shard, "
                                                            "concurrently)" if len(cpu) > 1 else ""),
                               "seconds": round(secs, 2)}
        if cpu[0].get("single_thread"):  # rank 0's single-threaded timing of a bounded sample
            out["cpu_baseline"]["single_thread"] = cpu[0]["single_thread"]
    return out


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
