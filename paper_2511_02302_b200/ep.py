"""NEXT-3 host plumbing: peer tables for the expert-parallel dispatch / combine kernels.

The kernels (csrc/ep.cu) take HOST arrays of n device pointers, entry r = rank r's buffer as
mapped in the calling process.  This module builds those tables; it does no compute.

* ``IpcPeers``   one process per GPU (the B200 box): each rank exports the CUDA IPC handle of
                 every registered buffer (fp8flow_ipc_get_handle: handle + offset inside the
                 caching allocator's block), the records are all-gathered over torch.distributed
                 (gloo or NCCL; outside the hot loop) and the peers' handles are opened once.
* ``LocalPeers`` several ranks inside one process on one device (tests, single-GPU bench): the
                 table is the ranks' own device pointers.

Rank r of n owns tokens [r*T_per_rank, (r+1)*T_per_rank) and experts [r*E/n, (r+1)*E/n)
(R34).  The per-step sequence on rank r (all on one stream, graph-capturable):
    barrier -> peer_gather(topk) -> permute_plan(gathered, own experts) -> dispatch_permute_pad
    ... experts ...  barrier -> combine_unpermute
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import fp8flow as F


def expert_range(rank: int, world: int, num_experts: int) -> tuple[int, int]:
    """(expert_begin, experts_per_rank) of a rank; the experts split evenly (EP partition)."""
    if num_experts % world:
        raise ValueError(f"{num_experts} experts do not split over {world} ranks")
    per = num_experts // world
    return rank * per, per


def token_range(rank: int, tokens_per_rank: int) -> tuple[int, int]:
    """Global token ids [begin, end) owned by a rank (R34: rank-major token order)."""
    return rank * tokens_per_rank, (rank + 1) * tokens_per_rank


def resolve_tables(records: list[dict], rank: int, local: dict[str, int], open_fn) -> dict[str, list[int]]:
    """records[r] = {name: (handle bytes, offset)} from every rank; returns name -> per-rank device
    addresses in this process (own entries from `local`, peers' via open_fn(handle) + offset; each
    distinct handle is opened once)."""
    opened: dict[bytes, int] = {}
    tables: dict[str, list[int]] = {}
    for name in records[rank]:
        row = []
        for r, rec in enumerate(records):
            if r == rank:
                row.append(local[name])
                continue
            handle, offset = rec[name]
            if handle not in opened:
                opened[handle] = open_fn(handle)
            row.append(opened[handle] + offset)
        tables[name] = row
    return tables, list(opened.values())


class IpcPeers:
    """Peer tables over CUDA IPC for one process per GPU.  `buffers` maps a name to this rank's
    device tensor; every rank must register the same names.  Collective (all ranks call it)."""

    def __init__(self, buffers: dict[str, torch.Tensor], group=None):
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        try:
            mine = {name: F.fp8flow_ipc_get_handle(t) for name, t in buffers.items()}
        except F.Fp8FlowError:
            mine = None  # still join the collective, so no rank is left waiting in it
        records: list = [None] * self.world
        dist.all_gather_object(records, mine, group=group)
        bad = [r for r, rec in enumerate(records) if rec is None]
        if bad:
            raise F.Fp8FlowError(f"CUDA IPC export failed on rank(s) {bad}")
        local = {name: t.data_ptr() for name, t in buffers.items()}
        self.tables, self._bases = resolve_tables(records, self.rank, local, F.fp8flow_ipc_open)
        self._keep = buffers

    def table(self, name: str) -> list[int]:
        return self.tables[name]

    def close(self) -> None:
        for b in self._bases:
            F.fp8flow_ipc_close(b)
        self._bases = []


class LocalPeers:
    """n ranks inside one process: buffers[r][name] = rank r's tensor (tables for the names every
    rank holds)."""

    def __init__(self, buffers: list[dict[str, torch.Tensor]]):
        self.world = len(buffers)
        names = [k for k in buffers[0] if all(k in b for b in buffers)]
        self.tables = {name: [b[name].data_ptr() for b in buffers] for name in names}
        self._keep = buffers

    def table(self, name: str) -> list[int]:
        return self.tables[name]


def signal_buffer(world: int, device) -> torch.Tensor:
    """A rank's barrier signal buffer: n + 1 uint32 (held as int32), zeroed once."""
    return torch.zeros(world + 1, dtype=torch.int32, device=device)


def dispatch_permute(peers, rank: int, tokens_per_rank: int, hidden: int, top_k: int, num_experts: int,
                     ld_s_tok: int, topk_all: torch.Tensor, row_map: torch.Tensor, src_of_row: torch.Tensor,
                     expert_offsets: torch.Tensor, ws: torch.Tensor, q_out: torch.Tensor, s_out: torch.Tensor,
                     align: int = 16, kernel: int = F.DISPATCH_AUTO, status: torch.Tensor | None = None,
                     stream=None) -> None:
    """Rank `rank`'s receive side: gather every rank's routing (peers table "topk"), plan its own
    experts over the global tokens, then pull + permute + pad the routed FP8 tokens (tables "q",
    "s").  Outputs as fp8flow_permute_pad on the rank-order concatenation.  status: the preceding
    barrier's device flag (gather and dispatch write nothing if it is nonzero) or None."""
    world = peers.world
    e0, per = expert_range(rank, world, num_experts)
    F.fp8flow_peer_gather(peers.table("topk"), tokens_per_rank * top_k * 4, topk_all, status=status, stream=stream)
    F.fp8flow_permute_plan(topk_all, e0, per, align, row_map, src_of_row, expert_offsets, ws, stream=stream)
    F.fp8flow_dispatch_permute_pad(peers.table("q"), peers.table("s"), ld_s_tok, tokens_per_rank, hidden, row_map,
                                   src_of_row, expert_offsets, q_out, s_out, kernel=kernel, status=status,
                                   stream=stream)


def combine(peers, rank: int, tokens_per_rank: int, hidden: int, num_experts: int, topk_idx: torch.Tensor,
            probs: torch.Tensor | None, y: torch.Tensor, status: torch.Tensor | None = None, stream=None) -> None:
    """Owner side: y = sum_k p * (expert output row) pulled from the ranks' "x" buffers located by
    their "row_map" plans."""
    _, per = expert_range(rank, peers.world, num_experts)
    F.fp8flow_combine_unpermute(peers.table("x"), peers.table("row_map"), hidden, topk_idx, per, probs,
                                token_range(rank, tokens_per_rank)[0], y, status=status, stream=stream)
