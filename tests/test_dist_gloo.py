"""The N>1 host path on CPU: expert-group sharding and the post-timing collectives of
paper_2511_02302_b200/dist.py, run with world_size 2 over gloo (the GPU box uses NCCL)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update({"RANK": str(rank), "LOCAL_RANK": str(rank), "WORLD_SIZE": str(world),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    from paper_2511_02302_b200 import dist as D

    assert D.env() == (rank, rank, world)
    assert D.init("gloo")
    g = D.expert_group(rank)
    t_max = D.max_over_ranks(10.0 + rank)
    b_sum = D.sum_over_ranks(100.0 * (rank + 1))
    big = (1 << 64) - 1 - rank                    # uint64 values above 2^63 survive the int64 carrier
    sums = D.gather_checksums([rank, big])
    D.barrier()
    q.put((rank, g, t_max, b_sum, sums))
    D.dist.destroy_process_group()


def test_two_rank_gloo_sharding_and_collectives():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [o[1] for o in out] == [0, 1]                      # distinct expert groups
    assert all(o[2] == 11.0 for o in out)                     # max over ranks
    assert all(o[3] == 300.0 for o in out)                    # sum over ranks
    expect = [[0, (1 << 64) - 1], [1, (1 << 64) - 2]]
    assert all(o[4] == expect for o in out)


def test_single_process_defaults(monkeypatch):
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE"):
        monkeypatch.delenv(k, raising=False)
    from paper_2511_02302_b200 import dist as D

    assert D.env() == (0, 0, 1)
    assert D.init("gloo") is False
    assert D.max_over_ranks(3.5) == 3.5 and D.sum_over_ranks(2.0) == 2.0
    assert D.gather_checksums([5]) == [[5]]
    assert [D.expert_group(r) for r in range(10)] == [0, 1, 2, 3, 4, 5, 6, 7, 0, 1]


def test_roofline_byte_formulas():
    from paper_2511_02302_b200 import roofline as RL

    assert RL.quantize_bytes(4096, 7168) == 4096 * 7168 * 3 + 4096 * 56          # 3.008 B/elem
    assert RL.transpose_bytes([4096], 7168) == 4096 * 7168 * 2 + 4096 * 56 + 32 * 7168
    assert RL.transpose_bytes([16, 0, 144], 128) == 160 * 128 * 2 + 160 + (1 + 0 + 2) * 128
    assert RL.swiglu_quant_bytes(10, 2048) == 10 * (4 * 2048 + 2048 + 16)           # 5.008 B/output
    assert RL.unpermute_bytes(5, 3, 8, 128, True) == 5 * 256 + 3 * 256 + 3 * 8 * 8
    assert RL.permute_move_bytes(3, 16, 128) == 3 * 129 + 16 * 129 + 16 * 4
    p = RL.measured_peaks("/nonexistent")
    assert p["hbm_gbs"] == 6650.0 and "fallback" in p["source"]


@pytest.mark.parametrize("group", [0, 3])
def test_expert_shard_is_what_dispatch_would_deliver(group):
    import numpy as np

    import synth

    idx, probs = synth.routing(2000, 7)
    sh = synth.expert_shard(idx, probs, group, 8)
    e0 = group * 32
    local = (idx.numpy() >= e0) & (idx.numpy() < e0 + 32)
    assert np.array_equal(sh.recv_tokens, np.nonzero(local.any(1))[0])
    assert np.array_equal(sh.topk_idx, idx.numpy()[sh.recv_tokens])
    # every token's experts are distinct (precondition of the plan) and routing is group-limited
    assert all(len(set(r)) == 8 for r in idx.numpy()[:200])
    assert all(len({e // 32 for e in r}) <= 4 for r in idx.numpy()[:200])


# ------------------------------------------------------------------ NEXT-3 peer-table plumbing
def _ep_worker(rank, world, port, q):
    """The IpcPeers exchange with fake handles: every rank publishes {name: (handle, offset)} over
    gloo's all_gather_object and resolves the peer table with a recording open function."""
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import torch.distributed as dist

    from paper_2511_02302_b200 import ep

    dist.init_process_group("gloo", rank=rank, world_size=world)
    # names q and s live in one allocation (same handle, different offsets), x in another
    mine = {"q": (b"A%d" % rank, 0), "s": (b"A%d" % rank, 4096), "x": (b"B%d" % rank, 64)}
    records = [None] * world
    dist.all_gather_object(records, mine)
    opened = []

    def fake_open(h):
        opened.append(h)
        return 1_000_000 * (1 + int(h[1:])) + (0 if h[:1] == b"A" else 500_000)

    local = {"q": 11, "s": 22, "x": 33}
    tables, bases = ep.resolve_tables(records, rank, local, fake_open)
    dist.destroy_process_group()
    q.put((rank, tables, sorted(opened), sorted(bases)))


def test_two_rank_gloo_peer_table_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ep_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, t0, o0, b0), (r1, t1, o1, b1) = out
    # own entries are local pointers; peers' = opened base + the exporter's offset
    assert t0 == {"q": [11, 2_000_000], "s": [22, 2_004_096], "x": [33, 2_500_064]}
    assert t1 == {"q": [1_000_000, 11], "s": [1_004_096, 22], "x": [1_500_064, 33]}
    assert o0 == [b"A1", b"B1"] and o1 == [b"A0", b"B0"]          # each distinct handle opened once
    assert b0 == [2_000_000, 2_500_000] and b1 == [1_000_000, 1_500_000]


def test_expert_and_token_ranges():
    from paper_2511_02302_b200 import ep

    assert [ep.expert_range(r, 8, 256) for r in (0, 7)] == [(0, 32), (224, 32)]
    assert ep.token_range(3, 2048) == (6144, 8192)
    with pytest.raises(ValueError):
        ep.expert_range(0, 3, 256)
    from paper_2511_02302_b200 import roofline as RL

    assert RL.dispatch_permute_bytes(10, 32, 100, 8, 256) == 10 * 258 + 32 * 258 + 100 * 8 * 4
    assert RL.combine_bytes(4, 8, 128, True) == 4 * 8 * 256 + 4 * 256 + 4 * 8 * 12


def _ipc_fail_worker(rank, world, port, q):
    """IpcPeers when one rank cannot export a handle: every rank still joins the all-gather and
    every rank raises (no rank is left waiting in a collective)."""
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import torch
    import torch.distributed as dist

    from paper_2511_02302_b200 import ep
    from paper_2511_02302_b200 import fp8flow as F

    dist.init_process_group("gloo", rank=rank, world_size=world)

    def fake_get(t):
        if rank == 1:
            raise F.Fp8FlowError("export failed (simulated)")
        return b"H" * 64, 0

    F.fp8flow_ipc_get_handle = fake_get          # this process only (spawned)
    F.fp8flow_ipc_open = lambda h: 1000
    raised = None
    try:
        ep.IpcPeers({"q": torch.zeros(4)})
    except F.Fp8FlowError as e:
        raised = str(e)
    dist.barrier()                               # both ranks reach this: nobody hung in all_gather
    dist.destroy_process_group()
    q.put((rank, raised))


def test_ipc_export_failure_raises_on_every_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_fail_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(msg is not None and "rank(s) [1]" in msg for _, msg in out), out


# ------------------------------------------------------------------ strong partition + N>1 reports
def _strong_worker(rank, world, port, q):
    """bench.py's N>1 host logic on gloo: the strong split of the layer (experts and entry-cast
    tokens), the per-rank verification reports gathered to every rank and merged (parity of every
    rank, checksum agreement, the CPU-oracle baseline as one job)."""
    os.environ.update({"RANK": str(rank), "LOCAL_RANK": str(rank), "WORLD_SIZE": str(world),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import numpy as np

    import synth
    from paper_2511_02302_b200 import dist as D

    assert D.init("gloo")
    sh = D.shard(rank, world, "strong")
    idx, probs = synth.routing(16384, synth.BASE_SEED)
    rs = synth.expert_range_shard(idx, probs, sh["expert_begin"], sh["num_local_experts"])
    counts = np.bincount(idx.numpy().ravel(), minlength=256)
    per = counts[sh["expert_begin"]: sh["expert_begin"] + sh["num_local_experts"]]
    rows = int(np.sum((per + 15) // 16 * 16))
    rep = {"parity": {"A1_quantize_x": True, "A2_transpose_xperm": rank == 0 or world == 1},
           "checksums_match": True,
           "cpu": {"seconds": 2.0 + rank, "bytes": 1e9 * (rank + 1), "cores": 4, "sample": "shard",
                   "single_thread": {"value": 0.1 + rank, "unit": "GB/s", "cores": 1}}}
    reports = D.gather_objects(rep)
    merged = D.merge_rank_reports(reports)
    D.barrier()
    q.put((rank, sh, len(rs.recv_tokens), rows, merged))
    D.dist.destroy_process_group()


def test_two_rank_gloo_strong_partition_and_reports():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_strong_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, s0, n0, r0, m0), (_, s1, n1, r1, m1) = out
    # GPU g of n owns experts [g*256/n, (g+1)*256/n) and tokens [g*T/n, (g+1)*T/n)
    assert (s0["expert_begin"], s0["num_local_experts"], s0["token_begin"], s0["token_end"]) == (0, 128, 0, 8192)
    assert (s1["expert_begin"], s1["num_local_experts"], s1["token_begin"], s1["token_end"]) == (128, 128, 8192, 16384)
    # the two halves cover the whole layer: ~133k padded rows, every token received by >= 1 rank
    import synth
    import numpy as np
    idx, _ = synth.routing(16384, synth.BASE_SEED)
    counts = np.bincount(idx.numpy().ravel(), minlength=256)
    assert r0 + r1 == int(np.sum((counts + 15) // 16 * 16)) and r0 != r1       # skewed: imbalance
    assert n0 <= 16384 and n1 <= 16384 and n0 + n1 >= 16384
    # merged reports: every rank's parity, a failing rank flips the overall flag, baseline as one job
    assert m0 == m1
    assert m0["parity"] == {"rank0": {"A1_quantize_x": True, "A2_transpose_xperm": True},
                            "rank1": {"A1_quantize_x": True, "A2_transpose_xperm": False}}
    assert m0["parity_all_ranks"] is False and m0["checksums_match"] is True
    assert m0["cpu_baseline"]["value"] == round(3e9 / 3.0 / 1e9, 4) and m0["cpu_baseline"]["cores"] == 8
    assert m0["cpu_baseline"]["single_thread"]["value"] == 0.1         # rank 0's single-threaded timing


def test_partition_modes_single_process():
    from paper_2511_02302_b200 import dist as D

    whole = D.shard(0, 1, "strong")
    assert (whole["expert_begin"], whole["num_local_experts"], whole["token_begin"], whole["token_end"]) == \
        (0, 256, 0, 16384)
    assert [D.shard(r, 8, "strong")["expert_begin"] for r in range(8)] == [32 * r for r in range(8)]
    assert D.shard(3, 4, "weak")["expert_begin"] == 96 and D.shard(9, 16, "weak")["group"] == 1
    with pytest.raises(ValueError):
        D.shard(0, 3, "strong")
    with pytest.raises(ValueError):
        D.shard(0, 1, "sideways")


def test_balanced_placement_is_a_partition_and_balances():
    """--partition balanced: every expert on exactly one GPU, 256/n per GPU, padded rows within
    0.2 % of the mean on the layer's routing (contiguous ranges: up to 1.46x at n = 8)."""
    import numpy as np

    import synth
    from paper_2511_02302_b200 import dist as D

    idx, _ = synth.routing(16384, synth.BASE_SEED)
    counts = np.bincount(idx.numpy().ravel(), minlength=256)
    padded = (counts + 15) // 16 * 16
    for n in (1, 2, 4, 8):
        sets = D.balanced_placement(counts, n)
        assert sorted(e for s in sets for e in s) == list(range(256))
        assert all(len(s) == 256 // n for s in sets)
        loads = [int(padded[s].sum()) for s in sets]
        assert max(loads) / np.mean(loads) < 1.002, loads
        new_id = D.balanced_relabel(counts, n)
        assert sorted(new_id) == list(range(256))
        for g, s in enumerate(sets):             # GPU g's set becomes the id range of rank g
            assert sorted(new_id[e] for e in s) == list(range(g * 256 // n, (g + 1) * 256 // n))
    contiguous = [int(padded[g * 32:(g + 1) * 32].sum()) for g in range(8)]
    assert max(contiguous) / np.mean(contiguous) > 1.4
