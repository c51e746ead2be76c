"""GPU parity for NEXT-3 (expert-parallel FP8 dispatch fused with permute + pad, BF16 combine fused
with unpermute; R34) through the C ABI, against the oracle (oracle.dispatch_permute_pad,
oracle.combine) on the same seeded inputs.

Bar: bit-exact codes, scale bytes, plan and BF16 outputs.  The ranks are "virtual" (n ranks'
buffers on the one device, peer tables = local pointers) except in the IPC test, where two
processes share the GPU through CUDA IPC handles exchanged over gloo -- the same plumbing as one
process per GPU on the 8-GPU box.
"""
import os
import socket

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_02302_b200 import fp8flow

    fp8flow.fp8flow_device_check()
    return fp8flow


def host(t):
    return t.cpu().numpy()


def make_ranks(F, n, tpr, H, E, K, seed, gain_sigma=1.0):
    """Per rank: BF16 activations -> A1 on the device (codes + scales), routing, gates."""
    ranks = []
    ld = (tpr + 15) // 16 * 16
    for r in range(n):
        x = synth.activations_bf16(tpr, H, seed + r, gain_sigma=gain_sigma)
        q = torch.empty(tpr, H, dtype=torch.uint8, device="cuda")
        s = torch.zeros(H // 128, ld, dtype=torch.uint8, device="cuda")
        if tpr:
            F.fp8flow_quantize_rowwise(x.cuda(), q, s)
        idx, p = synth.routing(tpr, seed * 7 + r, num_experts=E, top_k=K, num_groups=min(8, E // 4),
                               topk_groups=min(4, max(1, K // 2)))
        ranks.append({"q": q, "s": s, "topk": idx.cuda(), "probs": p.cuda()})
    torch.cuda.synchronize()
    return ranks, ld


def run_dispatch(F, ranks, ld, rank, tpr, H, E, K, align=16, kernel=0):
    from paper_2511_02302_b200 import ep

    n = len(ranks)
    peers = ep.LocalPeers(ranks)
    _, per = ep.expert_range(rank, n, E)
    max_rows = F.permute_max_rows(n * tpr, K, per, align)
    topk_all = torch.empty(max(n * tpr, 1), K, dtype=torch.int32, device="cuda")[: n * tpr]
    row_map = torch.empty(n * tpr, K, dtype=torch.int32, device="cuda")
    src = torch.empty(max_rows, dtype=torch.int32, device="cuda")
    off = torch.empty(per + 1, dtype=torch.int32, device="cuda")
    ws = torch.empty(F.fp8flow_permute_workspace_bytes(n * tpr, K, per), dtype=torch.uint8, device="cuda")
    q_out = torch.full((max_rows, H), 0xEE, dtype=torch.uint8, device="cuda")
    s_out = torch.full((H // 128, max_rows), 0xEE, dtype=torch.uint8, device="cuda")
    ep.dispatch_permute(peers, rank, tpr, H, K, E, ld, topk_all, row_map, src, off, ws, q_out, s_out, align=align,
                        kernel=kernel)
    torch.cuda.synchronize()
    return dict(topk_all=topk_all, row_map=row_map, src=src, off=off, q_out=q_out, s_out=s_out, max_rows=max_rows)


@pytest.mark.parametrize("kernel", ["engine", "lsu"])
@pytest.mark.parametrize("n,tpr,H,E,K", [(1, 300, 1024, 16, 4), (2, 256, 7168, 32, 8), (4, 100, 1152, 64, 8),
                                         (8, 64, 7168, 256, 8), (2, 0, 256, 8, 2)])
def test_dispatch_permute_parity(F, orc, n, tpr, H, E, K, kernel):
    """Both dispatch kernels: the bulk-copy engine (peers on this device) and the register-copy
    kernel the launcher takes when a peer lives on another GPU (NVLink)."""
    kern = F.DISPATCH_REGISTER if kernel == "lsu" else F.DISPATCH_ENGINE
    ranks, ld = make_ranks(F, n, tpr, H, E, K, 1000 + n * tpr)
    qs = [host(r["q"]) for r in ranks]
    ss = [host(r["s"]) for r in ranks]
    ts = [host(r["topk"]) for r in ranks]
    for g in range(n):
        out = run_dispatch(F, ranks, ld, g, tpr, H, E, K, kernel=kern)
        qo_ref, so_ref, rm_ref, src_ref, off_ref = orc.dispatch_permute_pad(qs, ss, ts, g, E,
                                                                            max_rows=out["max_rows"])
        off = host(out["off"])
        R = int(off[-1])
        assert np.array_equal(host(out["topk_all"]), np.concatenate(ts) if tpr else np.zeros((0, K), np.int32))
        assert np.array_equal(off, off_ref) and np.array_equal(host(out["row_map"]), rm_ref)
        qo, so = host(out["q_out"]), host(out["s_out"])
        assert np.array_equal(qo[:R], qo_ref[:R]) and np.array_equal(so[:, :R], so_ref[:, :R])
        assert np.all(qo[R:] == 0xEE) and np.all(so[:, R:] == 0xEE)             # rows >= R untouched


def test_dispatch_equals_device_permute_of_concatenation_full_size(F):
    """DeepSeek-V3 sizes: 8 ranks x 2048 tokens (16384), hidden 7168, top-8 of 256 experts.  Every
    rank's result is byte-identical to A3 (itself oracle-parity-tested) on the concatenated tokens,
    and sampled rows equal their source token's bytes (the definition, R34)."""
    n, tpr, H, E, K = 8, 2048, 7168, 256, 8
    ranks, ld = make_ranks(F, n, tpr, H, E, K, 77)
    q_cat = torch.cat([r["q"] for r in ranks])
    s_cat = torch.cat([r["s"][:, :tpr] for r in ranks], dim=1).contiguous()
    rng = np.random.default_rng(0)
    for g in (0, 5, 7):
        out = run_dispatch(F, ranks, ld, g, tpr, H, E, K)
        ref_q = torch.full_like(out["q_out"], 0xEE)
        ref_s = torch.full_like(out["s_out"], 0xEE)
        F.fp8flow_permute_pad(q_cat, s_cat, out["row_map"], out["src"], out["off"], ref_q, ref_s)
        torch.cuda.synchronize()
        assert torch.equal(out["q_out"], ref_q) and torch.equal(out["s_out"], ref_s)
        src, R = host(out["src"]), int(host(out["off"])[-1])
        for r in rng.integers(0, R, 64):
            t = int(src[r])
            if t < 0:
                assert int(out["q_out"][r].abs().sum()) == 0
                continue
            assert torch.equal(out["q_out"][r], ranks[t // tpr]["q"][t % tpr])
            assert torch.equal(out["s_out"][:, r], ranks[t // tpr]["s"][:, t % tpr])


@pytest.mark.parametrize("with_probs", [True, False])
@pytest.mark.parametrize("n,tpr,H,E,K", [(1, 200, 1024, 16, 4), (2, 128, 7168, 32, 8), (4, 96, 2048, 64, 8),
                                         (8, 40, 7168, 256, 8)])
def test_combine_parity(F, orc, n, tpr, H, E, K, with_probs):
    from paper_2511_02302_b200 import ep

    ranks, ld = make_ranks(F, n, tpr, 256, E, K, 2000 + n)   # codes unused here; routing + gates
    plans = [run_dispatch(F, ranks, ld, g, tpr, 256, E, K) for g in range(n)]
    for g in range(n):
        rows = plans[g]["max_rows"]
        ranks[g]["x"] = synth.normal_bf16(rows, H, 3000 + g).cuda()
        ranks[g]["row_map"] = plans[g]["row_map"]
    peers = ep.LocalPeers(ranks)
    xs = [synth.bf16_bits(r["x"].cpu()) for r in ranks]
    rms = [host(p["row_map"]) for p in plans]
    for g in range(n):
        y = torch.empty(tpr, H, dtype=torch.bfloat16, device="cuda")
        p = ranks[g]["probs"] if with_probs else None
        ep.combine(peers, g, tpr, H, E, ranks[g]["topk"], p, y)
        torch.cuda.synchronize()
        y_ref = orc.combine(xs, rms, host(ranks[g]["topk"]), E // n, probs=host(p) if with_probs else None,
                            token_begin=g * tpr)
        assert np.array_equal(host(y.view(torch.int16)).view(np.uint16), y_ref)


def test_dispatch_then_combine_round_trip_is_K_times_dequant(F):
    """Identity experts (exact dequant of the dispatched rows to BF16) and gates = 1: the combine of
    the dispatch returns K * dequant(Q) exactly (K = 8 copies summed in fp32 are exact)."""
    from paper_2511_02302_b200 import ep

    n, tpr, H, E, K = 4, 256, 7168, 256, 8
    ranks, ld = make_ranks(F, n, tpr, H, E, K, 99)

    def dequant(q, s):   # torch's own E4M3 decode, times 2^(s-127): exact in BF16
        v = q.view(torch.float8_e4m3fn).to(torch.float64)
        return (v * torch.exp2(s.t().to(torch.float64) - 127).repeat_interleave(128, dim=1)).to(torch.bfloat16)

    for g in range(n):
        out = run_dispatch(F, ranks, ld, g, tpr, H, E, K)
        R = int(host(out["off"])[-1])
        x = torch.zeros(out["max_rows"], H, dtype=torch.bfloat16, device="cuda")
        x[:R] = dequant(out["q_out"][:R], out["s_out"][:, :R])
        ranks[g]["x"], ranks[g]["row_map"] = x, out["row_map"]
    peers = ep.LocalPeers(ranks)
    for g in range(n):
        y = torch.empty(tpr, H, dtype=torch.bfloat16, device="cuda")
        ep.combine(peers, g, tpr, H, E, ranks[g]["topk"], None, y)
        torch.cuda.synchronize()
        ref = dequant(ranks[g]["q"], ranks[g]["s"][:, :tpr]).to(torch.float64) * K
        assert torch.equal(y.to(torch.float64), ref)


def test_peer_barrier_virtual_ranks_and_timeout(F):
    """n ranks on n streams (co-resident): every barrier completes with status 0 and advances each
    rank's epoch; a barrier with an absent peer returns status 1 after its timeout, not a hang."""
    from paper_2511_02302_b200 import ep

    n = 4
    sig = [ep.signal_buffer(n, "cuda") for _ in range(n)]
    status = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    table = [t.data_ptr() for t in sig]
    streams = [torch.cuda.Stream() for _ in range(n)]
    torch.cuda.synchronize()
    for it in range(3):
        for r in range(n):
            F.fp8flow_peer_barrier(table, r, status[r:r + 1], timeout_ms=5000, stream=streams[r])
        torch.cuda.synchronize()
        assert status.tolist() == [0] * n
        for r in range(n):
            assert sig[r].tolist() == [it + 1] * (n + 1)
    lone = [ep.signal_buffer(2, "cuda") for _ in range(2)]
    st = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    F.fp8flow_peer_barrier([t.data_ptr() for t in lone], 0, st, timeout_ms=50)
    torch.cuda.synchronize()
    assert st.item() == 1


# ------------------------------------------------------------------------------- two processes
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q, kernel=0):
    try:
        os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
        import torch.distributed as dist

        import oracle
        from paper_2511_02302_b200 import ep
        from paper_2511_02302_b200 import fp8flow as F

        dist.init_process_group("gloo", rank=rank, world_size=world)
        tpr, H, E, K = 192, 2048, 32, 8
        ranks, ld = make_ranks(F, world, tpr, H, E, K, 4242)   # same seeds everywhere: rank r keeps ranks[r]
        mine = ranks[rank]
        qs = [r["q"].cpu().numpy() for r in ranks]
        ss = [r["s"].cpu().numpy() for r in ranks]
        ts = [r["topk"].cpu().numpy() for r in ranks]
        for r in range(world):               # peers' data is reachable only through IPC from here on
            if r != rank:
                ranks[r] = None
        _, per = ep.expert_range(rank, world, E)
        max_rows = F.permute_max_rows(world * tpr, K, per)
        bufs = dict(q=mine["q"], s=mine["s"], topk=mine["topk"],
                    x=synth.normal_bf16(max_rows, H, 5000 + rank).cuda(),
                    row_map=torch.empty(world * tpr, K, dtype=torch.int32, device="cuda"))
        torch.cuda.synchronize()
        peers = ep.IpcPeers(bufs)
        topk_all = torch.empty(world * tpr, K, dtype=torch.int32, device="cuda")
        src = torch.empty(max_rows, dtype=torch.int32, device="cuda")
        off = torch.empty(per + 1, dtype=torch.int32, device="cuda")
        ws = torch.empty(F.fp8flow_permute_workspace_bytes(world * tpr, K, per), dtype=torch.uint8, device="cuda")
        q_out = torch.zeros(max_rows, H, dtype=torch.uint8, device="cuda")
        s_out = torch.zeros(H // 128, max_rows, dtype=torch.uint8, device="cuda")
        ep.dispatch_permute(peers, rank, tpr, H, K, E, ld, topk_all, bufs["row_map"], src, off, ws, q_out, s_out,
                            kernel=kernel)
        torch.cuda.synchronize()
        dist.barrier()                       # every rank's row_map is complete before the combine
        y = torch.empty(tpr, H, dtype=torch.bfloat16, device="cuda")
        ep.combine(peers, rank, tpr, H, E, mine["topk"], mine["probs"], y)
        torch.cuda.synchronize()
        # oracle side
        qo_ref, so_ref, rm_ref, _, off_ref = oracle.dispatch_permute_pad(qs, ss, ts, rank, E, max_rows=max_rows)
        R = int(off_ref[-1])
        ok_d = (np.array_equal(off.cpu().numpy(), off_ref) and np.array_equal(bufs["row_map"].cpu().numpy(), rm_ref)
                and np.array_equal(q_out.cpu().numpy()[:R], qo_ref[:R])
                and np.array_equal(s_out.cpu().numpy()[:, :R], so_ref[:, :R]))
        xs = [None] * world
        rms = [None] * world
        dist.all_gather_object(xs, synth.bf16_bits(bufs["x"].cpu()))
        dist.all_gather_object(rms, bufs["row_map"].cpu().numpy())
        y_ref = oracle.combine(xs, rms, ts[rank], per, probs=mine["probs"].cpu().numpy(), token_begin=rank * tpr)
        ok_c = np.array_equal(y.view(torch.int16).cpu().numpy().view(np.uint16), y_ref)
        dist.barrier()                       # peers stop reading before the mappings go away
        peers.close()
        dist.destroy_process_group()
        q.put((rank, ok_d, ok_c, None))
    except Exception as e:  # noqa: BLE001 -- reported to the parent
        import traceback

        q.put((rank, False, False, traceback.format_exc()))
        del e


@pytest.mark.parametrize("kernel", [0, 2])
def test_two_processes_over_cuda_ipc(F, kernel):
    """kernel 0 (AUTO): the launcher's own choice (same device -> bulk-copy engine); 2 (REGISTER): the
    register-copy kernel used across GPUs."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q, kernel)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_d, ok_c, err in res:
        assert err is None, err
        assert ok_d and ok_c, (rank, ok_d, ok_c)


@pytest.mark.parametrize("kernel", ["engine", "lsu"])
def test_dispatch_combine_edge_cases(F, orc, kernel):
    """A rank that receives nothing (every token routed to the other rank's experts), top_k = 1 and
    top_k = 16, an odd token count (routing bytes not a multiple of 16): both dispatch kernels and
    the combine stay bit-exact against the oracle."""
    from paper_2511_02302_b200 import ep

    kern = F.DISPATCH_REGISTER if kernel == "lsu" else F.DISPATCH_ENGINE
    H = 512
    # (37 tokens x top-1 = 148 routing bytes per rank: the routing gather's 4-byte-word path)
    for n, tpr, E, K, force in [(2, 64, 8, 2, "low"), (2, 48, 32, 1, None), (2, 40, 64, 16, None),
                                (2, 37, 16, 1, None)]:
        ranks, ld = make_ranks(F, n, tpr, H, E, K, 555 + K)
        if force == "low":   # every token picks experts of rank 0 only: rank 1 receives nothing
            for r in ranks:
                r["topk"] = torch.stack([torch.arange(K, dtype=torch.int32)] * tpr).cuda().contiguous()
        qs = [host(r["q"]) for r in ranks]
        ss = [host(r["s"]) for r in ranks]
        ts = [host(r["topk"]) for r in ranks]
        outs = []
        for g in range(n):
            out = run_dispatch(F, ranks, ld, g, tpr, H, E, K, kernel=kern)
            qo_ref, so_ref, rm_ref, _, off_ref = orc.dispatch_permute_pad(qs, ss, ts, g, E, max_rows=out["max_rows"])
            R = int(off_ref[-1])
            if force == "low" and g == 1:
                assert R == 0
            assert np.array_equal(host(out["off"]), off_ref) and np.array_equal(host(out["row_map"]), rm_ref)
            assert np.array_equal(host(out["q_out"])[:R], qo_ref[:R])
            assert np.array_equal(host(out["s_out"])[:, :R], so_ref[:, :R])
            outs.append(out)
        for g in range(n):
            ranks[g]["x"] = synth.normal_bf16(outs[g]["max_rows"], H, 700 + g).cuda()
            ranks[g]["row_map"] = outs[g]["row_map"]
        peers = ep.LocalPeers(ranks)
        xs = [synth.bf16_bits(r["x"].cpu()) for r in ranks]
        rms = [host(o["row_map"]) for o in outs]
        for g in range(n):
            y = torch.empty(tpr, H, dtype=torch.bfloat16, device="cuda")
            ep.combine(peers, g, tpr, H, E, ranks[g]["topk"], ranks[g]["probs"], y)
            torch.cuda.synchronize()
            y_ref = orc.combine(xs, rms, ts[g], E // n, probs=host(ranks[g]["probs"]), token_begin=g * tpr)
            assert np.array_equal(host(y.view(torch.int16)).view(np.uint16), y_ref)


def test_next3_sequence_captures_into_a_cuda_graph(F):
    """Barrier -> routing gather -> plan -> fused dispatch, then combine: every launch is graph-
    capturable (peer tables by value, sizes on the device, the barrier's epoch on the device); a
    replay reproduces the eager outputs bit for bit."""
    from paper_2511_02302_b200 import ep

    n, tpr, H, E, K = 2, 256, 1024, 16, 4
    ranks, ld = make_ranks(F, n, tpr, H, E, K, 4321)
    for r in ranks:
        r["sig"] = ep.signal_buffer(n, "cuda")
    _, per = ep.expert_range(0, n, E)
    mr = F.permute_max_rows(n * tpr, K, per)
    bufs = []
    for g in range(n):
        b = dict(topk_all=torch.empty(n * tpr, K, dtype=torch.int32, device="cuda"),
                 row_map=torch.empty(n * tpr, K, dtype=torch.int32, device="cuda"),
                 src=torch.empty(mr, dtype=torch.int32, device="cuda"),
                 off=torch.empty(per + 1, dtype=torch.int32, device="cuda"),
                 ws=torch.empty(F.fp8flow_permute_workspace_bytes(n * tpr, K, per), dtype=torch.uint8, device="cuda"),
                 q_out=torch.zeros(mr, H, dtype=torch.uint8, device="cuda"),
                 s_out=torch.zeros(H // 128, mr, dtype=torch.uint8, device="cuda"),
                 y=torch.zeros(tpr, H, dtype=torch.bfloat16, device="cuda"),
                 st=torch.full((1,), -1, dtype=torch.int32, device="cuda"))
        bufs.append(b)
        ranks[g]["x"] = synth.normal_bf16(mr, H, 90 + g).cuda()
        ranks[g]["row_map"] = b["row_map"]
    peers = ep.LocalPeers(ranks)
    streams = [torch.cuda.Stream() for _ in range(n)]

    def layer(g, stream):
        b = bufs[g]
        F.fp8flow_peer_barrier(peers.table("sig"), g, b["st"], timeout_ms=2000, stream=stream)
        ep.dispatch_permute(peers, g, tpr, H, K, E, ld, b["topk_all"], b["row_map"], b["src"], b["off"], b["ws"],
                            b["q_out"], b["s_out"], stream=stream)

    def combine(g, stream):
        ep.combine(peers, g, tpr, H, E, ranks[g]["topk"], ranks[g]["probs"], bufs[g]["y"], stream=stream)

    torch.cuda.synchronize()
    for g in range(n):                       # eager, ranks on their own streams (the barrier needs both)
        layer(g, streams[g])
    torch.cuda.synchronize()
    for g in range(n):
        combine(g, streams[g])
    torch.cuda.synchronize()
    eager = [{k: bufs[g][k].clone() for k in ("row_map", "off", "q_out", "s_out", "y")} for g in range(n)]
    for g in range(n):
        for k in ("q_out", "s_out", "y"):
            bufs[g][k].zero_()
    # capture rank g's sequence into its own graph, then replay both graphs concurrently
    graphs = []
    for g in range(n):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=streams[g]):
            layer(g, streams[g])
        graphs.append(gr)
    torch.cuda.synchronize()
    for g in range(n):
        with torch.cuda.stream(streams[g]):
            graphs[g].replay()
    torch.cuda.synchronize()
    for g in range(n):
        combine(g, streams[g])
    torch.cuda.synchronize()
    for g in range(n):
        assert bufs[g]["st"].item() == 0
        for k, v in eager[g].items():
            assert torch.equal(bufs[g][k], v), (g, k)


def test_timed_out_barrier_gates_gather_dispatch_and_combine(F):
    """with the barrier's status nonzero (a peer did not arrive), the gather, both
    dispatch kernels and the combine write nothing; with status 0 they run."""
    n, tpr, H, E, K = 2, 64, 512, 16, 4
    ranks, ld = make_ranks(F, n, tpr, H, E, K, 31337)
    from paper_2511_02302_b200 import ep

    peers = ep.LocalPeers(ranks)
    per = E // n
    mr = F.permute_max_rows(n * tpr, K, per)
    bad = torch.ones(1, dtype=torch.int32, device="cuda")
    topk_all = torch.full((n * tpr, K), -5, dtype=torch.int32, device="cuda")
    F.fp8flow_peer_gather(peers.table("topk"), tpr * K * 4, topk_all, status=bad)
    torch.cuda.synchronize()
    assert torch.all(topk_all == -5)
    good = run_dispatch(F, ranks, ld, 0, tpr, H, E, K)                    # a valid plan for rank 0
    for kernel in (F.DISPATCH_ENGINE, F.DISPATCH_REGISTER):
        q_out = torch.full((mr, H), 0xEE, dtype=torch.uint8, device="cuda")
        s_out = torch.full((H // 128, mr), 0xEE, dtype=torch.uint8, device="cuda")
        F.fp8flow_dispatch_permute_pad(peers.table("q"), peers.table("s"), ld, tpr, H, good["row_map"], good["src"],
                                       good["off"], q_out, s_out, kernel=kernel, status=bad)
        torch.cuda.synchronize()
        assert torch.all(q_out == 0xEE) and torch.all(s_out == 0xEE), kernel
        F.fp8flow_dispatch_permute_pad(peers.table("q"), peers.table("s"), ld, tpr, H, good["row_map"], good["src"],
                                       good["off"], q_out, s_out, kernel=kernel, status=bad.zero_() + 0)
        torch.cuda.synchronize()
        R = int(good["off"][-1])
        assert torch.equal(q_out[:R], good["q_out"][:R]), kernel
        bad.fill_(1)
    for r in range(n):
        ranks[r]["x"] = synth.normal_bf16(mr, H, 90 + r).cuda()
        ranks[r]["row_map"] = good["row_map"]
    peers = ep.LocalPeers(ranks)
    y = torch.full((tpr, H), 7.0, dtype=torch.bfloat16, device="cuda")
    F.fp8flow_combine_unpermute(peers.table("x"), peers.table("row_map"), H, ranks[0]["topk"], per, None, 0, y,
                                status=bad)
    torch.cuda.synchronize()
    assert torch.all(y == 7.0)
