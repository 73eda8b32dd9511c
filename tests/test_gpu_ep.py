"""GPU: expert parallelism on one B200 through the in-process
loopback transport: P engines (ranks) each own E/P experts and stream only
those; tokens are dispatched to the owners and combined back. The result must
be BIT-IDENTICAL to the single-GPU engine on the same requests: every expert
row is computed by the same kernel in the same K order."""
import dataclasses
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

B, N, PREFIX = 4, 5, 300


def _run_ep(shape, P, tokens, prefix, s_max, debug=True, **kw):
    import torch
    from paper_2508_21706_b200.engine import EpGroup, VerifyEngine
    grp = EpGroup.loopback(P)
    bl = B // P
    engines = [VerifyEngine(shape, max_batch=bl, max_verify=N, max_seq=s_max, debug=debug, ep_rank=r, ep_size=P,
                            ep_group=grp, **kw) for r in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    results, errors = [None] * P, []
    for r, e in enumerate(engines):
        e.fill_prefix(prefix[r * bl:(r + 1) * bl])

    def work(r):
        try:
            results[r] = engines[r].verify(tokens[r * bl:(r + 1) * bl], prefix[r * bl:(r + 1) * bl],
                                           stream=streams[r].cuda_stream)
        except Exception as ex:  # surfaced below
            errors.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errors, errors
    return engines, results, grp


@pytest.mark.parametrize("P,compress,batch_one", [(2, False, False), (4, False, False), (2, True, False),
                                                 (2, False, True), (4, True, True)])
def test_ep_loopback_bit_identical_to_single_gpu(cuda, P, compress, batch_one):
    """Rank r's tokens go to every owner and come back; each token's result
    depends only on its own request, so rank r's EP outputs must equal a
    single-GPU engine run on rank r's requests alone, bit for bit (the
    procedural prefix KV is indexed by the engine-local request). BATCH_ONE:
    each owner streams only its local experts that received rows."""
    from paper_2508_21706_b200.engine import TINY, VerifyEngine
    shape = dataclasses.replace(TINY, seed=0x5EED + 3, lm_scale=8.0, router_scale=4.0)
    s_max = PREFIX + N + 64
    rng = np.random.default_rng(11)
    tokens = rng.integers(0, shape.vocab, size=(B, N)).astype(np.int32)
    prefix = np.array([PREFIX, PREFIX - 3, 200, 1], np.int32)
    engines, results, grp = _run_ep(shape, P, tokens, prefix, s_max, compress_experts=compress, batch_one=batch_one)
    bl = B // P
    for r in range(P):
        ref = VerifyEngine(shape, max_batch=bl, max_verify=N, max_seq=s_max, debug=True)
        ref.fill_prefix(prefix[r * bl:(r + 1) * bl])
        want = ref.verify(tokens[r * bl:(r + 1) * bl], prefix[r * bl:(r + 1) * bl])
        assert np.array_equal(results[r].target, want.target), r
        assert np.array_equal(results[r].acc_len, want.acc_len)
        assert np.array_equal(results[r].bonus, want.bonus)
        for layer in range(shape.n_layers):
            full = ref.debug_tensor("x_out", layer, (bl * N, shape.hidden), np.float32)
            mine = engines[r].debug_tensor("x_out", layer, (bl * N, shape.hidden), np.float32)
            assert np.array_equal(mine.view(np.uint32), full.view(np.uint32)), (r, layer)
        ref.close()
    # each rank streamed only its shard of the experts
    t0 = engines[0].last_times()
    raw = shape.n_layers * (shape.n_expert // P) * shape.expert_bytes
    if batch_one:  # only the routed local experts
        assert 0 < t0["h2d_raw_bytes"] <= raw and t0["h2d_raw_bytes"] % shape.expert_bytes == 0
        raw = t0["h2d_raw_bytes"]
    assert t0["h2d_raw_bytes"] == raw
    if compress:  # coded blocks (unary or tile code), below the 3-bit window's 1456 B per 1024 weights
        assert 0 < t0["h2d_bytes"] <= raw * 1456 // 2048
    else:
        assert t0["h2d_bytes"] == raw
    for e in engines:
        e.close()
    grp.close()


@pytest.mark.parametrize("kind", ["nccl", "loopback"])
def test_ep_single_rank_transport_path(cuda, kind):
    """The full dispatch/combine path through a 1-rank group — NCCL grouped
    send/recv to self (dlopen'd libnccl) or loopback — equals the plain engine
    bit for bit: exercises the NCCL transport on the one GPU available."""
    from paper_2508_21706_b200.engine import TINY, EpGroup, VerifyEngine
    shape = dataclasses.replace(TINY, seed=0x5EED + 4)
    s_max = PREFIX + N + 64
    rng = np.random.default_rng(5)
    tokens = rng.integers(0, shape.vocab, size=(B, N)).astype(np.int32)
    prefix = np.array([PREFIX, 17, 200, 1], np.int32)
    grp = EpGroup.nccl(EpGroup.nccl_unique_id(), 1, 0) if kind == "nccl" else EpGroup.loopback(1)
    outs = []
    for g in (None, grp):
        e = VerifyEngine(shape, max_batch=B, max_verify=N, max_seq=s_max, debug=True, ep_group=g)
        e.fill_prefix(prefix)
        r = e.verify(tokens, prefix)
        outs.append((r, e.debug_tensor("x_out", shape.n_layers - 1, (B * N, shape.hidden), np.float32)))
        e.close()
    assert np.array_equal(outs[0][0].target, outs[1][0].target)
    assert np.array_equal(outs[0][1].view(np.uint32), outs[1][1].view(np.uint32))
    grp.close()


def _ipc_rank(rank, world, port, out_q, staged=False):
    """One process of the IPC expert-parallel test (both on cuda:0)."""
    import os
    import sys
    os.environ["SMO_EP_STAGED"] = "1" if staged else "0"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    try:
        import torch
        import torch.distributed as dist
        from paper_2508_21706_b200.engine import TINY, EpGroup, VerifyEngine
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        shape = dataclasses.replace(TINY, seed=0x5EED + 3, lm_scale=8.0, router_scale=4.0)
        s_max = PREFIX + N + 64
        rng = np.random.default_rng(11)
        tokens = rng.integers(0, shape.vocab, size=(B, N)).astype(np.int32)
        prefix = np.array([PREFIX, PREFIX - 3, 200, 1], np.int32)
        bl = B // world

        def all_gather(blob):
            out = [None] * world
            dist.all_gather_object(out, blob)
            return out

        slot = EpGroup.ipc_slot_bytes(shape, bl, N)
        assert slot % (4 * shape.hidden) == 0  # whole fp32 rows: the engine takes the direct path
        grp = EpGroup.ipc(world, rank, slot, all_gather, dist.barrier)
        eng = VerifyEngine(shape, max_batch=bl, max_verify=N, max_seq=s_max, ep_rank=rank, ep_size=world,
                           ep_group=grp, compress_experts=True)
        mine = slice(rank * bl, (rank + 1) * bl)
        eng.fill_prefix(prefix[mine])
        stream = torch.cuda.Stream()
        # 12 steps: the device-side round flags of the mailbox exchange cycle many times
        got = [eng.verify(tokens[mine], prefix[mine], stream=stream.cuda_stream) for _ in range(12)]
        stream.synchronize()
        eng.close()
        dist.barrier()
        ref = VerifyEngine(shape, max_batch=bl, max_verify=N, max_seq=s_max, compress_experts=True)
        ref.fill_prefix(prefix[mine])
        want = ref.verify(tokens[mine], prefix[mine])
        ok = all(np.array_equal(g.target, want.target) and np.array_equal(g.acc_len, want.acc_len)
                 and np.array_equal(g.bonus, want.bonus) for g in got)
        ref.close()
        grp.close()
        dist.destroy_process_group()
        out_q.put((rank, ok, ""))
    except Exception as ex:  # reported to the parent
        import traceback
        out_q.put((rank, False, traceback.format_exc()))


@pytest.mark.parametrize("staged", [False, True], ids=["direct", "staged"])
def test_ep_ipc_two_processes_bit_identical(cuda, staged):
    """Expert parallelism across two PROCESSES over the peer-memory (CUDA IPC)
    transport — the multi-process path with no NCCL, run here with both ranks
    on one B200: each rank's verify results equal a single-GPU engine's on its
    requests, bit for bit. `direct`: the dispatch / combine kernels store into
    the peer's mailbox themselves; `staged`: pack buffer + copies."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_rank, args=(r, 2, port, q, staged)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for rank, ok, err in sorted(res):
        assert ok, f"rank {rank}: {err}"


def test_ep_dispatch_combine_standalone(cuda):
    """smo_ep_dispatch / smo_ep_combine (the C-ABI pair SURVEY.md §8(b) names)
    around a caller-run expert shard, P = 2 ranks on a loopback group (one host
    thread each): every rank receives exactly the rows routed to its experts,
    grouped by local expert, and the combined output equals the single-device
    sum_j w[t,j] * f_{e(t,j)}(x[t]) for its own tokens."""
    import torch
    from paper_2508_21706_b200.engine import EpGroup
    P, E, k, h, T = 2, 8, 2, 256, 12
    C = T * k
    g = torch.Generator(device="cuda").manual_seed(7)
    xs = [(torch.randn((T, h), generator=g, device="cuda") * 0.5).to(torch.bfloat16) for _ in range(P)]
    ids = [torch.stack([torch.randperm(E, generator=g, device="cuda")[:k] for _ in range(T)]).to(torch.int32)
           for _ in range(P)]
    ws_ = [torch.rand((T, k), generator=g, device="cuda") for _ in range(P)]
    grp = EpGroup.loopback(P)
    nbytes = EpGroup.workspace_bytes(P, T, k, h, E, C)
    out, err = [None] * P, [None] * P

    def scale(e):  # the "expert": y = x * (e + 1) / 2
        return (e + 1) * 0.5

    def rank_fn(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
                xl, off, back, pos_ep = grp.dispatch(r, xs[r], ids[r], E, C, ws, st.cuda_stream)
                st.synchronize()
                offs = off.cpu().numpy()
                yl = torch.zeros((P * C, h), dtype=torch.float32, device="cuda")
                got_rows = []
                for le in range(E // P):
                    rows = slice(int(offs[le]), int(offs[le + 1]))
                    yl[rows] = xl[rows].float() * scale(le * P + r)
                    got_rows.append(xl[rows].float())
                x = torch.zeros((T, h), dtype=torch.float32, device="cuda")
                grp.combine(r, yl, back, off, pos_ep, ws_[r].contiguous(), x, E, C, ws, st.cuda_stream)
                st.synchronize()
                out[r] = (x, got_rows)
        except Exception as ex:  # reported below
            err[r] = ex

    th = [threading.Thread(target=rank_fn, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert all(e is None for e in err), err
    for r in range(P):
        x, got_rows = out[r]
        want = torch.zeros((T, h), dtype=torch.float32, device="cuda")
        for j in range(k):
            f = torch.tensor([scale(int(e)) for e in ids[r][:, j].tolist()], device="cuda")
            want += ws_[r][:, j:j + 1] * f[:, None] * xs[r].float()
        assert torch.allclose(x, want, rtol=1e-5, atol=1e-6), (r, (x - want).abs().max())
        # rank r received exactly the (token, slot) pairs routed to its experts
        for le in range(E // P):
            e = le * P + r
            n_want = sum(int((ids[s] == e).sum()) for s in range(P))
            assert got_rows[le].shape[0] == n_want, (r, le)
    grp.close()


def test_ep_loopback_decode_loop_matches_single_gpu(cuda):
    """The decode loop under expert parallelism: each rank drafts (on-device
    drafter) and commits its own requests; the verify step dispatches their
    rows to the expert owners. Committed histories equal single-GPU engines
    run on each rank's requests, bit for bit."""
    import torch
    from paper_2508_21706_b200.engine import TINY, EpGroup, VerifyEngine
    shape = dataclasses.replace(TINY, seed=0x5EED + 6, lm_scale=8.0, router_scale=4.0, draft_layers=1,
                                draft_inter=512)
    P, k, steps = 2, 3, 3
    s_max = PREFIX + (k + 1) * steps + 64
    rng = np.random.default_rng(21)
    kv = np.array([PREFIX, PREFIX - 3, 200, 9], np.int32)
    root = rng.integers(0, shape.vocab, size=B).astype(np.int32)
    grp = EpGroup.loopback(P)
    bl = B // P
    engines = [VerifyEngine(shape, max_batch=bl, max_verify=k + 1, max_seq=s_max, ep_rank=r, ep_size=P,
                            ep_group=grp) for r in range(P)]
    for r, e in enumerate(engines):
        e.fill_prefix(kv[r * bl:(r + 1) * bl])
        e.decode_begin(root[r * bl:(r + 1) * bl], kv[r * bl:(r + 1) * bl])
    streams = [torch.cuda.Stream() for _ in range(P)]
    errors = []

    def work(r):
        try:
            for _ in range(steps):
                engines[r].decode_step(k, stream=streams[r].cuda_stream)
            streams[r].synchronize()
        except Exception as ex:
            errors.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errors, errors
    for r in range(P):
        mine = slice(r * bl, (r + 1) * bl)
        got = engines[r].decode_read(bl, 64)
        ref = VerifyEngine(shape, max_batch=bl, max_verify=k + 1, max_seq=s_max)
        ref.fill_prefix(kv[mine])
        ref.decode_begin(root[mine], kv[mine])
        for _ in range(steps):
            ref.decode_step(k)
        want = ref.decode_read(bl, 64)
        ref.close()
        for a, b in zip(got, want):
            assert np.array_equal(a, b), r
        assert np.all(got[1] >= steps)
    for e in engines:
        e.close()
    grp.close()
