"""CPU, world_size 2 over gloo: the host-side logic of the N>1 path.

1. bench.py's rendezvous: rank 0 makes the NCCL unique id through the C-ABI
   (smo_nccl_unique_id needs no GPU) and broadcasts it; max-over-ranks timing.
2. The expert-parallel exchange protocol of ep.cu, restated in numpy and run
   over real gloo all_to_all: owner-major permutation, fixed-capacity blocks
   with per-local-expert counts at the block tail, src-major unpack per local
   expert, return by `back` index, combine at owner-major positions. Every
   (token, slot) pair must get back exactly its own expert's output.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

E, K, H = 8, 2, 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def ep_exchange(ids, x, rank, P, C, expert_fn):
    """numpy restatement of ep.cu's per-layer dispatch/combine around experts."""
    T = ids.shape[0]
    E_loc = E // P
    oid = (ids % P) * E_loc + ids // P                          # ep_remap_kernel
    flat = oid.ravel()
    order = np.argsort(flat, kind="stable")                      # permute_kernel (stable)
    offsets = np.concatenate([[0], np.cumsum(np.bincount(flat, minlength=E))])
    pos = np.empty_like(order)
    pos[order] = np.arange(order.size)
    xp = x[order // K]
    blk_rows = np.zeros((P, C, H), np.float32)                   # ep_pack_kernel
    counts = np.zeros((P, E_loc), np.int64)
    for d in range(P):
        seg = xp[offsets[d * E_loc]:offsets[(d + 1) * E_loc]]
        blk_rows[d, :len(seg)] = seg
        counts[d] = np.diff(offsets[d * E_loc:(d + 1) * E_loc + 1])
    pos_ep = (flat // E_loc) * C + (pos - offsets[(flat // E_loc) * E_loc])   # ep_pos_kernel
    rrows = torch.empty((P, C, H))
    rcnt = torch.empty((P, E_loc), dtype=torch.int64)
    dist.all_to_all_single(rrows, torch.from_numpy(blk_rows))
    dist.all_to_all_single(rcnt, torch.from_numpy(counts))
    rrows, rcnt = rrows.numpy(), rcnt.numpy()
    xl, back, le_of = [], [], []                                 # ep_unpack_kernel
    for le in range(E_loc):
        for s in range(P):
            start = rcnt[s, :le].sum()
            for i in range(rcnt[s, le]):
                xl.append(rrows[s, start + i])
                back.append(s * C + start + i)
                le_of.append(le)
    yl = np.stack([expert_fn(le * P + rank, v) for le, v in zip(le_of, xl)]) if xl else np.zeros((0, H))
    sendback = np.zeros((P * C, H), np.float32)                  # ep_pack_back_kernel
    sendback[back] = yl
    recvback = torch.empty((P, C, H))
    dist.all_to_all_single(recvback, torch.from_numpy(sendback.reshape(P, C, H)))
    return recvback.numpy().reshape(P * C, H)[pos_ep].reshape(T, K, H)   # combine gather


def _worker(rank, P, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        # 1. rendezvous as bench.py does it
        from paper_2508_21706_b200.engine import EpGroup
        uid = [EpGroup.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        got = [None] * P
        dist.all_gather_object(got, uid[0])
        assert all(g == got[0] for g in got) and len(got[0]) == 128
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == P
        # 2. EP exchange protocol
        rng = np.random.default_rng(100 + rank)
        T = 6
        ids = np.stack([rng.choice(E, K, replace=False) for _ in range(T)]).astype(np.int64)
        x = rng.normal(size=(T, H)).astype(np.float32)
        C = T * K

        def expert_fn(e, v):  # owner-only: a rank may only evaluate experts it owns
            assert e % P == rank
            return v * (e + 1)
        out = ep_exchange(ids, x, rank, P, C, expert_fn)
        want = x[:, None, :] * (ids[:, :, None] + 1)
        assert np.allclose(out, want)
        q.put((rank, "ok"))
    except Exception as ex:  # report to the parent
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P", [2])
def test_ep_protocol_and_rendezvous_gloo(P):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, q)) for r in range(P)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(P))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(P)}, res
