"""World-size-2 gloo tests of the multi-GPU host logic (no GPU needed).

The device kernels (ss_route_records, ss_export_moves_dev,
ss_import_blob_dev) are replaced here by their specifications -- a stable
split by owner into packed 8-byte records, and the migration blob layout --
so that the control exchange, the one-message record exchange in
source-rank order, the count all-reduce and the blob exchange of
paper_1309_0634_b200/sharded.py are exercised across real processes.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _stable_split(g, a, owner, world):
    """Specification of ss_route: stable partition by owner."""
    o = owner[g]
    order = np.argsort(o, kind="stable")
    return g[order], a[order], np.bincount(o, minlength=world)


def _worker_exchange(rank, world, port, q):
    from paper_1309_0634_b200 import sharded as S
    _init(rank, world, port)
    rng = np.random.default_rng(5)
    G, B = 50, 4000
    gl = rng.integers(0, G, B)
    al = rng.integers(-1000, 1000, B)
    owner = (np.arange(G) * 7 % world).astype(np.int64)
    lo, hi = rank * B // world, (rank + 1) * B // world
    sg, sa, cnt = _stable_split(gl[lo:hi], al[lo:hi], owner, world)
    # control block: tuples per peer, bad-tuple status, migration words
    ctrl = torch.stack([torch.as_tensor(cnt, dtype=torch.int64), torch.full((world,), -1, dtype=torch.int64),
                        torch.arange(world, dtype=torch.int64) + 10 * rank], dim=1)
    sent, got = S.exchange_control(ctrl)
    ok = sent[:, 0].tolist() == cnt.tolist() and got[:, 2].tolist() == [10 * r + rank for r in range(world)]
    # one packed 8-byte record per tuple: (u32 group, i32 attr) little-endian
    rec = torch.as_tensor((sg.astype(np.uint32).astype(np.uint64)
                           | (sa.astype(np.int32).view(np.uint32).astype(np.uint64) << np.uint64(32))).view(np.int64))
    out = S.exchange_records(rec, sent[:, 0], got[:, 0]).numpy().view(np.uint32).reshape(-1, 2)
    mine = owner[gl] == rank
    ok = ok and out[:, 0].tolist() == gl[mine].tolist() and out[:, 1].view(np.int32).tolist() == al[mine].tolist()
    # count all-reduce: each group's count lives on its owner only
    c = torch.as_tensor(np.bincount(out[:, 0].astype(np.int64), minlength=G).astype(np.int32))
    S.allreduce_counts(c)
    ok = ok and c.tolist() == np.bincount(gl, minlength=G).tolist()
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


def _blob_encode(states, moves, rank, world):
    """Specification of k_export_plan: per destination [n] ++ n records
    (g, fill, next_pos, sum_lo, sum_hi, min, max, span) ++ ring images."""
    segs = []
    for d in range(world):
        gs = [g for g, s, dd, _ in moves if s == rank and dd == d and d != rank]
        if not gs:
            segs.append(np.zeros(0, dtype=np.int32))
            continue
        recs, vals = [], []
        for g in gs:
            f, np_, sm, mn, mx, v = states[g]
            u = np.uint64(np.int64(sm).view(np.uint64))
            recs += [g, f, np_, int(np.uint32(u & np.uint64(0xffffffff)).view(np.int32)),
                     int(np.uint32(u >> np.uint64(32)).view(np.int32)), mn, mx, len(v)]
            vals += list(v)
        segs.append(np.asarray([len(gs)] + recs + vals, dtype=np.int32))
    return segs


def _blob_decode(buf, seg_off):
    """Specification of k_import."""
    out = {}
    for s in range(len(seg_off) - 1):
        seg = buf[seg_off[s]:seg_off[s + 1]]
        if not len(seg):
            continue
        n = int(seg[0])
        v = 1 + 8 * n
        for j in range(n):
            r = seg[1 + 8 * j:9 + 8 * j].astype(np.int64)
            sm = int((np.uint64(np.uint32(r[4])) << np.uint64(32) | np.uint64(np.uint32(r[3]))).view(np.int64))
            out[int(r[0])] = (int(r[1]), int(r[2]), sm, int(r[5]), int(r[6]), seg[v:v + r[7]].tolist())
            v += int(r[7])
    return out


def _worker_migrate(rank, world, port, q):
    from paper_1309_0634_b200 import sharded as S
    _init(rank, world, port)
    # per-rank window states: group -> (fill, next_pos, sum, min, max, ring image)
    states = {g: (g + 1, g % 3, -(10 ** 12) * g - 7, -g, g, (np.arange(g + 1) + 100 * g).tolist())
              for g in range(8) if g % world == rank}
    moves = [(0, 0, 1, "back"), (3, 1, 0, "back"), (5, 1, 0, "front"), (6, 0, 0, "back"), (4, 0, 1, "front")]
    segs = _blob_encode(states, moves, rank, world)
    send_w = np.asarray([len(x) for x in segs], dtype=np.int64)
    ctrl = torch.stack([torch.zeros(world, dtype=torch.int64), torch.full((world,), -1, dtype=torch.int64),
                        torch.as_tensor(send_w)], dim=1)
    sent, got = S.exchange_control(ctrl)
    buf = torch.as_tensor(np.concatenate(segs) if send_w.sum() else np.zeros(1, dtype=np.int32))
    recv = S.exchange_words(buf, sent[:, 2], got[:, 2]).numpy()
    seg_off = np.concatenate([[0], np.cumsum(got[:, 2])])
    got_states = _blob_decode(recv, seg_off)
    expect = {}
    for g, src, dst, _ in moves:
        if dst == rank and src != rank:
            f = g + 1
            expect[g] = (f, g % 3, -(10 ** 12) * g - 7, -g, g, (np.arange(f) + 100 * g).tolist())
    q.put((rank, got_states == expect))
    dist.destroy_process_group()


@pytest.mark.parametrize("worker", [_worker_exchange, _worker_migrate])
def test_two_ranks(worker):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
