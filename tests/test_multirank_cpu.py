"""World-size-2 gloo tests of the multi-GPU host logic (no GPU needed).

The device route (ss_route) is replaced here by its specification -- a
stable split by owner -- so that the exchange, its source-rank ordering,
the count all-reduce and the state-migration protocol of
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
    rc = S.exchange_counts(cnt)
    rg, ra = S.exchange_tuples(torch.as_tensor(sg, dtype=torch.int32), torch.as_tensor(sa, dtype=torch.int32),
                               cnt, rc)
    mine = owner[gl] == rank
    ok = (rg.numpy().tolist() == gl[mine].tolist()) and (ra.numpy().tolist() == al[mine].tolist())
    # count all-reduce: each group's count lives on its owner only
    c = np.bincount(rg.numpy(), minlength=G).astype(np.int32)
    tot = S.allreduce_counts(c)
    ok = ok and tot.tolist() == np.bincount(gl, minlength=G).tolist()
    q.put((rank, ok))
    dist.destroy_process_group()


def _worker_migrate(rank, world, port, q):
    from paper_1309_0634_b200 import sharded as S
    _init(rank, world, port)
    # per-rank "window store": group -> (meta, values)
    store = {g: (np.array([g + 1, g % 3, 10 * g, -g, g], dtype=np.int64),
                 np.arange(g + 1, dtype=np.int32) + 100 * g)
             for g in range(8) if g % world == rank}
    moves = [(0, 0, 1, "back"), (3, 1, 0, "back"), (5, 1, 0, "front"), (6, 0, 0, "back")]

    def export_fn(gs):
        meta = np.stack([store[int(g)][0] for g in gs])
        vals = np.concatenate([store[int(g)][1] for g in gs])
        return meta, vals

    got = {}

    def import_fn(gs, meta, vals):
        pos = 0
        for i, g in enumerate(gs):
            n = int(meta[i][0])
            got[int(g)] = (meta[i].tolist(), vals[pos:pos + n].tolist())
            pos += n

    S.migrate(moves, rank, world, export_fn, import_fn)
    expect = {}
    for g, src, dst, _ in moves:
        if dst == rank and src != rank:
            expect[g] = ([g + 1, g % 3, 10 * g, -g, g], (np.arange(g + 1) + 100 * g).tolist())
    q.put((rank, got == expect))
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
