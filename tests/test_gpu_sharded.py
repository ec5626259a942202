"""Two key-sharded ranks end to end on the GPU box.

Only one GPU is available to the tests, so both ranks run their engines
on cuda:0 and exchange through gloo (host tensors); on an 8-GPU box the
same ShardedEngine uses NCCL over NVLink.  Route into packed records
(device), control + record exchange, local fused step on the received
records, GPU-level balancing (device policy on all-reduced device counts,
moves applied on the device) and device-blob window migration are all
exercised, also under a drifting hot set (C5 semantics at a small shape);
the merged state must equal the single-stream oracle (aggregates are
assignment-independent).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stream(G, B, nb, drift):
    from paper_1309_0634_b200 import datagen as D
    if drift:
        # C5 semantics at a small shape: Zipf s=1.2 whose hot set moves every 2 batches
        return D.drifting_zipf(nb * B, G, 1.2, 2 * B, seed=31)
    return D.stream_for(D.DatasetSpec(D.DatasetKind.ZIPF, nb * B, G, 1.2, 31))


def _worker(rank, world, port, q, G, W, B, nb, gpu_policy, drift, pool=0):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1309_0634_b200 import datagen as D
        from paper_1309_0634_b200.sharded import ShardedEngine
        from paper_1309_0634_b200.stream_engine import StreamEngine
        eng = ShardedEngine(G, W, n_partitions=16, aggregates=("count", "sum", "avg", "min", "max"),
                            device=0, max_batch=B, sub_batch=16384, pool_values=pool)
        bal = StreamEngine.balancer_struct("prob", max(1, B // 160), 0.5)
        gbal = StreamEngine.balancer_struct(gpu_policy, max(1, B // 20), 0.5)
        n_moves = 0
        for b in D.batches(_stream(G, B, nb, drift), B):
            lo, hi = rank * len(b) // world, (rank + 1) * len(b) // world
            eng.step(b.groups[lo:hi].astype(np.int32), b.attrs[lo:hi].astype(np.int32), bal, gbal)
            n_moves += len(eng.last_gpu_moves)
        eng.settle()                                    # the last batch's moves land
        snap = eng.local.snapshot()
        owned = np.flatnonzero(eng.owner == rank)
        contents = {int(g): eng.local.contents(int(g)).tolist() for g in owned if g % 13 == 0}
        q.put((rank, owned, {k: snap[k][owned] for k in ("fill", "next_pos", "window_sum", "min", "max", "avg")},
               contents, n_moves, None))
        eng.close()
    except Exception as ex:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, None, None, None, 0, traceback.format_exc()))
    dist.destroy_process_group()


@pytest.mark.parametrize("gpu_policy,drift,pool", [("no", False, 0), ("prob", False, 0), ("prob", True, 0),
                                                    ("best", True, 0), ("prob", True, 3000 * 40 * 4)])
def test_two_ranks_match_oracle(gpu_policy, drift, pool):
    """(pool > 0: occupancy-proportional rings, so imported windows reserve
    ring space on the device)"""
    import torch.multiprocessing as mp
    from oracle import port as O
    from paper_1309_0634_b200 import datagen as D
    G, W, B, nb = 3000, 40, 40_000, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, G, W, B, nb, gpu_policy, drift, pool)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[5] is None, r[5]
    store = O.OStore(G, W)
    for b in D.batches(_stream(G, B, nb, drift), B):
        store.ingest(b.groups, b.attrs)
    cnt, sm, avg, mn, mx = store.aggregates()
    seen = np.zeros(G, dtype=bool)
    moves = 0
    for rank, owned, snap, contents, n_moves, _ in res:
        moves = max(moves, n_moves)
        seen[owned] = True
        assert np.array_equal(snap["fill"], cnt[owned])
        assert np.array_equal(snap["next_pos"], store.next_pos[owned])
        assert np.array_equal(snap["window_sum"], sm[owned])
        assert np.array_equal(snap["min"], mn[owned]) and np.array_equal(snap["max"], mx[owned])
        assert np.array_equal(snap["avg"], avg[owned])
        for g, c in contents.items():
            assert c == store.contents(g).tolist()
    assert seen.all()
    if gpu_policy != "no":
        assert moves > 0


def _worker_bad(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1309_0634_b200.errors import DataError
        from paper_1309_0634_b200.sharded import ShardedEngine
        G = 100
        eng = ShardedEngine(G, 8, n_partitions=4, device=0, max_batch=1000)
        g = (np.arange(500) % G).astype(np.int32)
        a = np.arange(500, dtype=np.int32)
        eng.step(g, a)                                  # a clean batch first
        snap0 = eng.local.snapshot()["window_sum"].copy()
        bad = g.copy()
        if rank == 1:
            bad[37] = G + 5
        msg = None
        try:
            eng.step(bad, a)
        except DataError as ex:
            msg = str(ex)
        # the rejected batch changed nothing; the next clean one is accepted
        same = np.array_equal(eng.local.snapshot()["window_sum"], snap0)
        eng.step(g, a)
        q.put((rank, msg, same, None))
        eng.close()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, None, False, traceback.format_exc()))
    dist.destroy_process_group()


def test_two_ranks_bad_tuple_rejected_everywhere():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_bad, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r[0]: r for r in (q.get(timeout=300) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
    for r in res.values():
        assert r[3] is None, r[3]
        assert r[2]
    assert res[1][1] == "tuple 37 has group 105, outside [0, 100)"
    assert res[0][1].startswith("rank 1 rejected")


def _worker64(rank, world, port, q, G, W, B, nb, pool=0):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1309_0634_b200 import datagen as D
        from paper_1309_0634_b200.sharded import ShardedEngine
        from paper_1309_0634_b200.stream_engine import StreamEngine
        eng = ShardedEngine(G, W, n_partitions=16, aggregates=("count", "sum", "avg", "min", "max"),
                            device=0, max_batch=B, sub_batch=16384, key_bits=64, pool_values=pool)
        bal = StreamEngine.balancer_struct("prob", max(1, B // 160), 0.5)
        gbal = StreamEngine.balancer_struct("prob", max(1, B // 20), 0.5)
        n_moves = 0
        for b in D.batches(_stream(G, B, nb, True), B):
            lo, hi = rank * len(b) // world, (rank + 1) * len(b) // world
            eng.step(D.mix64(b.groups[lo:hi]), b.attrs[lo:hi].astype(np.int32), bal, gbal)
            n_moves += len(eng.last_gpu_moves)
        eng.settle()
        snap = eng.local.snapshot()
        keys = eng.local.slot_keys()
        q.put((rank, keys, eng.owner, {k: snap[k][:len(keys)] for k in ("fill", "next_pos", "window_sum", "min", "max")},
               n_moves, None))
        eng.close()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, None, None, None, 0, traceback.format_exc()))
    dist.destroy_process_group()


@pytest.mark.parametrize("pool", [0, 3000 * 40 * 4])
def test_two_ranks_int64_keys_match_oracle(pool):
    """C5 semantics at a small shape: int64 keys routed by key-hash bucket,
    drifting skew, GPU-level moves of buckets with their keys' windows; every
    key's state on the GPU owning its bucket equals the oracle's."""
    import torch.multiprocessing as mp
    from oracle import port as O
    from paper_1309_0634_b200 import datagen as D
    G, W, B, nb = 3000, 40, 40_000, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker64, args=(r, 2, port, q, G, W, B, nb, pool)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[5] is None, r[5]
    store = O.OStore(G, W)
    for b in D.batches(_stream(G, B, nb, True), B):
        store.ingest(b.groups, b.attrs)
    cnt, sm, avg, mn, mx = store.aggregates()
    seen = np.zeros(G, dtype=np.int64)
    for rank, keys, owner, snap, n_moves, _ in res:
        bucket = (D.mix64(keys).view(np.uint64) >> np.uint64(48)).astype(np.int64)
        mine = owner[bucket] == rank
        g = D.unmix64(keys[mine])
        seen[g] += 1
        assert np.array_equal(snap["fill"][mine], cnt[g])
        assert np.array_equal(snap["next_pos"][mine], store.next_pos[g])
        assert np.array_equal(snap["window_sum"][mine], sm[g])
        assert np.array_equal(snap["min"][mine], mn[g]) and np.array_equal(snap["max"][mine], mx[g])
    touched = np.flatnonzero(cnt > 0)
    assert (seen[touched] == 1).all()
    assert max(r[4] for r in res) > 0
