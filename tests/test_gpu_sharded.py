"""Two key-sharded ranks end to end on the GPU box.

Only one GPU is available to the tests, so both ranks run their engines
on cuda:0 and exchange through gloo (host tensors); on an 8-GPU box the
same ShardedEngine uses NCCL over NVLink.  Route (device), exchange,
local fused step, GPU-level balancing (device policy on all-reduced
counts) and window migration are all exercised; the merged state must
equal the single-stream oracle (aggregates are assignment-independent).
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


def _worker(rank, world, port, q, G, W, B, nb, gpu_policy):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1309_0634_b200 import datagen as D
        from paper_1309_0634_b200.sharded import ShardedEngine
        from paper_1309_0634_b200.stream_engine import StreamEngine
        spec = D.DatasetSpec(D.DatasetKind.ZIPF, nb * B, G, 1.2, 31)
        eng = ShardedEngine(G, W, n_partitions=16, aggregates=("count", "sum", "avg", "min", "max"),
                            device=0, max_batch=B, sub_batch=16384)
        bal = StreamEngine.balancer_struct("prob", max(1, B // 160), 0.5)
        gbal = StreamEngine.balancer_struct(gpu_policy, max(1, B // 20), 0.5)
        n_moves = 0
        for b in D.batches(D.stream_for(spec), B):
            lo, hi = rank * len(b) // world, (rank + 1) * len(b) // world
            eng.step(b.groups[lo:hi].astype(np.int32), b.attrs[lo:hi].astype(np.int32), bal, gbal)
            n_moves += len(eng.last_gpu_moves)
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


@pytest.mark.parametrize("gpu_policy", ["no", "prob"])
def test_two_ranks_match_oracle(gpu_policy):
    import torch.multiprocessing as mp
    from oracle import port as O
    from paper_1309_0634_b200 import datagen as D
    G, W, B, nb = 3000, 40, 40_000, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, G, W, B, nb, gpu_policy)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[5] is None, r[5]
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, nb * B, G, 1.2, 31)
    store = O.OStore(G, W)
    for b in D.batches(D.stream_for(spec), B):
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
