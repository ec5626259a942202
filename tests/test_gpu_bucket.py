"""The bucketed placement (bucket.cuh, G > 2^14 and W >= 8192) against the
radix passes and against the window identities of test_gpu_fullsize, with
the window CONTENTS of sampled groups compared in arrival order (the order
is what later evictions depend on, engine.py:72-77,243-248): hot groups
(batch count >= 8192, written straight to their runs by pass 1), cold
groups (staged by bucket, sorted locally by pass 2), ragged batches, and
windows that wrap across batches."""

import numpy as np
import pytest

from test_gpu_fullsize import _expected, _zipf

pytestmark = pytest.mark.gpu


def _contents(groups, attrs, G, W, sample):
    out = {}
    for g in sample:
        v = attrs[groups == g]
        out[int(g)] = v[-W:] if len(v) > W else v
    return out


@pytest.mark.parametrize("bucket", ["1", "0"])
@pytest.mark.parametrize("G,W,s,B,nb,policy,split", [
    (20_000, 8_192, 0.0, (1 << 22) - 13, 5, "no", False),          # cold windows wrap (~1050/batch)
    (100_000, 1_000_000, 1.5, (1 << 24) - 777, 2, "prob", True),   # C3 shape: hot groups drop tuples
    (50_000, 10_000, 1.1, (1 << 21) + 5, 4, "best", False),       # hot groups wrap, cold buckets
    (1_000_000, 10_000_000, 1.0, 1 << 22, 2, "prob", True),       # C4 G/W at a smaller batch
])
def test_bucket_placement(monkeypatch, bucket, G, W, s, B, nb, policy, split):
    import torch
    from paper_1309_0634_b200.stream_engine import StreamEngine
    monkeypatch.setenv("SS_B200_BUCKET", bucket)  # 1 = bucketed passes, 0 = radix passes
    rng = np.random.default_rng(G + nb)
    eng = StreamEngine(G, W, n_partitions=148, aggregates=("count", "sum", "avg", "min", "max"),
                       max_batch=B, initial="hash")
    bal = StreamEngine.balancer_struct(policy, max(1, B // 1480), 0.5, split=split)
    gs, avs = [], []
    for i in range(nb):
        n = B - 3 * i
        g = _zipf(n, G, s, rng) if s > 0 else rng.integers(0, G, n)
        a = rng.integers(-2 ** 31, 2 ** 31, n, dtype=np.int64)
        rep = eng.step(torch.from_numpy(g.astype(np.int32)).cuda(), torch.from_numpy(a.astype(np.int32)).cuda(), bal)
        assert rep.tuples == n
        gs.append(g)
        avs.append(a)
    groups, attrs = np.concatenate(gs), np.concatenate(avs)
    fill, wsum, mn, mx, nxt, t = _expected(groups, attrs, G, W)
    snap = eng.snapshot()
    assert np.array_equal(snap["fill"], fill)
    assert np.array_equal(snap["next_pos"], nxt)
    assert np.array_equal(snap["window_sum"], wsum)
    assert np.array_equal(snap["min"][t], mn[t]) and np.array_equal(snap["max"][t], mx[t])
    # window contents in arrival order: the hottest groups and a random sample
    K = np.bincount(groups, minlength=G)
    sample = list(np.argsort(-K, kind="stable")[:8]) + list(rng.choice(np.nonzero(K)[0], 24, replace=False))
    if len(attrs) < 60_000_000:
        exp = _contents(groups, attrs, G, W, sample)
        for g, v in exp.items():
            assert np.array_equal(eng.contents(g), v), g
    eng.close()
