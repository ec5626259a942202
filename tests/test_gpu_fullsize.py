"""Parity at BASELINE.json's full shapes (batch 2^24, the configs' G and W)
through size-independent window identities: after a stream of batches the
window of every group holds exactly its last min(K, W) values in arrival
order, so COUNT, SUM, MIN, MAX, AVG and next_pos follow from a stable sort
of the whole stream (numpy, on the box's host).  The per-batch oracle is too
slow at these sizes; these checks are exact (integer, tolerance 0)."""

import numpy as np
import pytest

from paper_1309_0634_b200 import datagen as D

pytestmark = pytest.mark.gpu


def _zipf(n, G, s, rng):
    w = np.arange(1, G + 1, dtype=np.float64) ** -s
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    return np.minimum(np.searchsorted(cdf, rng.random(n), side="right"), G - 1).astype(np.int64)


def _expected(groups, attrs, G, W):
    order = np.argsort(groups, kind="stable")
    sg = groups[order]
    sv = attrs[order].astype(np.int64)
    K = np.bincount(groups, minlength=G)
    start = np.zeros(G + 1, dtype=np.int64)
    np.cumsum(K, out=start[1:])
    end = start[1:]
    ws = np.maximum(start[:-1], end - W)
    csum = np.zeros(len(sv) + 1, dtype=np.int64)
    np.cumsum(sv, out=csum[1:])
    fill = np.minimum(K, W)
    wsum = csum[end] - csum[ws]
    t = K > 0
    idx = np.empty(2 * int(t.sum()), dtype=np.int64)
    idx[0::2] = ws[t]
    idx[1::2] = end[t]
    mn = np.zeros(G, dtype=np.int64)
    mx = np.zeros(G, dtype=np.int64)
    if len(idx):
        sv_pad = np.append(sv, 0)
        mn[t] = np.minimum.reduceat(sv_pad, idx)[0::2]
        mx[t] = np.maximum.reduceat(sv_pad, idx)[0::2]
    next_pos = np.where(K > W, (K - W) % W, 0)
    return fill, wsum, mn, mx, next_pos, t


@pytest.mark.parametrize("name,G,W,s,split,nb", [
    ("C2", 10_000, 100_000, 1.0, False, 2),
    ("C3", 100_000, 1_000_000, 1.5, True, 2),
])
def test_full_shape_windows(name, G, W, s, split, nb):
    import torch
    from paper_1309_0634_b200.stream_engine import StreamEngine
    B = 1 << 24
    rng = np.random.default_rng(17)
    eng = StreamEngine(G, W, n_partitions=148, aggregates=("count", "sum", "avg", "min", "max"),
                       max_batch=B, initial="hash")
    bal = StreamEngine.balancer_struct("prob", B // 1480, 0.5, split=split)
    gs, avs = [], []
    for i in range(nb):
        g = _zipf(B, G, s, rng)
        a = rng.integers(-2 ** 31, 2 ** 31, B, dtype=np.int64)
        rep = eng.step(torch.from_numpy(g.astype(np.int32)).cuda(), torch.from_numpy(a.astype(np.int32)).cuda(), bal)
        assert rep.tuples == B
        gs.append(g)
        avs.append(a)
    fill, wsum, mn, mx, nxt, t = _expected(np.concatenate(gs), np.concatenate(avs), G, W)
    snap = eng.snapshot()
    assert np.array_equal(snap["fill"], fill)
    assert np.array_equal(snap["next_pos"], nxt)
    assert np.array_equal(snap["window_sum"], wsum)
    assert np.array_equal(snap["min"][t], mn[t]) and np.array_equal(snap["max"][t], mx[t])
    eng.close()


def test_full_shape_int64_keys_c4():
    """C4 shape: G = 1M, W = 1e7, int64 keys, MIN/MAX/SUM, batch 2^24."""
    import torch
    from paper_1309_0634_b200.stream_engine import StreamEngine
    G, W, B = 1_000_000, 10_000_000, 1 << 24
    rng = np.random.default_rng(23)
    ids = _zipf(B, G, 1.0, rng)
    a = rng.integers(-2 ** 31, 2 ** 31, B, dtype=np.int64)
    eng = StreamEngine(G, W, n_partitions=148, aggregates=("count", "sum", "min", "max"), max_batch=B,
                       key_bits=64, initial="hash")
    bal = StreamEngine.balancer_struct("prob", B // 1480, 0.5, split=True)
    eng.step(torch.from_numpy(D.mix64(ids)).cuda(), torch.from_numpy(a.astype(np.int32)).cuda(), bal)
    fill, wsum, mn, mx, nxt, t = _expected(ids, a, G, W)
    slot_ids = D.unmix64(eng.slot_keys())            # dense slot -> group id
    snap = eng.snapshot()
    n = len(slot_ids)
    assert n == int(t.sum())
    assert np.array_equal(snap["fill"][:n], fill[slot_ids])
    assert np.array_equal(snap["window_sum"][:n], wsum[slot_ids])
    assert np.array_equal(snap["min"][:n], mn[slot_ids]) and np.array_equal(snap["max"][:n], mx[slot_ids])
    eng.close()
