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
    ("C1", 1_000, 1_000, 0.0, False, 3),        # few live chunks: sub-chunk placement
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
        g = _zipf(B, G, s, rng) if s > 0 else rng.integers(0, G, B)
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


def test_c4_twelve_batches_wrap_the_top_window():
    """C4 shape over 12 batches (2^24 each): the top group (~7 % of every
    batch) fills W = 1e7 after ~9 batches and then evicts part of its window
    every batch -- ring wrap, next_pos, retraction and the multi-chunk
    MIN/MAX maintenance all run at W = 1e7.  Checked after the first
    partial eviction and at the end, every touched group, int64 keys."""
    import torch
    from paper_1309_0634_b200.stream_engine import StreamEngine
    G, W, B, NB = 1_000_000, 10_000_000, 1 << 24, 12
    rng = np.random.default_rng(31)
    eng = StreamEngine(G, W, n_partitions=148, aggregates=("count", "sum", "min", "max"), max_batch=B,
                       key_bits=64, initial="hash")
    bal = StreamEngine.balancer_struct("prob", B // 1480, 0.5, split=True)
    ids = np.empty(NB * B, dtype=np.int32)
    vals = np.empty(NB * B, dtype=np.int32)
    wrapped_checked = False
    for i in range(NB):
        g = _zipf(B, G, 1.0, rng)
        a = rng.integers(-2 ** 31, 2 ** 31, B, dtype=np.int64).astype(np.int32)
        ids[i * B:(i + 1) * B] = g
        vals[i * B:(i + 1) * B] = a
        rep = eng.step(torch.from_numpy(D.mix64(g)).cuda(), torch.from_numpy(a).cuda(), bal)
        assert rep.tuples == B
        n_seen = (i + 1) * B
        K0 = int(np.count_nonzero(ids[:n_seen] == 0))
        if (K0 > W and not wrapped_checked) or i == NB - 1:
            fill, wsum, mn, mx, nxt, t = _expected(ids[:n_seen].astype(np.int64), vals[:n_seen], G, W)
            slot_ids = D.unmix64(eng.slot_keys())
            snap = eng.snapshot()
            n = len(slot_ids)
            assert n == int(t.sum())
            assert fill[0] == W and nxt[0] > 0                  # the top window has wrapped
            for k in ("fill", "next_pos", "window_sum", "min", "max"):
                ref = {"fill": fill, "next_pos": nxt, "window_sum": wsum, "min": mn, "max": mx}[k]
                assert np.array_equal(snap[k][:n], ref[slot_ids]), (i, k)
            # the ring of the top group in arrival order: its last W values
            s0 = int(np.flatnonzero(slot_ids == 0)[0])
            last = vals[:n_seen][ids[:n_seen] == 0][-W:]
            assert np.array_equal(eng.contents(s0), last.astype(np.int64))
            wrapped_checked = True
    assert wrapped_checked
    eng.close()


@pytest.mark.parametrize("policy", ["first", "all", "prob", "best"])
@pytest.mark.parametrize("G,W", [(10_000, 100_000), (1_000_000, 10_000_000)])
def test_full_shape_movelists(policy, G, W):
    """C2 and C4 group domains (G = 10K staged in the policy CTA's shared
    memory; G = 1M scanned CTA-wide from global memory), P = 148, B = 2^24:
    the fused step's MoveList and scanned count equal the oracle's policy
    (balance.py:141-293) on the same batch and the assignment in force
    before it, batch after batch."""
    import torch
    from oracle import port as O
    from paper_1309_0634_b200.stream_engine import StreamEngine
    B, P = 1 << 24, 148
    if policy == "prob" and G > 100_000:
        # the oracle's per-tuple segment scan (balance.py:230-264) takes
        # minutes per batch here; the CTA-wide prob_check path is checked
        # against it at G = 20K by test_step_vs_oracle
        pytest.skip("oracle prob_check too slow at G = 1M")
    rng = np.random.default_rng(41)
    eng = StreamEngine(G, W, n_partitions=P, aggregates=("count", "sum"), max_batch=B, initial="contiguous")
    thr = B // (10 * P)
    bal = StreamEngine.balancer_struct(policy, thr, 0.5)
    cfg = O.balancer_cfg(policy, thr, 0.5)
    for i in range(3):
        g = _zipf(B, G, 1.0, rng)
        a = rng.integers(-2 ** 31, 2 ** 31, B, dtype=np.int64)
        g2t, lists = eng.get_lists()
        asg = O.OAssignment(g2t, [list(x) for x in lists])
        rep = eng.step(torch.from_numpy(g.astype(np.int32)).cuda(), torch.from_numpy(a.astype(np.int32)).cuda(), bal)
        counts, tpt = O.histogram(g, asg)
        if policy == "prob":
            rg, _, ind = O.place(g, a, asg, counts, tpt)
        else:                       # these policies read counts / segment lengths only
            rg, ind = None, np.concatenate(([0], np.cumsum(tpt)))
        v = O.POLICY_FNS[policy](counts, tpt, asg, rg, ind, cfg)
        assert eng.last_moves() == [tuple(m) for m in v.moves], i
        assert rep.scanned == v.scanned and rep.moves == len(v.moves)
        assert rep.imbalance == int(tpt.max() - tpt.min())
    eng.close()
