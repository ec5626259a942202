"""Both placement paths of the fused step -- the single-pass chunk walk
(k_rank_place, G <= 2^14) and the radix passes -- forced in turn through
SS_B200_RANK_PLACE, at full batch size, with ragged batch lengths and with
heavy dropping of never-stored tuples (W far below the group counts).
Checked exactly against the window identities of test_gpu_fullsize."""

import numpy as np
import pytest

from test_gpu_fullsize import _expected, _zipf

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rank", ["1", "0"])
@pytest.mark.parametrize("G,W,s,B,policy,split", [
    (10_000, 100_000, 1.0, (1 << 24) - 777, "prob", False),     # C2 shape, ragged tail
    (1_000, 1_000, 1.0, 1 << 22, "no", False),                  # most tuples never stored
    (16_384, 50, 1.2, (1 << 20) + 3, "prob", True),             # maximum G, tiny window
    (3, 7, 0.0, 100_003, "no", False),                          # a handful of groups
])
def test_placement_paths(monkeypatch, rank, G, W, s, B, policy, split):
    import torch
    from paper_1309_0634_b200.stream_engine import StreamEngine
    monkeypatch.setenv("SS_B200_RANK_PLACE", rank)
    rng = np.random.default_rng(G + W)
    eng = StreamEngine(G, W, n_partitions=148, aggregates=("count", "sum", "avg", "min", "max"),
                       max_batch=B, initial="hash")
    bal = StreamEngine.balancer_struct(policy, max(1, B // 1480), 0.5, split=split)
    gs, avs = [], []
    for i in range(3):
        n = B - 5 * i
        g = _zipf(n, G, s, rng) if s > 0 else rng.integers(0, G, n)
        a = rng.integers(-2 ** 31, 2 ** 31, n, dtype=np.int64)
        rep = eng.step(torch.from_numpy(g.astype(np.int32)).cuda(), torch.from_numpy(a.astype(np.int32)).cuda(), bal)
        assert rep.tuples == n
        gs.append(g)
        avs.append(a)
    fill, wsum, mn, mx, nxt, t = _expected(np.concatenate(gs), np.concatenate(avs), G, W)
    snap = eng.snapshot()
    assert np.array_equal(snap["fill"], fill)
    assert np.array_equal(snap["next_pos"], nxt)
    assert np.array_equal(snap["window_sum"], wsum)
    assert np.array_equal(snap["min"][t], mn[t]) and np.array_equal(snap["max"][t], mx[t])
    eng.close()


@pytest.mark.parametrize("P", [148, 700])
def test_work_grid_extreme_skew(P):
    """The reassignment policy without splitting under extreme skew (one
    group holds most of the batch): the window update runs on the
    work-proportional CTA grid; windows stay exact over several batches."""
    import torch
    from paper_1309_0634_b200.stream_engine import StreamEngine
    G, W, B = 5000, 200_000, 1 << 21
    rng = np.random.default_rng(P)
    eng = StreamEngine(G, W, n_partitions=P, aggregates=("count", "sum", "avg", "min", "max"),
                       max_batch=B, initial="hash")
    bal = StreamEngine.balancer_struct("prob", max(1, B // (10 * P)), 0.5, split=False)
    gs, avs = [], []
    for i in range(4):
        g = _zipf(B, G, 2.0, rng)
        a = rng.integers(-2 ** 31, 2 ** 31, B, dtype=np.int64)
        eng.step(torch.from_numpy(g.astype(np.int32)).cuda(), torch.from_numpy(a.astype(np.int32)).cuda(), bal)
        gs.append(g)
        avs.append(a)
    fill, wsum, mn, mx, nxt, t = _expected(np.concatenate(gs), np.concatenate(avs), G, W)
    snap = eng.snapshot()
    assert np.array_equal(snap["fill"], fill)
    assert np.array_equal(snap["next_pos"], nxt)
    assert np.array_equal(snap["window_sum"], wsum)
    assert np.array_equal(snap["min"][t], mn[t]) and np.array_equal(snap["max"][t], mx[t])
    eng.close()
