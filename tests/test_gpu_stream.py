"""Streaming use of the engine: host input buffers are
copied on a side stream into alternating staging buffers while the
previous batch computes, and each batch's rows (group + the configured
aggregates) are written into pinned host memory and pulled one batch late.
Results must equal the oracle batch by batch (bit-exact, tolerance 0)."""

import numpy as np
import pytest

from oracle import port as O
from paper_1309_0634_b200 import datagen as D

pytestmark = pytest.mark.gpu


def _check_rows(rows, store, g_expected, aggs, to_group=None):
    """Pulled rows of one batch against the oracle's windows after it."""
    pg = rows.groups
    grp = to_group[pg] if to_group is not None else pg.astype(np.int64)
    o = np.argsort(grp)
    assert np.array_equal(grp[o], g_expected)
    cnt, sm, avg, mn, mx = store.aggregates(g_expected)
    assert np.array_equal(rows.count[o], cnt)
    assert np.array_equal(rows.sum[o], sm)
    if "avg" in aggs:
        assert np.array_equal(rows.avg[o], avg)            # AVG bit-exact
    else:
        assert rows.avg is None
    if "min" in aggs:
        assert np.array_equal(rows.min[o], mn) and np.array_equal(rows.max[o], mx)


@pytest.mark.parametrize("key_bits,aggs", [(32, ("count", "sum", "avg")), (64, ("count", "sum", "avg")),
                                           (64, ("count", "sum", "min", "max")), (32, ("count", "sum"))])
def test_stream_pipeline_matches_oracle(key_bits, aggs):
    import torch
    from paper_1309_0634_b200.stream_engine import StreamEngine
    G, W, P, B = 3000, 700, 16, 150_000
    eng = StreamEngine(G, W, n_partitions=P, aggregates=aggs, max_batch=B, key_bits=key_bits)
    bal = eng.balancer_struct("prob", thread_threshold=B // 160, pot=0.5)
    eng.set_host_emit(True)
    assert eng.pulled_row_bytes() == 4 + 4 + 8 + 8 * ("avg" in aggs) + 8 * ("min" in aggs)
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, 7 * B, G, 1.1, 5)
    batches = list(D.batches(D.stream_for(spec), B))
    to_group = None
    for i, b in enumerate(batches):
        keys = D.mix64(b.groups) if key_bits == 64 else b.groups.astype(np.int32)
        hk = torch.from_numpy(np.ascontiguousarray(keys)).pin_memory()
        ha = torch.from_numpy(b.attrs.astype(np.int32)).pin_memory()
        eng.step(hk, ha, bal, sync=False)            # H2D overlaps the previous batch
        if i > 0:
            rows = eng.results_pull()                # the previous batch's rows
            if key_bits == 64:
                to_group = D.unmix64(eng.slot_keys())   # dense slot -> group
            _check_rows(rows, store, prev_g, aggs, to_group)
        if i == 0:
            store = O.OStore(G, W)
        store.ingest(b.groups, b.attrs)
        prev_g = np.unique(b.groups)
    # (the oracle is one batch ahead of the pulls above: re-check the last)
    rows = eng.results_pull()
    if key_bits == 64:
        to_group = D.unmix64(eng.slot_keys())
    _check_rows(rows, store, prev_g, aggs, to_group)
    eng.close()


def test_pull_reports_a_rejected_batch():
    """A batch with a group id >= G, issued without a report, is raised as
    DataError by the pull of that batch (partition.py:119-126); it and the
    batch issued after it are not applied, and the engine goes on."""
    from paper_1309_0634_b200.errors import DataError
    from paper_1309_0634_b200.stream_engine import StreamEngine
    G, W, B = 500, 50, 20_000
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, 5 * B, G, 1.1, 3)
    bl = list(D.batches(D.stream_for(spec), B))
    eng = StreamEngine(G, W, n_partitions=8, max_batch=B)
    eng.set_host_emit(True)
    store = O.OStore(G, W)
    eng.step(bl[0].groups, bl[0].attrs, sync=False)
    store.ingest(bl[0].groups, bl[0].attrs)
    bad = bl[1].groups.astype(np.uint32).copy()
    bad[777] = G + 5
    eng.step(bad, bl[1].attrs, sync=False)
    eng.results_pull()                                   # batch 0: fine
    eng.step(bl[2].groups, bl[2].attrs, sync=False)      # issued behind the bad batch
    with pytest.raises(DataError, match="tuple 777 has group 505"):
        eng.results_pull()
    s = eng.snapshot()
    assert np.array_equal(s["fill"], store.fill) and np.array_equal(s["window_sum"], store.window_sum)
    eng.step(bl[3].groups, bl[3].attrs, sync=False)
    store.ingest(bl[3].groups, bl[3].attrs)
    _check_rows(eng.results_pull(), store, np.unique(bl[3].groups), ("count", "sum", "avg"))
    eng.close()


def test_pull_requires_an_emitted_batch():
    from paper_1309_0634_b200.errors import InvalidConfigError
    from paper_1309_0634_b200.stream_engine import StreamEngine
    eng = StreamEngine(100, 10, n_partitions=4, max_batch=1 << 16)
    eng.set_host_emit(True)
    with pytest.raises(InvalidConfigError):
        eng.results_pull()
    eng.close()


@pytest.mark.parametrize("split", [False, True])
def test_graph_replay_equals_direct_launches(split):
    """The fused step replayed from cached CUDA graphs (default) and launched
    kernel by kernel give identical state, rows and balancer decisions."""
    import torch
    from paper_1309_0634_b200.stream_engine import StreamEngine
    G, W, P, B = 4000, 900, 24, 120_000
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, 6 * B, G, 1.3, 21)
    bl = list(D.batches(D.stream_for(spec), B))
    dev = [(torch.from_numpy(b.groups.astype(np.int32)).cuda(), torch.from_numpy(b.attrs.astype(np.int32)).cuda())
           for b in bl[:2]]
    engs = []
    for graphs in (True, False):
        e = StreamEngine(G, W, n_partitions=P, aggregates=("count", "sum", "avg", "min", "max"), max_batch=B)
        e.set_graphs(graphs)
        engs.append(e)
    bal = StreamEngine.balancer_struct("prob", B // 240, 0.5, split=split)
    for i in range(8):
        g, a = dev[i % 2]                      # two device batches, reused: graph hits
        reps = [e.step(g, a, bal) for e in engs]
        assert reps[0] == reps[1]
        r0, r1 = engs[0].results(), engs[1].results()
        o0, o1 = np.argsort(r0.groups), np.argsort(r1.groups)
        assert np.array_equal(r0.groups[o0], r1.groups[o1])
        assert np.array_equal(r0.avg[o0], r1.avg[o1])
    s0, s1 = engs[0].snapshot(), engs[1].snapshot()
    for k in ("fill", "next_pos", "window_sum", "min", "max"):
        assert np.array_equal(s0[k], s1[k]), k
    assert engs[0].get_lists() [1] == engs[1].get_lists()[1]
    for e in engs:
        e.close()


def test_replay_file_ingest_matches_oracle(tmp_path):
    """a replay file (the reference's 8-byte record format)
    streamed through pinned double buffers and the device-side record split
    gives the oracle's per-batch rows and final state."""
    from paper_1309_0634_b200.replay import ReplayIngest
    from paper_1309_0634_b200.stream_engine import StreamEngine
    G, W, P, B = 2500, 400, 16, 90_001            # odd batch: exercises the record tail
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, 5 * B + 1234, G, 1.1, 44)
    path = tmp_path / "stream.replay"
    D.write_replay(D.stream_for(spec), path)
    eng = StreamEngine(G, W, n_partitions=P, aggregates=("count", "sum", "avg"), max_batch=B)
    bal = eng.balancer_struct("prob", B // 160, 0.5)
    rows = {}
    ri = ReplayIngest(eng, path, B)
    for _ in ri.batches(bal, on_rows=lambda i, r: rows.__setitem__(i, (r.groups.copy(), r.avg.copy()))):
        pass
    store = O.OStore(G, W)
    for i, b in enumerate(D.batches(D.read_replay(path, G), B)):
        store.ingest(b.groups, b.attrs)
        g = np.unique(b.groups)
        pg, pa = rows[i]
        o = np.argsort(pg)
        assert np.array_equal(pg[o].astype(np.int64), g)
        assert np.array_equal(pa[o], store.aggregates()[2][g])
    s = eng.snapshot()
    assert np.array_equal(s["fill"], store.fill) and np.array_equal(s["window_sum"], store.window_sum)
    eng.close()


def test_replay_file_with_bad_group_raises(tmp_path):
    """A replay record whose group is >= G raises DataError naming the tuple
    (batch-relative index) instead of silently emitting nothing."""
    from paper_1309_0634_b200.errors import DataError
    from paper_1309_0634_b200.replay import ReplayIngest
    from paper_1309_0634_b200.stream_engine import StreamEngine
    G, B = 300, 10_000
    rec = np.zeros(4 * B, dtype=D.REPLAY_DTYPE)
    rng = np.random.default_rng(5)
    rec["group"] = rng.integers(0, G, 4 * B)
    rec["attr"] = rng.integers(-1000, 1000, 4 * B)
    rec["group"][2 * B + 17] = G
    path = tmp_path / "bad.replay"
    rec.tofile(path)
    eng = StreamEngine(G, 40, n_partitions=4, max_batch=B)
    seen = []
    with pytest.raises(DataError, match=f"tuple 17 has group {G}"):
        for _ in ReplayIngest(eng, path, B).batches(on_rows=lambda i, r: seen.append(i)):
            pass
    assert seen == [0, 1]
    eng.close()


def test_device_trace_matches_reference_serial_trace(golden):
    """the device per-tuple trace equals the reference's
    serial_reference trace (tests/golden/pipeline.json, produced by the
    reference) per group, for any batching."""
    import paper_1309_0634_b200 as ss
    ser = golden("pipeline.json")["serial"]
    n, G, s, seed = ser["spec"]
    W = ser["window"]
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, n, G, s, seed)
    groups = np.concatenate([b.groups for b in D.batches(D.stream_for(spec), n)])
    ref_g = groups[np.argsort(groups, kind="stable")]
    ref_s = np.asarray(ser["trace_sums"], dtype=np.int64)[np.argsort(groups, kind="stable")]
    for bsz in (n, 997, 64):
        store, trace = ss.serial_reference(D.stream_for(spec), W, batch_size=bsz)
        pg, ps = trace.grouped_projection()
        assert np.array_equal(pg, ref_g) and np.array_equal(ps, ref_s), bsz
        assert store.window_sum.tolist() == ser["window_sum"] and store.fill.tolist() == ser["fill"]
        store.engine.close()


@pytest.mark.parametrize("rank", ["1", "0"])
@pytest.mark.parametrize("W", [3, 1000])
def test_trace_and_ingest_sequence_sums(monkeypatch, W, rank):
    """Trace mode on the fused step with evictions from the old window and
    from the batch itself; ingest_sequence(want_sums) returns them in input
    order; the windows stay equal to the oracle."""
    import paper_1309_0634_b200 as ss
    from paper_1309_0634_b200.stream_engine import StreamEngine
    monkeypatch.setenv("SS_B200_RANK_PLACE", rank)     # both placement paths
    G, B = 300, 20_000
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, 4 * B, G, 1.2, 8)
    bl = list(D.batches(D.stream_for(spec), B))
    eng = StreamEngine(G, W, n_partitions=8, max_batch=B)
    eng.set_trace(True)
    ref = O.OStore(G, W)
    for b in bl[:3]:
        eng.step(b.groups, b.attrs)
        tg, ts = eng.trace()
        # oracle per-tuple sums: running window sums per group in arrival order
        sums = _oracle_sums(ref, b.groups, b.attrs, W)
        order = np.argsort(b.groups, kind="stable")
        assert np.array_equal(tg, b.groups[order])
        assert np.array_equal(ts, sums[order])
    eng.set_trace(False)
    store = ss.WindowStore(G, W, n_partitions=8, max_batch=B)
    b = bl[3]
    for prev in bl[:3]:
        ss.ingest_sequence(store, prev.groups, prev.attrs)
    sums, _ = ss.ingest_sequence(store, b.groups, b.attrs, want_sums=True)
    assert np.array_equal(sums, _oracle_sums(ref, b.groups, b.attrs, W))
    s = store.engine.snapshot()
    assert np.array_equal(s["window_sum"], ref.window_sum) and np.array_equal(s["fill"], ref.fill)
    store.engine.close()
    eng.close()


def _oracle_sums(store, groups, attrs, W):
    """Per-tuple window sums (input order) by feeding the oracle tuple runs
    one at a time per group position -- the reference's per-tuple semantics
    (engine.py:96-122), vectorised over groups."""
    out = np.empty(len(groups), dtype=np.int64)
    order = np.argsort(groups, kind="stable")
    g_sorted = groups[order]
    starts = np.concatenate(([0], np.flatnonzero(g_sorted[1:] != g_sorted[:-1]) + 1, [len(groups)]))
    for a, b in zip(starts[:-1], starts[1:]):
        g = int(g_sorted[a])
        old = store.contents(g).astype(np.int64)
        run = attrs[order[a:b]].astype(np.int64)
        t = np.concatenate((old, run))
        c = np.concatenate(([0], np.cumsum(t)))
        f0 = len(old)
        idx = f0 + np.arange(1, b - a + 1)
        lo = np.maximum(0, idx - W)
        out[order[a:b]] = c[idx] - c[lo]
    store.ingest(groups, attrs)
    return out


@pytest.mark.parametrize("W,B", [(5000, 2000), (3000, 9000)])
def test_stream_scope_window(W, B):
    """scope='stream' -- COUNT / SUM / AVG / MIN / MAX per group
    over the last W tuples of the whole stream, batch by batch (windows
    smaller and larger than the batch)."""
    from paper_1309_0634_b200.stream_engine import StreamEngine, WindowSpec
    G = 700
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, 7 * B + 321, G, 1.1, 13)
    eng = StreamEngine(G, WindowSpec(W, "stream"), n_partitions=8, max_batch=B,
                       aggregates=("count", "sum", "avg", "min", "max"))
    seen_g, seen_a = [], []
    prev_touched = np.zeros(G, dtype=bool)
    for b in D.batches(D.stream_for(spec), B):
        rep = eng.step(b.groups, b.attrs)
        seen_g.append(b.groups)
        seen_a.append(b.attrs)
        wg = np.concatenate(seen_g)[-W:]
        wa = np.concatenate(seen_a)[-W:].astype(np.int64)
        cnt = np.bincount(wg, minlength=G)
        sm = np.bincount(wg, weights=wa, minlength=G).astype(np.int64)   # exact: |sum| < 2^53
        snap = eng.snapshot()
        assert np.array_equal(snap["fill"], cnt)
        assert np.array_equal(snap["window_sum"], sm)
        res = eng.results()
        for i, g in enumerate(res.groups):
            assert res.count[i] == cnt[g] and res.sum[i] == sm[g]
            if cnt[g]:
                vals = wa[wg == g]
                assert res.min[i] == vals.min() and res.max[i] == vals.max()
                assert res.avg[i] == np.float64(sm[g]) / np.float64(cnt[g])
    with pytest.raises(Exception):
        eng.step(b.groups, b.attrs, StreamEngine.balancer_struct("prob", 100, 0.5))
    eng.close()


def test_stream_scope_rejected_batch_changes_nothing():
    """A stream-scope batch with a bad group (no report requested) leaves the
    ring cursors and window untouched: later batches see the last W valid
    tuples (engine.py:281-282, validate before mutate)."""
    from paper_1309_0634_b200.errors import DataError
    from paper_1309_0634_b200.stream_engine import StreamEngine, WindowSpec
    G, W, B = 200, 3000, 1000
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, 8 * B, G, 1.1, 17)
    bl = list(D.batches(D.stream_for(spec), B))
    eng = StreamEngine(G, WindowSpec(W, "stream"), n_partitions=4, max_batch=B,
                       aggregates=("count", "sum", "min", "max"))
    good_g, good_a = [], []
    for i, b in enumerate(bl):
        if i == 1:                     # not yet full: an early bad batch
            bad = b.groups.astype(np.uint32).copy()
            bad[3] = G
            eng.step(bad, b.attrs, sync=False)
            with pytest.raises(DataError):
                eng.last_report()
            continue
        eng.step(b.groups, b.attrs)
        good_g.append(b.groups)
        good_a.append(b.attrs)
        wg = np.concatenate(good_g)[-W:]
        wa = np.concatenate(good_a)[-W:].astype(np.int64)
        snap = eng.snapshot()
        assert np.array_equal(snap["fill"], np.bincount(wg, minlength=G))
        assert np.array_equal(snap["window_sum"], np.bincount(wg, weights=wa, minlength=G).astype(np.int64))
        res = eng.results()
        for k, g in enumerate(res.groups):
            vals = wa[wg == g]
            if len(vals):
                assert res.min[k] == vals.min() and res.max[k] == vals.max()
    eng.close()
