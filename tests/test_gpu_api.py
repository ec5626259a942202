"""The reference-compatible API (skewstream names) on the CUDA backend.

These read like the reference's own tests (pkg/tests/test_partition.py,
test_balance.py, test_harness.py): same calls, same objects, same
expected values -- the golden fixtures were produced by the reference.
"""

import numpy as np
import pytest

import paper_1309_0634_b200 as ss
from oracle import port as O
from paper_1309_0634_b200 import datagen as D

pytestmark = pytest.mark.gpu


def _asg(c):
    return ss.Assignment(np.asarray(c["g2t"]), [list(x) for x in c["lists"]])


def test_count_reorder_via_reference_api(golden):
    for c in golden("partition.json")["cases"][:60]:
        asg = _asg(c)
        batch = ss.Batch(np.asarray(c["groups"], dtype=np.int64), np.asarray(c["attrs"], dtype=np.int64), 0)
        stats = ss.count_batch(batch, asg)
        assert stats.group_counts.tolist() == c["counts"]
        assert stats.tpt.tolist() == c["tpt"]
        r = ss.reorder_batch(batch, asg, stats)
        assert r.groups.tolist() == c["rgroups"] and r.attrs.tolist() == c["rattrs"]
        assert r.indicator.tolist() == c["indicator"]


def test_reorder_rejects_stale_stats():
    asg = ss.initial_assignment(4, 2)
    batch = ss.Batch(np.array([0, 1, 2]), np.array([1, 2, 3]), 0)
    with pytest.raises(ss.ConsistencyError):
        ss.reorder_batch(batch, asg, ss.BatchStats(np.array([1, 1, 0, 0]), np.array([2, 0])))


def test_count_batch_data_error():
    asg = ss.initial_assignment(4, 2)
    with pytest.raises(ss.DataError, match="tuple 1 has group 9"):
        ss.count_batch(ss.Batch(np.array([0, 9, 1]), np.array([1, 2, 3]), 0), asg)


def test_policies_via_reference_api(golden):
    for c in golden("policies.json")["cases"][:80]:
        asg = _asg(c)
        g = np.asarray(c["groups"], dtype=np.int64)
        batch = ss.Batch(g, np.zeros(len(g), dtype=np.int64), 0)
        stats = ss.count_batch(batch, asg)
        r = ss.reorder_batch(batch, asg, stats)
        for pol, exp in c["out"].items():
            cfg = ss.BalancerConfig(pol, c["threshold"], c["pot"], c["max_moves"])
            v = ss.get_policy(pol)(stats, asg, r, cfg)
            assert [[m.group, m.src, m.dst, m.placement] for m in v.moves] == exp["moves"], pol
            assert v.scanned_tuples == exp["scanned"]
            assert v.final_tpt.tolist() == exp["final_tpt"]
            new = ss.apply_moves(asg, v.moves)
            new.audit()
            assert asg.thread_to_groups == c["lists"]      # input untouched


def test_harness_run_matches_golden_rows(golden):
    for r in golden("pipeline.json")["runs"][:14]:
        spec = ss.DatasetSpec(ss.DatasetKind(r["kind"]), r["n"], r["groups"], r["exponent"], 0)
        cfg = ss.RunConfig(dataset=spec, batch_size=r["batch"], window=r["window"],
                           grid_size=1, block_size=r["threads"], seed=r["seed"],
                           balancer=ss.BalancerConfig(r["policy"], r["threshold"], 0.5))
        rep = ss.run(cfg)
        got = [[x.tuples, x.imbalance, x.moves, x.scanned] for x in rep.rows]
        assert got == r["rows"], r["policy"]
        assert rep.total_moves == r["total_moves"]
        assert rep.store.fill.tolist() == r["fill"]
        assert rep.store.window_sum.tolist() == r["window_sum"]
        assert rep.final_assignment.thread_to_groups == r["final_lists"]
        # the sim backend (the reference's default): modelled costs, bit-exact
        assert [x.makespan for x in rep.rows] == r["makespans"]
        assert [x.per_thread_cost.tolist() for x in rep.rows] == r["per_thread_cost"]
        assert rep.total_makespan == r["total_makespan"] and rep.throughput == r["throughput"]
    # the measured backend: per-partition kernel time in ns, same decisions
    r = golden("pipeline.json")["runs"][3]
    spec = ss.DatasetSpec(ss.DatasetKind(r["kind"]), r["n"], r["groups"], r["exponent"], 0)
    cfg = ss.RunConfig(dataset=spec, batch_size=r["batch"], window=r["window"], grid_size=1,
                       block_size=r["threads"], seed=r["seed"], backend=ss.Backend.CUDA,
                       balancer=ss.BalancerConfig(r["policy"], r["threshold"], 0.5))
    rep = ss.run(cfg)
    assert [[x.tuples, x.imbalance, x.moves, x.scanned] for x in rep.rows] == r["rows"]
    assert rep.total_makespan > 0 and all(x.makespan > 0 for x in rep.rows)


def test_ingest_tuple_scalar_path():
    """ingest_tuple (engine.py:96-122): (window_sum, modelled cost) after each
    insert, equal to the scalar reference semantics."""
    st = ss.WindowStore(2, 3, n_partitions=1)
    m = ss.CostModel(window_passes=2, per_element_cost=3, per_tuple_overhead=1)
    vals, out = [4, -2, 7, 10, 1], []
    for v in vals:
        out.append(ss.ingest_tuple(st, 1, v, m))
    sums = [4, 2, 9, 15, 18]
    fills = [1, 2, 3, 3, 3]
    assert out == [(s_, 1 + 2 * 3 * f) for s_, f in zip(sums, fills)]
    with pytest.raises(ss.DataError):
        ss.ingest_tuple(st, 2, 1, m)
    st.engine.close()


def test_ingest_sequence_and_contents():
    st = ss.WindowStore(3, 4, n_partitions=2)
    ss.ingest_sequence(st, np.array([0, 1, 0, 0, 0, 0, 2]), np.array([5, -1, 3, 9, -7, 2, 4]))
    assert st.fill.tolist() == [4, 1, 1]
    assert st.contents(0).tolist() == [3, 9, -7, 2]
    agg = st.aggregates()
    assert agg["min"].tolist() == [-7, -1, 4] and agg["max"].tolist() == [9, -1, 4]
    assert agg["avg"][0] == 7 / 4
    with pytest.raises(ss.ConsistencyError):
        ss.ingest_sequence(st, np.array([0, 1, 0]), np.array([1, 2, 3]), assume_grouped=True)


def test_process_batch_cuda_matches_process_batch_sim():
    """The CUDA executor slot (engine.py:299-321 signature) on the reference
    pipeline's reordered batches: the store equals the oracle's, the rows'
    tuples / imbalance equal process_batch_sim's, and the per-thread cost is
    measured on the partition that holds each segment's groups."""
    import paper_1309_0634_b200 as ss
    from oracle import port as O
    G, W, P, B = 2000, 300, 16, 40_000
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, 4 * B, G, 1.2, 9)
    store = ss.WindowStore(G, W, n_partitions=P, max_batch=B)
    ref = O.OStore(G, W)
    asg = ss.initial_assignment(G, P)
    oasg = O.contiguous_assignment(G, P)
    cfg = O.balancer_cfg("prob", B // (10 * P), 0.5)
    for b in D.batches(D.stream_for(spec), B):
        stats = ss.count_batch(b, asg)
        r = ss.reorder_batch(b, asg, stats)
        rep = ss.process_batch_cuda(r, store)
        ref.ingest(r.groups, r.attrs, assume_grouped=True)
        tpt = np.diff(r.indicator)
        assert rep.tuples == len(b) and rep.imbalance == int(tpt.max() - tpt.min())
        assert len(rep.per_thread_cost) == P
        assert (rep.per_thread_cost[tpt > 0] > 0).all()
        counts, otpt = O.histogram(b.groups, oasg)
        rg, ra, ind = O.place(b.groups, b.attrs, oasg, counts, otpt)
        v = O.POLICY_FNS["prob"](counts, otpt, oasg, rg, ind, cfg)
        asg = ss.apply_moves(asg, [ss.Move(*m) for m in v.moves])
        oasg = O.apply_move_list(oasg, v.moves)
    s = store.engine.snapshot()
    assert np.array_equal(s["fill"], ref.fill) and np.array_equal(s["window_sum"], ref.window_sum)
    assert np.array_equal(s["next_pos"], ref.next_pos)
    for g in (0, 1, 7, G - 1):
        assert store.contents(g).tolist() == ref.contents(g).tolist()
    # process_batch_sim: the same execution, costs in the reference's model
    # units -- per tuple overhead + passes * elem * min(fill after insert, W)
    m = ss.CostModel(window_passes=3, per_element_cost=2, per_tuple_overhead=5, per_iteration_overhead=7)
    b = next(iter(D.batches(D.stream_for(spec), B)))
    stats = ss.count_batch(b, asg)
    r = ss.reorder_batch(b, asg, stats)
    f0 = store.engine.snapshot()["fill"]
    rep = ss.process_batch_sim(r, store, m)
    rg = np.asarray(r.groups)
    cost = np.empty(len(rg), dtype=np.int64)
    seen = {}
    for i, g in enumerate(rg.tolist()):
        seen[g] = seen.get(g, 0) + 1
        cost[i] = 5 + 3 * 2 * min(int(f0[g]) + seen[g], W)
    c = np.concatenate(([0], np.cumsum(cost)))
    per_thread = c[np.asarray(r.indicator)[1:]] - c[np.asarray(r.indicator)[:-1]]
    assert rep.per_thread_cost.tolist() == per_thread.tolist()
    assert rep.makespan == int(per_thread.max()) + 7
    ref.ingest(r.groups, r.attrs, assume_grouped=True)
    assert np.array_equal(store.engine.snapshot()["window_sum"], ref.window_sum)
    # a split run is refused before anything is ingested
    bad = ss.ReorderedBatch(np.array([1, 2, 1]), np.array([5, 6, 7]), np.array([0] * P + [3]))
    before = store.engine.snapshot()["window_sum"].copy()
    with pytest.raises(ss.ConsistencyError):
        ss.process_batch_cuda(bad, store)
    assert np.array_equal(store.engine.snapshot()["window_sum"], before)
    store.engine.close()


def test_large_partition_count_policies():
    """P = 2048 partitions with G = 16384 groups: the staged policy CTA would
    need more shared memory than it may use, so the global-list variant runs
    (every policy still equal to the oracle)."""
    from oracle import port as O
    from paper_1309_0634_b200.stream_engine import StreamEngine
    G, W, P, B = 16384, 50, 2048, 1 << 18
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, 2 * B, G, 1.1, 3)
    for policy in ("all", "prob", "best"):
        eng = StreamEngine(G, W, n_partitions=P, aggregates=("count", "sum"), max_batch=B)
        thr = max(1, B // (10 * P))
        bal = StreamEngine.balancer_struct(policy, thr, 0.5)
        cfg = O.balancer_cfg(policy, thr, 0.5)
        asg = O.contiguous_assignment(G, P)
        for b in D.batches(D.stream_for(spec), B):
            rep = eng.step(b.groups, b.attrs, bal)
            counts, tpt = O.histogram(b.groups, asg)
            rg, ra, ind = O.place(b.groups, b.attrs, asg, counts, tpt)
            v = O.POLICY_FNS[policy](counts, tpt, asg, rg, ind, cfg)
            assert eng.last_moves() == [tuple(m) for m in v.moves] and rep.scanned == v.scanned
            asg = O.apply_move_list(asg, v.moves)
        eng.close()


def test_sweep_window_passes_and_gpu_csv_columns(tmp_path):
    """The reference's window_passes sweep axis (harness.py:143-156): the SIM
    backend's modelled makespan grows with the passes, no-balance points are
    pinned to 1; the CSV keeps the reference schema and adds the device
    columns (step time, tuples/s, algorithmic GB/s, partition makespan)."""
    import csv
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, 60_000, 500, 1.1, 3)
    base = ss.RunConfig(dataset=spec, batch_size=20_000, window=64, grid_size=1, block_size=16,
                        balancer=ss.BalancerConfig(ss.Policy.NO_BALANCE, 100, 0.5))
    reps = ss.sweep(base, "window_passes", [1, 3])
    assert reps[1].total_makespan > reps[0].total_makespan
    assert all(r.normalized_throughput == 1.0 for r in reps)
    path = tmp_path / "run.csv"
    ss.write_csv(reps[0], path)
    rows = list(csv.reader(open(path)))
    assert tuple(rows[0][:10]) == ("iter", "policy", "grid", "makespan", "imbalance", "moves", "scanned",
                                   "tuples", "throughput", "normalized_throughput")
    hdr = rows[0]
    for r in rows[1:-1]:
        assert float(r[hdr.index("gpu_step_ns")]) > 0
        assert float(r[hdr.index("gpu_tuples_per_s")]) > 0
        assert float(r[hdr.index("gpu_alg_gbs")]) > 0
    assert rows[-1][0] == "total" and float(rows[-1][hdr.index("gpu_tuples_per_s")]) > 0
    with pytest.raises(ss.InvalidConfigError):
        ss.sweep(base, "bogus", [1])
