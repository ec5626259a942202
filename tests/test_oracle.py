"""Pin the CPU oracle (oracle/port.py) to the reference's own outputs.

Every fixture under tests/golden/ was produced by running the reference
package (tests/golden/make_golden.py).  If these pass, the oracle is a
faithful restatement and can check the CUDA path.
"""

import hashlib

import numpy as np
import pytest

from oracle import port as O
from paper_1309_0634_b200 import datagen as D


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.int64).tobytes())
    return h.hexdigest()


def _asg(g2t, lists):
    return O.OAssignment(np.asarray(g2t, dtype=np.int64), [list(x) for x in lists])


def test_ingest_cases(golden):
    data = golden("ingest.json")
    for case in data["cases"]:
        st = O.OStore(case["n_groups"], case["window"])
        g = np.asarray(case["groups"], dtype=np.int64)
        a = np.asarray(case["attrs"], dtype=np.int64)
        sums, lo = [], 0
        for snap, hi in zip(case["snaps"], case["cuts"] + [len(g)]):
            s = st.ingest(g[lo:hi], a[lo:hi], want_sums=True)
            sums.extend(s.tolist())
            assert st.fill.tolist() == snap["fill"]
            assert st.window_sum.tolist() == snap["window_sum"]
            lo = hi
        fin = case["final"]
        assert sums == case["sums"]
        assert st.fill.tolist() == fin["fill"]
        assert st.next_pos.tolist() == fin["next_pos"]
        assert st.window_sum.tolist() == fin["window_sum"]
        for gi in range(case["n_groups"]):
            assert st.contents(gi).tolist() == fin["contents"][gi]


def test_ingest_sparse_store_matches_dense(golden):
    # the occupancy-proportional store must be indistinguishable
    for case in golden("ingest.json")["cases"][:60]:
        st = O.OStore(case["n_groups"], case["window"], dense_limit=0)
        st.ingest(np.asarray(case["groups"]), np.asarray(case["attrs"]))
        fin = case["final"]
        assert st.window_sum.tolist() == fin["window_sum"]
        for gi in range(case["n_groups"]):
            assert st.contents(gi).tolist() == fin["contents"][gi]


def test_hand_vectors(golden):
    data = golden("ingest.json")
    for h in data["hand"]:
        st = O.OStore(1, h["window"])
        st.ingest(np.zeros(h["n"], dtype=np.int64), np.arange(1, h["n"] + 1))
        assert st.contents(0).tolist() == h["final"]["contents"][0]
        assert st.next_pos.tolist() == h["final"]["next_pos"]
    ev = data["evict"]
    st = O.OStore(1, 3)
    for v in (5, 7, 9, 4):
        st.ingest([0], [v])
    assert st.contents(0).tolist() == ev["contents"][0] == [7, 9, 4]
    assert st.window_sum.tolist() == ev["window_sum"] == [20]


def test_count_and_place(golden):
    for c in golden("partition.json")["cases"]:
        asg = _asg(c["g2t"], c["lists"])
        counts, tpt = O.histogram(np.asarray(c["groups"], dtype=np.int64), asg)
        assert counts.tolist() == c["counts"] and tpt.tolist() == c["tpt"]
        rg, ra, ind = O.place(np.asarray(c["groups"]), np.asarray(c["attrs"]),
                              asg, counts, tpt)
        assert rg.tolist() == c["rgroups"]
        assert ra.tolist() == c["rattrs"]
        assert ind.tolist() == c["indicator"]


def test_initial_assignment(golden):
    for c in golden("partition.json")["initial"]:
        a = O.contiguous_assignment(c["n_groups"], c["n_threads"])
        assert [len(x) for x in a.lists] == c["sizes"]
        assert _digest(a.g2t) == c["digest"]


def test_apply_moves(golden):
    for c in golden("partition.json")["moves"]:
        asg = _asg(c["g2t"], c["lists"])
        before = (asg.g2t.copy(), [list(x) for x in asg.lists])
        mv = [tuple(m) for m in c["moves"]]
        if c["error"] == "stale":
            with pytest.raises(O.OracleStaleMoveError):
                O.apply_move_list(asg, mv)
        elif c["error"] == "config":
            with pytest.raises(O.OracleConfigError):
                O.apply_move_list(asg, mv)
        else:
            new = O.apply_move_list(asg, mv)
            assert new.g2t.tolist() == c["result"]["g2t"]
            assert new.lists == c["result"]["lists"]
        assert asg.g2t.tolist() == before[0].tolist() and asg.lists == before[1]


def test_policies(golden):
    for c in golden("policies.json")["cases"]:
        asg = _asg(c["g2t"], c["lists"])
        groups = np.asarray(c["groups"], dtype=np.int64)
        counts, tpt = O.histogram(groups, asg)
        rg, _, ind = O.place(groups, np.zeros(len(groups), np.int64), asg, counts, tpt)
        for pol, exp in c["out"].items():
            cfg = O.balancer_cfg(pol, c["threshold"], c["pot"], c["max_moves"])
            v = O.POLICY_FNS[pol](counts, tpt, asg, rg, ind, cfg)
            assert [list(m) for m in v.moves] == exp["moves"], pol
            assert v.scanned == exp["scanned"], pol
            assert v.final_tpt.tolist() == exp["final_tpt"], pol


def test_pipeline_runs(golden):
    data = golden("pipeline.json")
    for r in data["runs"]:
        spec = D.DatasetSpec(D.DatasetKind(r["kind"]), r["n"], r["groups"],
                             r["exponent"], r["seed"])
        it = ((b.groups, b.attrs) for b in D.batches(D.stream_for(spec), r["batch"]))
        cfg = O.balancer_cfg(r["policy"], r["threshold"], 0.5)
        store, asg, rows = O.run_batches(it, r["groups"], r["window"], r["threads"], cfg)
        got = [[x.tuples, x.imbalance, x.moves_applied_before, x.scanned] for x in rows]
        assert got == r["rows"], r["policy"]
        assert sum(len(x.moves) for x in rows) == r["total_moves"]
        assert store.fill.tolist() == r["fill"]
        assert store.next_pos.tolist() == r["next_pos"]
        assert store.window_sum.tolist() == r["window_sum"]
        assert _digest(store.pool[: r["groups"] * r["window"]]) == r["values_digest"]
        assert asg.lists == r["final_lists"]


def test_serial_trace(golden):
    s = golden("pipeline.json")["serial"]
    n, g, e, seed = s["spec"]
    gs, at = D.stream_for(D.DatasetSpec(D.DatasetKind.ZIPF, n, g, e, seed)).arrays()
    st = O.OStore(g, s["window"])
    sums = []
    for lo in range(0, n, D.CHUNK):
        sums.extend(st.ingest(gs[lo:lo + D.CHUNK], at[lo:lo + D.CHUNK],
                              want_sums=True).tolist())
    assert sums == s["trace_sums"]
    assert st.window_sum.tolist() == s["window_sum"]


def test_aggregates_from_contents():
    st = O.OStore(3, 4)
    st.ingest([0, 1, 0, 0, 0, 0, 2], [5, -1, 3, 9, -7, 2, 4])
    cnt, sm, avg, mn, mx = st.aggregates()
    assert cnt.tolist() == [4, 1, 1]
    assert sm.tolist() == [3 + 9 - 7 + 2, -1, 4]
    assert mn.tolist() == [-7, -1, 4] and mx.tolist() == [9, -1, 4]
    assert avg[0] == 7 / 4
