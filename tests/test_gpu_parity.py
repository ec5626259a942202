"""CUDA path vs the oracle and the reference's golden fixtures (B200 only).

Every test calls through the C ABI (libss_b200.so via StreamEngine) and
compares against tests/golden/ (produced by the reference itself) or the
CPU oracle (oracle/port.py, pinned by test_oracle.py).  Integer results
must be bit-exact; AVG is the correctly rounded double quotient, also
compared exactly (tolerance 0).
"""

import hashlib

import numpy as np
import pytest

from oracle import port as O
from paper_1309_0634_b200 import datagen as D
from paper_1309_0634_b200.errors import DataError, InvalidConfigError, StaleMoveError

pytestmark = pytest.mark.gpu


def _engine(G, W, P=4, **kw):
    from paper_1309_0634_b200.stream_engine import StreamEngine
    kw.setdefault("max_batch", 1 << 20)
    return StreamEngine(G, W, n_partitions=P, **kw)


def _dense_values(eng, G, W):
    snap = eng.snapshot()
    vals = np.zeros((G, W), dtype=np.int64)
    for g in range(G):
        c = eng.contents(g)
        p = int(snap["next_pos"][g])
        vals[g, (p + np.arange(len(c))) % W] = c
    return vals


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.int64).tobytes())
    return h.hexdigest()


# ---- window update: golden ingest cases (engine.py:185-296) -----------------

@pytest.mark.parametrize("sub_batch", [0, 16384])
def test_ingest_golden(golden, sub_batch):
    data = golden("ingest.json")
    for case in data["cases"]:
        G, W = case["n_groups"], case["window"]
        eng = _engine(G, W, P=3, sub_batch=sub_batch)
        g = np.asarray(case["groups"], dtype=np.int64)
        a = np.asarray(case["attrs"], dtype=np.int64)
        lo = 0
        for snap, hi in zip(case["snaps"], case["cuts"] + [len(g)]):
            eng.ingest(g[lo:hi], a[lo:hi])
            s = eng.snapshot()
            assert s["fill"].tolist() == snap["fill"]
            assert s["window_sum"].tolist() == snap["window_sum"]
            lo = hi
        fin = case["final"]
        s = eng.snapshot()
        assert s["next_pos"].tolist() == fin["next_pos"]
        for gi in range(G):
            assert eng.contents(gi).tolist() == fin["contents"][gi]
        eng.close()


def test_hand_vectors(golden):
    data = golden("ingest.json")
    for h in data["hand"]:
        eng = _engine(1, h["window"], P=1)
        eng.ingest(np.zeros(h["n"], dtype=np.int64), np.arange(1, h["n"] + 1))
        assert eng.contents(0).tolist() == h["final"]["contents"][0]
        assert eng.snapshot()["next_pos"].tolist() == h["final"]["next_pos"]
        eng.close()
    eng = _engine(1, 3, P=1)
    for v in (5, 7, 9, 4):       # test_engine.py:45-56
        eng.ingest(np.array([0]), np.array([v]))
    assert eng.contents(0).tolist() == [7, 9, 4]
    assert eng.snapshot()["window_sum"].tolist() == [20]


# ---- partition step (partition.py:117-203) ------------------------------------

def test_count_and_reorder_golden(golden):
    for c in golden("partition.json")["cases"]:
        lists = c["lists"]
        G, P = len(c["g2t"]), len(lists)
        eng = _engine(G, 4, P=P)
        eng.set_lists(lists)
        counts, tpt = eng.count(np.asarray(c["groups"], dtype=np.int64))
        assert counts.tolist() == c["counts"] and tpt.tolist() == c["tpt"]
        rg, ra, ind = eng.reorder(np.asarray(c["groups"]), np.asarray(c["attrs"]))
        assert rg.tolist() == c["rgroups"]
        assert ra.tolist() == c["rattrs"]
        assert ind.tolist() == c["indicator"]
        eng.close()


def test_apply_moves_golden(golden):
    for c in golden("partition.json")["moves"]:
        lists = c["lists"]
        G, P = len(c["g2t"]), len(lists)
        eng = _engine(G, 4, P=P)
        eng.set_lists(lists)
        mv = [tuple(m) for m in c["moves"]]
        if c["error"] == "stale":
            with pytest.raises(StaleMoveError):
                eng.apply_moves(mv)
        elif c["error"] == "config":
            with pytest.raises(InvalidConfigError):
                eng.apply_moves(mv)
        else:
            eng.apply_moves(mv)
            g2t, new = eng.get_lists()
            assert g2t.tolist() == c["result"]["g2t"]
            assert new == c["result"]["lists"]
        if c["error"]:
            g2t, same = eng.get_lists()
            assert same == lists
        eng.close()


def test_count_data_error_leaves_state():
    eng = _engine(10, 4, P=2)
    eng.ingest(np.array([1, 2, 3]), np.array([5, 6, 7]))
    with pytest.raises(DataError, match="tuple 2 has group 10"):
        eng.count(np.array([0, 1, 10, 3]))
    with pytest.raises(DataError, match="tuple 1 has group"):
        eng.step(np.array([0, 11, 3]), np.array([1, 1, 1]))
    s = eng.snapshot()
    assert s["fill"].tolist() == [0, 1, 1, 1, 0, 0, 0, 0, 0, 0]
    eng.step(np.array([1]), np.array([9]))
    assert eng.snapshot()["window_sum"][1] == 14


# ---- balancer (balance.py) -------------------------------------------------------

def test_policies_golden(golden):
    from paper_1309_0634_b200.stream_engine import StreamEngine
    for c in golden("policies.json")["cases"]:
        lists = c["lists"]
        G, P = len(c["g2t"]), len(lists)
        eng = _engine(G, 4, P=P)
        eng.set_lists(lists)
        groups = np.asarray(c["groups"], dtype=np.int64)
        for pol, exp in c["out"].items():
            bal = StreamEngine.balancer_struct(pol, c["threshold"], c["pot"], c["max_moves"])
            moves, scanned, final = eng.balance(groups, bal)
            assert [list(m) for m in moves] == exp["moves"], pol
            assert scanned == exp["scanned"], pol
            assert final.tolist() == exp["final_tpt"], pol
        eng.close()


# ---- fused step: the harness loop (harness.py:99-117) ------------------------------

def test_pipeline_golden(golden):
    from paper_1309_0634_b200.stream_engine import StreamEngine
    for r in golden("pipeline.json")["runs"]:
        G, W, P = r["groups"], r["window"], r["threads"]
        spec = D.DatasetSpec(D.DatasetKind(r["kind"]), r["n"], G, r["exponent"], r["seed"])
        eng = _engine(G, W, P=P, sub_batch=16384)
        bal = StreamEngine.balancer_struct(r["policy"], r["threshold"], 0.5)
        rows = []
        for b in D.batches(D.stream_for(spec), r["batch"]):
            rep = eng.step(b.groups, b.attrs, bal)
            rows.append([rep.tuples, rep.imbalance, rep.moves_applied_before, rep.scanned])
        assert rows == r["rows"], r["policy"]
        s = eng.snapshot()
        assert s["fill"].tolist() == r["fill"]
        assert s["next_pos"].tolist() == r["next_pos"]
        assert s["window_sum"].tolist() == r["window_sum"]
        assert _digest(_dense_values(eng, G, W)) == r["values_digest"]
        _, lists = eng.get_lists()
        assert lists == r["final_lists"]
        eng.close()


@pytest.mark.parametrize("policy", ["no", "first", "all", "prob", "best", "shift", "shiftlocal"])
@pytest.mark.parametrize("G,W,P,B,sub", [(1000, 1000, 148, 1 << 17, 1 << 15),
                                         (10_000, 300, 64, 50_000, 16384),
                                         (5000, 7, 37, 30_000, 0),
                                         (20_000, 500, 48, 40_000, 0)])
def test_step_vs_oracle(policy, G, W, P, B, sub):
    """Multi-sub-batch, single-pass and one-/two-pass radix placement, every
    policy (G > 2^14: the policy CTA reads the lists from global memory)."""
    from paper_1309_0634_b200.stream_engine import StreamEngine
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, 4 * B, G, 1.1, 23)
    eng = _engine(G, W, P=P, sub_batch=sub, aggregates=("count", "sum", "avg", "min", "max"),
                  max_batch=B)
    thr = max(1, B // (10 * P))
    bal = StreamEngine.balancer_struct(policy, thr, 0.5)
    cfg = O.balancer_cfg(policy, thr, 0.5)
    store, asg = O.OStore(G, W), O.contiguous_assignment(G, P)
    for b in D.batches(D.stream_for(spec), B):
        rep = eng.step(b.groups, b.attrs, bal)
        counts, tpt = O.histogram(b.groups, asg)
        rg, ra, ind = O.place(b.groups, b.attrs, asg, counts, tpt)
        v = O.POLICY_FNS[policy](counts, tpt, asg, rg, ind, cfg)
        store.ingest(rg, ra, assume_grouped=True)
        assert rep.moves == len(v.moves) and rep.scanned == v.scanned
        assert rep.imbalance == int(tpt.max() - tpt.min())
        assert eng.last_moves() == [tuple(m) for m in v.moves]
        res = eng.results()
        touched = np.flatnonzero(counts)
        assert res.groups.tolist() == touched.tolist()
        cnt, sm, avg, mn, mx = store.aggregates(touched)
        assert np.array_equal(res.count, cnt) and np.array_equal(res.sum, sm)
        assert np.array_equal(res.avg, avg)
        assert np.array_equal(res.min, mn) and np.array_equal(res.max, mx)
        asg = O.apply_move_list(asg, v.moves)
    s = eng.snapshot()
    assert np.array_equal(s["fill"], store.fill)
    assert np.array_equal(s["next_pos"], store.next_pos)
    assert np.array_equal(s["window_sum"], store.window_sum)
    _, lists = eng.get_lists()
    assert lists == asg.lists
    for gi in (0, 1, G // 2, G - 1):
        assert eng.contents(gi).tolist() == store.contents(gi).tolist()
    eng.close()


@pytest.mark.parametrize("W", [1, 5, 64])
def test_sparse_store_matches_oracle(W):
    """Occupancy-proportional rings (capacity doubling up to W)."""
    G, B = 3000, 20_000
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, 6 * B, G, 1.3, 5)
    eng = _engine(G, W, P=16, pool_values=4 * G * W + 1_000_000, max_batch=B,
                  aggregates=("count", "sum", "avg", "min", "max"))
    store = O.OStore(G, W, dense_limit=0)
    for b in D.batches(D.stream_for(spec), B):
        eng.step(b.groups, b.attrs)
        store.ingest(b.groups, b.attrs)
    s = eng.snapshot()
    cnt, sm, avg, mn, mx = store.aggregates()
    assert np.array_equal(s["fill"], cnt) and np.array_equal(s["window_sum"], sm)
    assert np.array_equal(s["min"], mn) and np.array_equal(s["max"], mx)
    for gi in range(0, G, 97):
        assert eng.contents(gi).tolist() == store.contents(gi).tolist()
    eng.close()


def test_large_batch_properties():
    """Full-size C1 batch (2^24): conservation and window identities."""
    G, W, B = 1000, 1000, 1000 * 16384
    g, a = D.gen_uniform(B, G, 3).arrays()
    eng = _engine(G, W, P=148, max_batch=1 << 24)
    eng.step(g, a)
    s = eng.snapshot()
    # every group received B/G >= W values: full windows of the last W values
    assert (s["fill"] == W).all()
    gg = g.reshape(-1, G)           # round-robin: tuple i has group i % G
    tail = a.reshape(-1, G)[-W:]
    assert np.array_equal(s["window_sum"], tail.sum(axis=0))
    assert (gg[0] == np.arange(G)).all()
    eng.close()


# ---- hot-key splitting across blocks + final combine (new mechanism) -------------

@pytest.mark.parametrize("W", [50, 20_000])
@pytest.mark.parametrize("policy", ["no", "first", "all", "prob", "best", "shift", "shiftlocal"])
def test_split_aggregates_match_oracle(policy, W):
    """Aggregates are assignment-independent, so split
    execution must leave the windows bit-identical to the oracle.  The plan
    balances values to store, min(count, W): with W = 50 no group stores more
    than half a block's mean (nothing is split; the windows still wrap and
    evict every batch), with W = 20 000 every count is stored and the top
    groups are split."""
    from paper_1309_0634_b200.stream_engine import StreamEngine
    G, P, B = 2000, 64, 50_000
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, 8 * B, G, 1.5, 3)
    eng = _engine(G, W, P=P, sub_batch=16384, max_batch=B,
                  aggregates=("count", "sum", "avg", "min", "max"))
    bal = StreamEngine.balancer_struct(policy, max(1, B // (10 * P)), 0.5, split=True)
    store = O.OStore(G, W)
    ratios = []
    for b in D.batches(D.stream_for(spec), B):
        rep = eng.step(b.groups, b.attrs, bal)
        ratios.append(rep.load_ratio)
        store.ingest(b.groups, b.attrs)
        loads = eng.last_loads()
        # with a split plan the block loads are values to store, min(count, W)
        assert loads.sum() == np.minimum(np.bincount(b.groups, minlength=G), W).sum()
        res = eng.results()
        cnt, sm, avg, mn, mx = store.aggregates(res.groups)
        assert np.array_equal(res.count, cnt) and np.array_equal(res.sum, sm)
        assert np.array_equal(res.avg, avg)
        assert np.array_equal(res.min, mn) and np.array_equal(res.max, mx)
    s = eng.snapshot()
    assert np.array_equal(s["fill"], store.fill)
    assert np.array_equal(s["next_pos"], store.next_pos)
    assert np.array_equal(s["window_sum"], store.window_sum)
    for gi in (0, 1, 2, 5, 100, G - 1):
        assert eng.contents(gi).tolist() == store.contents(gi).tolist()
    # without splitting the floor is P x top share ~ 24; with it, near 1
    # (policy 'no' never moves cold groups, so only the hot part is levelled)
    if W < B:
        pass                            # block loads are capped values, nothing to split
    elif policy in ("shift", "shiftlocal"):
        # neighbour cascades move one group per adjacent pair and round
        # (balance.py:296-385): the ratio falls batch by batch
        counts, tpt = O.histogram(b.groups, O.contiguous_assignment(G, P))
        assert ratios[-1] < ratios[0] and max(ratios) < tpt.max() / (len(b) / P) / 4, ratios
    elif policy != "no":
        assert min(ratios[2:]) <= 1.3, ratios
    else:
        # the plan is built from each batch's own counts, so every batch is
        # split; without splitting the top group alone sets the ratio
        counts, tpt = O.histogram(b.groups, O.contiguous_assignment(G, P))
        unsplit = tpt.max() / (len(b) / P)
        assert max(ratios) < unsplit / 4, (ratios, unsplit)
    eng.close()


# ---- int64 keys (C4 shape): hash table, slots in first-appearance order --------

def _first_appearance_ids(stream_batches, G):
    seen = np.full(G, -1, dtype=np.int64)
    nxt = 0
    for g in stream_batches:
        u, idx = np.unique(g, return_index=True)
        for x in u[np.argsort(idx)]:
            if seen[x] < 0:
                seen[x] = nxt
                nxt += 1
    return seen


@pytest.mark.parametrize("policy", ["no", "prob"])
def test_int64_keys_match_oracle(policy):
    from paper_1309_0634_b200.stream_engine import StreamEngine
    G, W, P, B = 5000, 30, 32, 40_000
    spec = D.DatasetSpec(D.DatasetKind.PERMUTED_ZIPF, 5 * B, G, 1.1, 9)
    bl = list(D.batches(D.stream_for(spec), B))
    slot_of = _first_appearance_ids([b.groups for b in bl], G)
    eng = _engine(G, W, P=P, key_bits=64, max_batch=B, sub_batch=16384,
                  aggregates=("count", "sum", "avg", "min", "max"))
    thr = max(1, B // (10 * P))
    bal = StreamEngine.balancer_struct(policy, thr, 0.5)
    cfg = O.balancer_cfg(policy, thr, 0.5)
    n_seen = int((slot_of >= 0).sum())
    store, asg = O.OStore(G, W), O.contiguous_assignment(G, P)
    for b in bl:
        keys = D.mix64(b.groups)
        rep = eng.step(keys, b.attrs, bal)
        rg = slot_of[b.groups]
        counts, tpt = O.histogram(rg, asg)
        pg, pa, ind = O.place(rg, b.attrs, asg, counts, tpt)
        v = O.POLICY_FNS[policy](counts, tpt, asg, pg, ind, cfg)
        store.ingest(pg, pa, assume_grouped=True)
        asg = O.apply_move_list(asg, v.moves)
        assert rep.moves == len(v.moves) and rep.scanned == v.scanned
    sk = eng.slot_keys()
    assert len(sk) == n_seen
    inv = np.empty(n_seen, dtype=np.int64)
    inv[slot_of[slot_of >= 0]] = np.flatnonzero(slot_of >= 0)
    assert np.array_equal(D.unmix64(sk), inv)
    s = eng.snapshot()
    assert np.array_equal(s["fill"], store.fill) and np.array_equal(s["window_sum"], store.window_sum)
    assert np.array_equal(s["next_pos"], store.next_pos)
    cnt, sm, avg, mn, mx = store.aggregates()
    assert np.array_equal(s["min"], mn) and np.array_equal(s["max"], mx)
    with pytest.raises(DataError):
        eng.step(D.mix64(np.arange(G, 2 * G + 100)), np.zeros(G + 100, dtype=np.int64), bal)
    # the rejected batch claimed nothing (validate before mutate,
    # engine.py:281-282): same slots, same windows, and the next batch lands
    # exactly as on an engine that never saw it
    assert np.array_equal(eng.slot_keys(), sk)
    s2 = eng.snapshot()
    assert np.array_equal(s2["window_sum"], s["window_sum"]) and np.array_equal(s2["fill"], s["fill"])
    b = bl[0]
    eng.step(D.mix64(b.groups), b.attrs, bal)
    rg = slot_of[b.groups]
    counts, tpt = O.histogram(rg, asg)
    pg, pa, ind = O.place(rg, b.attrs, asg, counts, tpt)
    store.ingest(pg, pa, assume_grouped=True)
    s3 = eng.snapshot()
    assert np.array_equal(s3["fill"], store.fill) and np.array_equal(s3["window_sum"], store.window_sum)
    eng.close()


@pytest.mark.parametrize("ready", [True, False])
def test_int64_keys_pipelined_probe(ready):
    """Large G: the key probe + count of batch t+1 runs on its own stream
    while batch t finishes (alternating slot buffers and count rows).  Device
    inputs declared ready overlap; the rest wait.  Unsynchronised steps, one
    host-input batch in the middle, windows checked against the oracle."""
    import torch
    from paper_1309_0634_b200.stream_engine import StreamEngine
    G, W, P, B = 20_000, 100, 64, 200_000
    spec = D.DatasetSpec(D.DatasetKind.PERMUTED_ZIPF, 6 * B, G, 1.1, 5)
    bl = list(D.batches(D.stream_for(spec), B))
    slot_of = _first_appearance_ids([b.groups for b in bl], G)
    eng = _engine(G, W, P=P, key_bits=64, max_batch=B, aggregates=("count", "sum", "avg", "min", "max"))
    eng.set_key_pipeline(ready)
    bal = StreamEngine.balancer_struct("prob", max(1, B // (10 * P)), 0.5, split=True)
    dev = [(torch.as_tensor(D.mix64(b.groups)).cuda(), torch.as_tensor(b.attrs.astype(np.int32)).cuda()) for b in bl]
    torch.cuda.synchronize()
    for i, b in enumerate(bl):
        if i == 3:
            eng.step(D.mix64(b.groups), b.attrs, bal, sync=False)       # host input
        else:
            eng.step(*dev[i], bal, sync=False)
    store = O.OStore(G, W)
    for b in bl:
        store.ingest(slot_of[b.groups], b.attrs)
    s = eng.snapshot()
    n = int((slot_of >= 0).sum())
    assert np.array_equal(s["fill"][:n], store.fill[:n]) and np.array_equal(s["window_sum"][:n], store.window_sum[:n])
    assert np.array_equal(s["next_pos"][:n], store.next_pos[:n])
    cnt, sm, avg, mn, mx = store.aggregates()
    assert np.array_equal(s["min"][:n], mn[:n]) and np.array_equal(s["max"][:n], mx[:n])
    eng.close()


@pytest.mark.parametrize("policy", ["prob", "no"])
@pytest.mark.parametrize("G", [1000, 20_000])
@pytest.mark.parametrize("ready", [True, False])
def test_u32_pipelined_count(ready, G, policy):
    """The count of batch t+1 runs on its own stream while batch t finishes
    (alternating count rows; captured graphs keyed by them; large G: after
    the previous batch's hot-group cache).
    Unsynchronised device batches, a host batch and a replay-record batch
    (split on the engine stream, so never overlapped), checked against the
    oracle."""
    import torch
    from paper_1309_0634_b200.stream_engine import StreamEngine
    W, P, B = 100, 32, 300_000
    spec = D.DatasetSpec(D.DatasetKind.ZIPF, 8 * B, G, 1.1, 21)
    bl = list(D.batches(D.stream_for(spec), B))
    eng = _engine(G, W, P=P, max_batch=B, aggregates=("count", "sum", "avg", "min", "max"))
    eng.set_key_pipeline(ready)
    # policy 'no' with G <= 2^14: statistics, scans and sub-chunk prefixes
    # run ahead on the count stream as well (alternating per-batch arrays)
    bal = StreamEngine.balancer_struct(policy, max(1, B // (10 * P)), 0.5)
    dev = [(torch.as_tensor(b.groups.astype(np.int32)).cuda(), torch.as_tensor(b.attrs.astype(np.int32)).cuda())
           for b in bl]
    torch.cuda.synchronize()
    for i, b in enumerate(bl):
        if i == 3:
            eng.step(b.groups, b.attrs, bal, sync=False)                 # host input
        elif i == 5:
            rec = np.empty(len(b), dtype=D.REPLAY_DTYPE)
            rec["group"], rec["attr"] = b.groups, b.attrs
            eng.step_records(torch.as_tensor(rec.view(np.int64)).cuda(), bal, sync=False)
        else:
            eng.step(*dev[i], bal, sync=False)
    store = O.OStore(G, W)
    for b in bl:
        store.ingest(b.groups, b.attrs)
    s = eng.snapshot()
    assert np.array_equal(s["fill"], store.fill) and np.array_equal(s["window_sum"], store.window_sum)
    assert np.array_equal(s["next_pos"], store.next_pos)
    cnt, sm, avg, mn, mx = store.aggregates()
    assert np.array_equal(s["min"], mn) and np.array_equal(s["max"], mx)
    eng.close()
