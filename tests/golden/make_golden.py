"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``skewstream`` from /root/reference/pkg/src (read-only; no
bytecode is written there) and records its outputs on seeded inputs into
``tests/golden/*.json``.  Those fixtures pin both the CPU oracle
(oracle/port.py) and, through the GPU parity tests, the CUDA path.  The
GPU box never runs this script; it only reads the committed JSON.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import skewstream as ss  # noqa: E402
from skewstream import engine as ss_engine  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def _dump(name, obj):
    path = os.path.join(HERE, name)
    with open(path, "w") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def _digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.int64).tobytes())
    return h.hexdigest()


def _store_state(store):
    return {
        "fill": store.fill.tolist(),
        "next_pos": store.next_pos.tolist(),
        "window_sum": store.window_sum.tolist(),
        "contents": [store.contents(g).tolist() for g in range(store.n_groups)],
    }


def streams():
    """Stream generators: short streams verbatim, long ones as digests."""
    out = []
    specs = [
        ("uniform", 2000, 37, 1.0, 5),
        ("zipf", 2000, 50, 1.0, 7),
        ("zipf", 2000, 500, 1.5, 11),
        ("pzipf", 2000, 64, 1.2, 13),
        ("uniform", 150_000, 1000, 1.0, 0),
        ("zipf", 150_000, 10_000, 1.0, 3),
        ("zipf", 140_000, 100_000, 1.5, 4),
        ("pzipf", 140_000, 4096, 1.0, 9),
    ]
    for kind, n, g, s, seed in specs:
        spec = ss.DatasetSpec(ss.DatasetKind(kind), n, g, s, seed)
        gs, at = ss.stream_for(spec).arrays()
        rec = {"kind": kind, "n": n, "groups": g, "exponent": s, "seed": seed,
               "digest": _digest(gs, at)}
        if n <= 5000:
            rec["g"] = gs.tolist()
            rec["a"] = at.tolist()
        out.append(rec)
        # batching pins: sizes of each batch and digest of the concatenation
    bt = []
    for bsz in (7, 5000, 65536, 70000):
        spec = ss.DatasetSpec(ss.DatasetKind.ZIPF, 150_000, 300, 1.0, 2)
        sizes, idx = [], []
        hs = hashlib.sha256()
        for b in ss.batches(ss.stream_for(spec), bsz):
            sizes.append(len(b))
            idx.append(b.index)
            hs.update(np.ascontiguousarray(b.groups, np.int64).tobytes())
        bt.append({"batch_size": bsz, "sizes_head": sizes[:5],
                   "n_batches": len(sizes), "last": sizes[-1],
                   "indices_ok": idx == list(range(len(idx))),
                   "digest": hs.hexdigest()})
    perm = np.random.default_rng(77).permutation(40)
    gs, at = ss.relabel_groups(ss.gen_zipf(3000, 40, 1.3, 8), perm).arrays()
    relabel = {"perm": perm.tolist(), "digest": _digest(gs, at)}
    _dump("streams.json", {"streams": out, "batches": bt, "relabel": relabel})


def ingest_cases():
    """Ring-update parity: random groups/attrs with split points."""
    rng = np.random.default_rng(4242)
    cases = []
    for i in range(120):
        g_n = int(rng.integers(1, 12))
        w = int(rng.choice([1, 2, 3, 5, 8, 13, 64]))
        n = int(rng.integers(0, 400))
        groups = rng.integers(0, g_n, size=n).astype(np.int64)
        if i % 3 == 0:
            attrs = rng.integers(-(1 << 31), 1 << 31, size=n, dtype=np.int64)
        else:
            attrs = rng.integers(-50, 50, size=n).astype(np.int64)
        cuts = sorted(rng.integers(0, n + 1, size=int(rng.integers(0, 4))).tolist())
        store = ss.WindowStore(g_n, w)
        sums, lo = [], 0
        snaps = []
        for hi in cuts + [n]:
            s, _ = ss.ingest_sequence(store, groups[lo:hi], attrs[lo:hi],
                                      want_sums=True)
            sums.extend(s.tolist())
            snaps.append({"fill": store.fill.tolist(),
                          "window_sum": store.window_sum.tolist()})
            lo = hi
        cases.append({"n_groups": g_n, "window": w, "groups": groups.tolist(),
                      "attrs": attrs.tolist(), "cuts": cuts, "sums": sums,
                      "snaps": snaps, "final": _store_state(store)})
    # hand vectors restated from the reference unit tests (test_engine.py:45-102)
    hand = []
    for w in (1, 2, 3, 5):
        for n in range(2 * w + 2):
            seq = np.arange(1, n + 1, dtype=np.int64)
            st = ss.WindowStore(1, w)
            ss.ingest_sequence(st, np.zeros(n, dtype=np.int64), seq)
            hand.append({"window": w, "n": n, "final": _store_state(st)})
    st = ss.WindowStore(1, 3)
    for v in (5, 7, 9, 4):
        ss.ingest_tuple(st, 0, v, ss.CostModel())
    evict = _store_state(st)
    _dump("ingest.json", {"cases": cases, "hand": hand, "evict": evict})


def partition_cases():
    rng = np.random.default_rng(2020)
    cases = []
    for _ in range(150):
        p = int(rng.integers(1, 7))
        g_n = int(rng.integers(1, 16))
        owners = rng.integers(0, p, size=g_n)
        lists = [[] for _ in range(p)]
        for g in rng.permutation(g_n):
            lists[int(owners[g])].append(int(g))
        asg = ss.Assignment(owners.astype(np.int64), lists)
        n = int(rng.integers(0, 80))
        groups = rng.integers(0, g_n, size=n).astype(np.int64)
        attrs = rng.integers(-1000, 1000, size=n).astype(np.int64)
        batch = ss.Batch(groups, attrs, 0)
        st = ss.count_batch(batch, asg)
        rb = ss.reorder_batch(batch, asg, st)
        cases.append({"g2t": owners.tolist(), "lists": lists,
                      "groups": groups.tolist(), "attrs": attrs.tolist(),
                      "counts": st.group_counts.tolist(), "tpt": st.tpt.tolist(),
                      "rgroups": rb.groups.tolist(), "rattrs": rb.attrs.tolist(),
                      "indicator": rb.indicator.tolist()})
    init = []
    for g_n, p in ((10, 3), (3, 5), (40000, 1024), (7, 7), (1000, 1184)):
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            a = ss.initial_assignment(g_n, p)
        init.append({"n_groups": g_n, "n_threads": p,
                     "sizes": [len(x) for x in a.thread_to_groups],
                     "digest": _digest(a.group_to_thread)})
    # apply_moves sequences including error cases
    moves_cases = []
    for _ in range(80):
        p = int(rng.integers(2, 6))
        g_n = int(rng.integers(2, 14))
        owners = rng.integers(0, p, size=g_n)
        lists = [[] for _ in range(p)]
        for g in rng.permutation(g_n):
            lists[int(owners[g])].append(int(g))
        asg = ss.Assignment(owners.astype(np.int64), lists)
        mv, cur = [], owners.copy()
        for _ in range(int(rng.integers(0, 8))):
            g = int(rng.integers(0, g_n))
            src = int(cur[g]) if rng.random() > 0.1 else int(rng.integers(0, p))
            dst = int(rng.integers(0, p))
            pl = ss.BACK if rng.random() < 0.5 else ss.FRONT
            mv.append([g, src, dst, pl])
            if src == cur[g]:
                cur[g] = dst
        err = None
        try:
            new = ss.apply_moves(asg, [ss.Move(*m) for m in mv])
            res = {"g2t": new.group_to_thread.tolist(), "lists": new.thread_to_groups}
        except ss.StaleMoveError:
            err, res = "stale", None
        except ss.InvalidConfigError:
            err, res = "config", None
        moves_cases.append({"g2t": owners.tolist(), "lists": lists, "moves": mv,
                            "error": err, "result": res})
    _dump("partition.json", {"cases": cases, "initial": init, "moves": moves_cases})


def _instance(rng, p, g_n, heavy):
    owners = rng.integers(0, p, size=g_n)
    lists = [[] for _ in range(p)]
    for g in rng.permutation(g_n):
        lists[int(owners[g])].append(int(g))
    asg = ss.Assignment(owners.astype(np.int64), lists)
    if heavy:
        w = (np.arange(1, g_n + 1, dtype=np.float64) ** -1.3)
        n = int(rng.integers(50, 3000))
        groups = rng.choice(g_n, size=n, p=w / w.sum()).astype(np.int64)
    else:
        n = int(rng.integers(0, 400))
        groups = rng.integers(0, g_n, size=n).astype(np.int64)
    return asg, groups


def policy_cases():
    rng = np.random.default_rng(3131)
    cases = []
    pols = [p.value for p in ss.Policy]
    for i in range(260):
        p = int(rng.integers(1, 12))
        g_n = int(rng.integers(1, 60))
        asg, groups = _instance(rng, p, g_n, heavy=bool(i % 2))
        batch = ss.Batch(groups, np.arange(len(groups), dtype=np.int64), 0)
        st = ss.count_batch(batch, asg)
        rb = ss.reorder_batch(batch, asg, st)
        thr = int(rng.choice([1, 2, 5, 20, 100]))
        pot = float(rng.choice([0.1, 0.3, 0.5, 0.77, 1.0]))
        mm = None if rng.random() < 0.6 else int(rng.integers(1, 12))
        rec = {"g2t": asg.group_to_thread.tolist(), "lists": asg.thread_to_groups,
               "groups": groups.tolist(), "threshold": thr, "pot": pot,
               "max_moves": mm, "out": {}}
        for pol in pols:
            cfg = ss.BalancerConfig(policy=pol, thread_threshold=thr, pot=pot,
                                    max_moves=mm)
            v = ss.get_policy(pol)(st, asg, rb, cfg)
            rec["out"][pol] = {"moves": [[m.group, m.src, m.dst, m.placement]
                                         for m in v.moves],
                               "scanned": v.scanned_tuples,
                               "final_tpt": v.final_tpt.tolist()}
        cases.append(rec)
    _dump("policies.json", {"cases": cases})


def pipeline_cases():
    """Whole run() loops: final store, per-row counters, final assignment."""
    out = []
    configs = [
        ("zipf", 20_000, 128, 1.0, 2000, 8, 2, 16, 50),
        ("uniform", 12_000, 100, 1.0, 1500, 16, 1, 8, 20),
        ("pzipf", 15_000, 300, 1.2, 1000, 5, 4, 8, 30),
        ("zipf", 18_000, 64, 1.5, 3000, 40, 2, 4, 100),
    ]
    for kind, n, g_n, s, bsz, w, grid, block, thr in configs:
        for pol in [p.value for p in ss.Policy]:
            cfg = ss.RunConfig(
                dataset=ss.DatasetSpec(ss.DatasetKind(kind), n, g_n, s),
                batch_size=bsz, window=w, grid_size=grid, block_size=block,
                balancer=ss.BalancerConfig(policy=pol, thread_threshold=thr, pot=0.5),
                seed=17)
            rep = ss.run(cfg)
            st = rep.store
            out.append({
                "kind": kind, "n": n, "groups": g_n, "exponent": s, "batch": bsz,
                "window": w, "threads": grid * block, "threshold": thr,
                "policy": pol, "seed": 17,
                "rows": [[r.tuples, r.imbalance, r.moves, r.scanned] for r in rep.rows],
                # the sim backend's modelled costs (engine.py:299-321)
                "makespans": [r.makespan for r in rep.rows],
                "per_thread_cost": [r.per_thread_cost.tolist() for r in rep.rows],
                "total_moves": rep.total_moves, "total_scanned": rep.total_scanned,
                "total_makespan": rep.total_makespan, "throughput": rep.throughput,
                "fill": st.fill.tolist(), "next_pos": st.next_pos.tolist(),
                "window_sum": st.window_sum.tolist(),
                "values_digest": _digest(st.values),
                "final_lists": rep.final_assignment.thread_to_groups,
            })
    # serial oracle with trace on a short stream
    spec = ss.DatasetSpec(ss.DatasetKind.ZIPF, 6000, 40, 1.1, 21)
    store, trace = ss_engine.serial_reference(ss.stream_for(spec), 7)
    ser = {"spec": [6000, 40, 1.1, 21], "window": 7,
           "trace_sums": trace.sums.tolist(),
           "window_sum": store.window_sum.tolist(), "fill": store.fill.tolist()}
    _dump("pipeline.json", {"runs": out, "serial": ser})


if __name__ == "__main__":
    streams()
    ingest_cases()
    partition_cases()
    policy_cases()
    pipeline_cases()
