"""Per-partition window-update time across the blocks (the north star's
"tail imbalance across blocks"): after warm-up batches, the distribution of
the measured per-partition K4 time (ns, %globaltimer inside k_ingest, summed
over the partition's CTAs), the per-partition work (values stored), members
and the plan's loads, for a config of bench.py.

    python scripts/partition_times.py c4 [batches]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1309_0634_b200.stream_engine import StreamEngine  # noqa: E402


def dist(x):
    x = np.asarray(x, dtype=np.float64)
    q = np.percentile(x, [0, 10, 50, 90, 100])
    return {"min": q[0], "p10": q[1], "median": q[2], "p90": q[3], "max": q[4],
            "max_over_mean": float(x.max() / x.mean()) if x.mean() > 0 else None}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    nb = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    desc, kind, s, G, W, B, aggs, policy, split = bench.CONFIGS[name]
    dev = torch.device("cuda", 0)
    eng = StreamEngine(G, W, n_partitions=148, aggregates=aggs, max_batch=B, initial="hash",
                       key_bits=64 if kind.endswith("64") else 32)
    bal = eng.balancer_struct(policy, max(1, B // 1480), 0.5, split=split)
    bs = bench.make_batches(kind, s, G, B, 2, dev, 7)
    ratios = []
    for i in range(nb):
        rep = eng.step(*bs[i % 2], bal)
        ns = eng.last_part_ns().astype(np.float64)
        if i >= nb // 2 and ns.sum() > 0:
            ratios.append(float(ns.max() / ns.mean()))
    ns = eng.last_part_ns()
    work = eng.last_part_work()
    _, lists = eng.get_lists()
    sizes = np.array([len(x) for x in lists])
    print(json.dumps({"config": name, "workload": desc, "policy": policy + ("+split" if split else ""),
                      "plan_load_ratio": rep.load_ratio,
                      "part_ns_max_over_mean_last_half": {"mean": float(np.mean(ratios)), "max": float(np.max(ratios))},
                      "part_ns": dist(ns), "part_work": dist(work), "members": dist(sizes)}))
    eng.close()


if __name__ == "__main__":
    main()
