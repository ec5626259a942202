"""All balancer instantiations compared on one configuration (BASELINE C4:
"all balancer instantiations compared").  For each policy, with and
without hot-key splitting: tuples/s over `steps` batches after `warmup`
batches (CUDA events, staged batches in HBM), mean/max per-block max/mean
load ratio (the plan's tuple loads), the measured per-partition window
update time max/mean, moves per batch.  Initial map: key hash (as bench.py); the
policies start from it and converge during the warm-up.

    python scripts/compare_policies.py --config c4 --steps 6 --warmup 12
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1309_0634_b200.stream_engine import StreamEngine  # noqa: E402

POLICIES = ("no", "first", "all", "prob", "best", "shift", "shiftlocal")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=12)
    ap.add_argument("--initial", default="hash")
    ap.add_argument("--batch", type=int, default=0)
    args = ap.parse_args()
    desc, kind, s, G, W, B, aggs, _, _ = bench.CONFIGS[args.config]
    B = args.batch or B
    dev = torch.device("cuda", 0)
    batches = bench.make_batches(kind, s, G, B, 2, dev, seed=99)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    for split in (False, True):
        for pol in POLICIES:
            eng = StreamEngine(G, W, n_partitions=148, aggregates=aggs, max_batch=B, initial=args.initial,
                               key_bits=64 if kind.endswith("64") else 32)
            eng.set_stream(stream)
            bal = eng.balancer_struct(pol, max(1, B // 1480), 0.5, split=split)
            for i in range(args.warmup):
                eng.step(*batches[i % 2], bal)
            ratios, moves = [], []
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for i in range(args.steps):
                eng.step(*batches[i % 2], bal, sync=False)
            e1.record(stream)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            part = []
            for i in range(2):
                r = eng.step(*batches[i % 2], bal)
                ratios.append(r.load_ratio)
                moves.append(r.moves)
                ns = eng.last_part_ns().astype(np.float64)
                if ns.sum() > 0:
                    part.append(float(ns.max() / ns.mean()))
            print(json.dumps({"config": args.config, "policy": pol, "split": split, "initial": args.initial,
                              "warmup": args.warmup,
                              "tuples_per_s": B * args.steps / (ms / 1e3),
                              "ms_per_step": ms / args.steps,
                              "load_ratio_mean": float(np.mean(ratios)), "load_ratio_max": float(np.max(ratios)),
                              "moves_per_batch": float(np.mean(moves)),
                              "part_ns_max_over_mean": float(np.mean(part)) if part else None}), flush=True)
            eng.close()


if __name__ == "__main__":
    main()
