"""Small runs of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck): the single-pass placement, the radix passes, the
look-back-free 7/10-bit passes, the bucketed passes, hot-key split shares,
int64 keys, MIN/MAX chunk summaries, the device trace, stream scope and the
policy kernels.  Each case checks its windows against the numpy identities
so a sanitizer run is also a correctness run.

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py [case ...]
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_fullsize import _expected, _zipf  # noqa: E402
from paper_1309_0634_b200.stream_engine import StreamEngine  # noqa: E402


def run(name, G, W, B, nb, s=1.1, policy="prob", split=False, env=None, keys64=False, trace=False, P=32,
        aggs=("count", "sum", "avg", "min", "max")):
    for k in ("SS_B200_BUCKET", "SS_B200_ONESWEEP", "SS_B200_OS_BITS", "SS_B200_RANK_PLACE", "SS_B200_NO_GRAPHS"):
        os.environ.pop(k, None)
    os.environ.update(env or {})
    rng = np.random.default_rng(G + B)
    eng = StreamEngine(G, W, n_partitions=P, aggregates=aggs, max_batch=B, initial="hash",
                       key_bits=64 if keys64 else 32)
    if trace:
        eng.set_trace(True)
    bal = StreamEngine.balancer_struct(policy, max(1, B // (10 * P)), 0.5, split=split)
    gs, avs = [], []
    for i in range(nb):
        n = B - 7 * i
        g = _zipf(n, G, s, rng) if s > 0 else rng.integers(0, G, n)
        a = rng.integers(-2 ** 31, 2 ** 31, n, dtype=np.int64)
        if keys64:
            k = torch.from_numpy(g.astype(np.int64) * np.int64(0x9E3779B97F4A7C15 - (1 << 64)))
            eng.step(k.cuda(), torch.from_numpy(a.astype(np.int32)).cuda(), bal)
        else:
            eng.step(torch.from_numpy(g.astype(np.int32)).cuda(), torch.from_numpy(a.astype(np.int32)).cuda(), bal)
        gs.append(g)
        avs.append(a)
    snap = eng.snapshot()
    if not keys64:
        fill, wsum, mn, mx, nxt, t = _expected(np.concatenate(gs), np.concatenate(avs), G, W)
        assert np.array_equal(snap["fill"], fill), name
        assert np.array_equal(snap["window_sum"], wsum), name
        assert np.array_equal(snap["min"][t], mn[t]) and np.array_equal(snap["max"][t], mx[t]), name
    eng.close()
    print("ok", name, flush=True)


CASES = {
    "rank_place": lambda: run("rank_place", 4000, 300, 200_000, 3, policy="prob", env={"SS_B200_RANK_PLACE": "1"}),
    "radix": lambda: run("radix", 4000, 300, 200_000, 3, policy="all", env={"SS_B200_RANK_PLACE": "0"}),
    "split": lambda: run("split", 3000, 50_000, 300_000, 3, s=1.3, policy="best", split=True),
    "os7": lambda: run("os7", 40_000, 10_000, 300_000, 3, env={"SS_B200_ONESWEEP": "1", "SS_B200_OS_BITS": "7"}),
    "os10": lambda: run("os10", 300_000, 20_000, 300_000, 3, s=1.0, env={"SS_B200_ONESWEEP": "1", "SS_B200_OS_BITS": "10"}),
    "bucket": lambda: run("bucket", 40_000, 10_000, 300_000, 3, env={"SS_B200_BUCKET": "1"}),
    "keys64": lambda: run("keys64", 50_000, 10_000, 200_000, 3, keys64=True),
    "minmax_sum": lambda: run("minmax_sum", 2000, 140_000, 400_000, 4, s=1.5, policy="no"),
    "trace": lambda: run("trace", 1000, 64, 50_000, 2, policy="no", trace=True),
    "wide_balance": lambda: run("wide_balance", 20_000, 500, 100_000, 3, policy="prob", P=48),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
    print("all cases done")
