"""Benchmark: sustained tuples/s of the fused per-batch step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A "step" is one batch of the hot path (harness.run's loop body,
harness.py:99-117): count -> balancer (device, overlapped) -> stable
placement -> per-group window update -> per-batch result emission ->
apply moves.  Default workload = BASELINE.json configs[1] (C2): Zipf
s=1.0 keys over 10K groups, per-group window W=1e5, SUM+COUNT, the
paper's prob_check group-reassignment balancer, batch 2^24 tuples,
P = 148 processing units (one aggregate CTA per SM).

Printed JSON line (rank 0):
  value      whole-job tuples/s with the staged batches already in HBM
  e2e        the same through StreamEngine.step with pinned HOST buffers:
             H2D of each batch and D2H of the emitted per-group AVG rows
             inside the timed region
  roofline   dominant kernel class: algorithmic bytes / its CUDA-event time
  path_roofline  whole step: SURVEY 8(d) algorithmic bytes / step time
  cpu_baseline   the oracle port (oracle/port.py) on the host, bounded sample
--impl reference times that CPU path alone (the reference package is pure
Python/numpy; its algorithm is restated in oracle/port.py).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (description, kind, exponent, G, W, B, aggregates, policy, split)
    "c1": ("C1 uniform keys, 1K groups, W=1000, AVG, static partitioning, no rebalancing",
           "uniform", 1.0, 1000, 1000, 1 << 24, ("count", "sum", "avg"), "no", False),
    "c2": ("C2 Zipf s=1.0, 10K groups, W=1e5, SUM+COUNT, prob_check group reassignment",
           "zipf", 1.0, 10_000, 100_000, 1 << 24, ("count", "sum"), "prob", False),
    "c3": ("C3 Zipf s=1.5, 100K groups, W=1e6, AVG, hot-key splitting across blocks + prob_check for cold groups",
           "zipf", 1.5, 100_000, 1_000_000, 1 << 24, ("count", "sum", "avg"), "prob", True),
    "c2split": ("C2 shape with hot-key splitting on top of prob_check",
                "zipf", 1.0, 10_000, 100_000, 1 << 24, ("count", "sum"), "prob", True),
    "c4": ("C4 1M groups, W=1e7, MIN/MAX/SUM, int64 keys, Zipf s=1.0, prob_check + hot-key split",
           "zipf64", 1.0, 1_000_000, 10_000_000, 1 << 24, ("count", "sum", "min", "max"), "prob", True),
    "c4u": ("C4 uniform twin: 1M groups, W=1e7, MIN/MAX/SUM, int64 keys",
            "uniform64", 1.0, 1_000_000, 10_000_000, 1 << 24, ("count", "sum", "min", "max"), "prob", True),
    "c5": ("C5 Zipf s=1.2 drifting (new hot set every 4 batches), 1M groups, W=1e7, SUM+COUNT+AVG",
           "zipfdrift", 1.2, 1_000_000, 10_000_000, 1 << 24, ("count", "sum", "avg"), "prob", True),
}
MIX = 0x9E3779B97F4A7C15 - (1 << 64)     # odd: key = id * MIX (mod 2^64) is a bijection
P_DEFAULT = 148
DRIFT_EVERY = 4
L2_BYTES = 126 * (1 << 20)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# synthetic input, generated on the device (inverse CDF of the zipf pmf)
# ---------------------------------------------------------------------------
def make_batches(kind, s, G, B, nbuf, device, seed):
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    out = []
    if kind.startswith("zipf"):
        w = torch.arange(1, G + 1, dtype=torch.float64, device=device).pow(-s)
        cdf = torch.cumsum(w, 0)
        cdf /= cdf[-1].clone()
        cdf[-1] = 1.0
    perm = None
    for i in range(nbuf):
        if kind.startswith("zipf"):
            u = torch.rand(B, dtype=torch.float64, device=device, generator=gen)
            g = torch.searchsorted(cdf, u, right=True).clamp_(max=G - 1)
            if kind == "zipfdrift":
                # the hot set moves every DRIFT_EVERY batches: a new seeded
                # relabelling of the groups (relabel_groups, datagen.py:181-192)
                if i % DRIFT_EVERY == 0:
                    perm = torch.randperm(G, device=device, generator=gen)
                g = perm[g]
        else:
            g = (torch.arange(B, device=device, dtype=torch.int64) + i * B) % G
        if kind.endswith("64"):
            g = g.to(torch.int64) * MIX          # int64 keys (wrapping multiply)
        else:
            g = g.to(torch.int32)
        a = torch.randint(-(2 ** 31), 2 ** 31, (B,), device=device, generator=gen,
                          dtype=torch.int64).to(torch.int32)
        out.append((g.contiguous(), a.contiguous()))
    return out


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=5)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU path: the oracle port of the reference pipeline, group-sharded over the
# host cores, bounded sample
# ---------------------------------------------------------------------------
def _cpu_worker(job):
    """One group shard: the reference pipeline (count, place, policy, ingest,
    apply) over the sub-stream of groups g with g % n == r, relabelled to the
    dense local ids g // n.  Batches are generated before the clock starts and
    cycled; returns (tuples, seconds) over `n_batches` batches."""
    cfg_name, r, n, batch, n_batches, seed = job
    from oracle import port as O
    from paper_1309_0634_b200 import datagen as D
    desc, kind, s, G, W, _, aggs, policy, _ = CONFIGS[cfg_name]
    dk = D.DatasetKind.UNIFORM if kind.startswith("uniform") else D.DatasetKind.ZIPF
    nbuf = 4
    spec = D.DatasetSpec(dk, batch * nbuf, G, s, seed)
    Gl = (G - r + n - 1) // n
    Pl = max(1, P_DEFAULT // n)
    staged = []
    for b in D.batches(D.stream_for(spec), batch):
        m = (b.groups % n) == r
        staged.append(((b.groups[m] // n).astype(np.int64), b.attrs[m].astype(np.int64)))
    asg = O.contiguous_assignment(Gl, Pl)
    cfg = O.balancer_cfg(policy, max(1, batch // (10 * P_DEFAULT)), 0.5)
    store = O.OStore(Gl, W)
    fn = O.POLICY_FNS[policy]
    done, t_work = 0, 0.0
    for i in range(n_batches):
        g, a = staged[i % len(staged)]
        t0 = time.perf_counter()
        counts, tpt = O.histogram(g, asg)
        rg, ra, ind = O.place(g, a, asg, counts, tpt)
        v = fn(counts, tpt, asg, rg, ind, cfg)
        store.ingest(rg, ra, assume_grouped=True)
        asg = O.apply_move_list(asg, v.moves)
        t_work += time.perf_counter() - t0
        done += len(g)
    return done, t_work


def cpu_cores():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count() or 1


def cpu_pipeline(cfg_name, seconds=15.0, batch=1 << 20, cores=None):
    """Group-sharded CPU pipeline on `cores` processes.  A calibration batch
    on one shard sizes the run to about `seconds` of wall time; the value is
    all tuples / the slowest shard's busy time."""
    import multiprocessing as mp
    cores = cores or cpu_cores()
    # shards never get fewer than ~1 batch-slice of 64K tuples
    cores = max(1, min(cores, batch // 65536))
    t, s = _cpu_worker((cfg_name, 0, cores, batch, 2, 11))
    per_batch = max(1e-4, s / 2)
    n_batches = int(max(3, min(400, seconds / per_batch)))
    jobs = [(cfg_name, r, cores, batch, n_batches, 11) for r in range(cores)]
    if cores == 1:
        res = [_cpu_worker(jobs[0])]
    else:
        with mp.get_context("fork").Pool(cores) as pool:
            res = pool.map(_cpu_worker, jobs)
    tuples = sum(r[0] for r in res)
    t_max = max(r[1] for r in res)
    return tuples / t_max, {"batches": n_batches, "batch": batch, "tuples": tuples,
                            "seconds": round(t_max, 2), "cores": cores}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args, rank, world):
    if rank != 0:
        return
    name = args.config
    desc = CONFIGS[name][0]
    per_step = max(2.0, args.cpu_seconds / max(1, args.steps))
    vals, info = [], None
    for i in range(args.steps + args.warmup):
        if i < args.warmup:
            # warm-up: one short shard pass (page-in, allocator, imports)
            _cpu_worker((name, 0, 1, 1 << 16, 2, 11))
            continue
        v, info = cpu_pipeline(name, seconds=per_step)
        vals.append(v)
    v = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": "sustained tuples/s (Zipf skew)", "value": v,
        "unit": "tuples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "dtype": "i64", "data": "synthetic (reference generators)",
        "config": {"workload": desc, "batch": 1 << 20, "partitions": P_DEFAULT},
        "cpu_baseline": {"value": v, "unit": "tuples/s", "cores": info["cores"], "kind": "port",
                         "sample": f"{args.steps} steps, each {info['batches']} batches of 2^20 tuples per "
                                   f"group shard on {info['cores']} processes (count, place, policy, ingest, "
                                   f"apply through oracle/port.py) on {cpu_model()}"},
        "e2e": {"value": v, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU path
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--partitions", type=int, default=P_DEFAULT)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--sub-batch", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--initial", default="hash", choices=["hash", "contiguous"],
                    help="initial group->partition map (north star: hash-partitioned groups)")
    args = ap.parse_args()
    # at least 3 warm-up steps (contract), and at least two passes over the
    # staged batches so every (batch, parity) CUDA graph of the fused step is
    # captured before the clock starts; the JSON line reports the number run
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_1309_0634_b200 import _lib as L
    from paper_1309_0634_b200.stream_engine import StreamEngine

    desc, kind, s, G, W, B, aggs, policy, split = CONFIGS[args.config]
    if args.batch:
        B = args.batch
    P = args.partitions
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)          # NCCL routing and the engine share one stream
    thr = max(1, B // (10 * P))
    sharded = None
    if world > 1:
        # key-sharded: each rank's B tuples are its slice of a global batch of
        # world*B; tuples travel to their owner GPU by NCCL all-to-all, and the
        # GPU-level balancer (prob_check on all-reduced counts) moves groups
        # between GPUs (weak scaling: per-rank input fixed)
        from paper_1309_0634_b200.sharded import ShardedEngine
        sharded = ShardedEngine(G, W, n_partitions=P, aggregates=aggs, device=local, max_batch=world * B,
                                sub_batch=args.sub_batch)
        eng = sharded.local
        gbal = eng.balancer_struct("prob", thread_threshold=max(1, B // 10), pot=0.5)
    else:
        eng = StreamEngine(G, W, n_partitions=P, aggregates=aggs, device=local, max_batch=B,
                           sub_batch=args.sub_batch, key_bits=64 if kind.endswith("64") else 32,
                           initial=args.initial)
    eng.set_stream(stream)
    bal = eng.balancer_struct(policy, thread_threshold=thr, pot=0.5, split=split)
    nbuf = 2 * DRIFT_EVERY if kind == "zipfdrift" else 4
    if world > 1 and kind.endswith("64"):
        raise SystemExit("int64 keys are single-GPU in this build (route is u32)")
    batches = make_batches(kind, s, G, B, nbuf, dev, seed=1234 + rank)
    args.warmup = max(args.warmup, 2 * nbuf)
    torch.cuda.synchronize()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def run_steps(k, start=0):
        for i in range(k):
            g, a = batches[(start + i) % nbuf]
            if sharded is not None:
                sharded.step(g, a, bal, gbal)
            else:
                eng.step(g, a, bal, sync=False)

    # the clock sampler (nvidia-smi) takes ~0.3 s to start: it is started
    # before the warm-up so that it samples the timed region without an
    # idle gap in front of it
    clocks = ClockSampler(local)
    clocks.start()
    # warm-up (also converges the balancer from the contiguous assignment)
    for i in range(args.warmup):
        run_steps(1, i)
        eng.last_report()
    lib = L.load()
    import ctypes as C

    # ---- (1) headline: staged batches in HBM -------------------------------
    barrier()
    # up to 0.3 s (at most 32 steps) of further untimed steps, counted in the
    # reported warm-up, so the timed region starts from a loaded GPU (a step
    # cap: with a growing window, e.g. the C4 uniform twin, every batch adds
    # ring storage; with several ranks every rank runs the same count)
    t_end = time.time() + 0.3
    extra = 0
    while extra < 32 and (world > 1 or time.time() < t_end):
        run_steps(1, args.warmup + extra)
        extra += 1
        torch.cuda.synchronize()
    args.warmup += extra
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    lib = L.load()
    lib.ss_launch_count(1)
    ev0.record(stream)
    run_steps(args.steps, args.warmup)
    ev1.record(stream)
    ev1.synchronize()
    launches = int(lib.ss_launch_count(1))
    ms = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    rep = eng.last_report()
    ms_t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = B * args.steps * world / (ms / 1e3)

    # ---- (2) kernel classes with CUDA events + algorithmic bytes --------------
    lib.ss_profile(eng._h, 1)
    kms = (C.c_double * 7)()
    kn = (C.c_int64 * 7)()
    lib.ss_profile_read(eng._h, kms, kn, 1)
    ab = C.c_int64()
    lib.ss_alg_bytes(eng._h, C.byref(ab), 1)
    ratios = []
    barrier()
    for i in range(args.steps):
        run_steps(1, args.warmup + i)
        ratios.append(eng.last_report().load_ratio)
    lib.ss_profile_read(eng._h, kms, kn, 1)
    lib.ss_alg_bytes(eng._h, C.byref(ab), 1)
    lib.ss_profile(eng._h, 0)
    alg_per_step = ab.value / args.steps
    peak, peak_kind = peaks()
    cls_ms = {n: kms[i] / args.steps for i, n in enumerate(L.KERNEL_CLASSES)}
    cls_launch = {n: kn[i] for i, n in enumerate(L.KERNEL_CLASSES)}
    # algorithmic bytes per class and step:
    # the input is read once in the model -- keys by the count, attrs by the
    # placement (its re-read of the keys is implementation overhead) -- and
    # the window update owns the ring and state bytes
    key_bytes = 8 if kind.endswith("64") else 4
    ingest_bytes = alg_per_step - (key_bytes + 4) * B
    cls_bytes = {"count": key_bytes * B, "place": 4 * B, "ingest": ingest_bytes}
    main_cls = max(("count", "place", "ingest"), key=lambda n: cls_ms[n])
    k_ms = cls_ms[main_cls]
    achieved = cls_bytes[main_cls] / (k_ms / 1e3) / 1e9 if k_ms > 0 else 0.0
    step_ms = ms / args.steps
    path_achieved = alg_per_step / (step_ms / 1e3) / 1e9
    # measured DRAM traffic per launch of that kernel class (ncu --set full of
    # this config, committed under profiles/), else null
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as fh:
            tj = json.load(fh)
        if args.config in tj and main_cls in tj[args.config] and B == (1 << 24) and world == 1:
            traffic = tj[args.config][main_cls]["bytes_per_launch"]
    except Exception:
        traffic = None

    # ---- (3) end to end through the public API with host buffers -------------
    e2e_steps = args.e2e_steps or max(4, args.steps // 2)
    hosts = []
    for g, a in batches[:2]:
        hg = torch.empty(B, dtype=g.dtype, pin_memory=True)
        ha = torch.empty(B, dtype=torch.int32, pin_memory=True)
        hg.copy_(g)
        ha.copy_(a)
        hosts.append((hg, ha))
    # streaming use of the public API: batch i+1 is issued
    # (its H2D overlaps batch i's compute) before batch i's rows are pulled
    # from pinned host memory
    eng.set_host_emit(True)

    def e2e_step(i):
        hg, ha = hosts[i % 2]
        if sharded is not None:
            sharded.step(hg, ha, bal, gbal)
        else:
            eng.step(hg, ha, bal, sync=False)

    # warm-up of the streaming path (its second staging buffer is allocated
    # on first use), not timed
    for i in range(2):
        e2e_step(i)
        eng.results_pull()
    d2h = 0
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for i in range(e2e_steps):
        e2e_step(i)
        if i > 0:
            rg, ra = eng.results_pull()
            d2h += len(rg) * 12 + 4
    rg, ra = eng.results_pull()
    d2h += len(rg) * 12 + 4
    e1.record(stream)
    e1.synchronize()
    e2e_wall = time.perf_counter() - t0
    e2e_ms = max(e0.elapsed_time(e1), e2e_wall * 1e3)
    e2e_value = B * e2e_steps * world / (e2e_ms / 1e3)

    # ---- CPU baseline (rank 0, N=1 only) ----------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, info = cpu_pipeline(args.config, seconds=args.cpu_seconds)
        cpu = {"value": v, "unit": "tuples/s", "cores": info["cores"], "kind": "port",
               "sample": f"{info['batches']} batches x 2^20 tuples ({info['seconds']} s busy per shard) of the "
                         f"same stream shape, group-sharded over {info['cores']} processes through "
                         f"oracle/port.py on {cpu_model()}"}

    eng_sub = eng.sub_batch if hasattr(eng, "sub_batch") else args.sub_batch
    if rank == 0:
        line = {
            "metric": "sustained tuples/s (Zipf skew)",
            "value": value, "unit": "tuples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "i32 keys/values, i64 sums",
            "data": f"synthetic {kind} (s={s}) keys generated on device, uniform int32 attrs; "
                    f"{nbuf} staged batches of {B * (12 if kind.endswith('64') else 8) >> 20} MB each (> L2), cycled",
            "config": {"workload": desc, "groups": G, "window": W, "batch": B,
                       "partitions": P, "initial_map": args.initial, "policy": policy + ("+split" if split else ""), "aggregates": list(aggs),
                       "sub_batch": eng_sub, "l2": "inputs larger than L2 (128 MB per batch)",
                       "parallelism": (f"key-sharded x{world}: NCCL all-to-all routing, GPU-level prob_check"
                                       if world > 1 else "single GPU"),
                       "global_batch": B * world},
            "roofline": {"bound": "hbm", "kernel": main_cls, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": "profiles/r1_traffic.json (ncu --set full, dram read+write per launch)"
                                           if traffic is not None else None,
                         "peak_source": peak_kind,
                         "alg_bytes_per_launch": cls_bytes[main_cls] / max(1, cls_launch[main_cls] / args.steps),
                         "ms_per_step": k_ms},
            "path_roofline": {"alg_bytes_per_tuple": alg_per_step / B, "achieved": path_achieved,
                              "peak": peak, "unit": "GB/s", "frac": path_achieved / peak},
            "kernel_ms_per_step": cls_ms,
            "load_ratio": {"last": rep.load_ratio, "mean": float(np.mean(ratios)),
                           "max": float(np.max(ratios))},
            "moves_last_step": rep.moves,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "tuples/s", "h2d_bytes_per_step": (12 if kind.endswith("64") else 8) * B,
                    "d2h_bytes_per_step": d2h // e2e_steps, "steps": e2e_steps},
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if sharded is not None:
        sharded.close()
    else:
        eng.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
