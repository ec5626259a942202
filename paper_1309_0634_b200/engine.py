"""Windowed aggregation, drop-in for the reference ``skewstream.engine``
(engine.py:1-445), executed by the CUDA engine.

``WindowStore`` keeps the reference's observable state (fill, next_pos,
window_sum, per-group ring contents in arrival order) but lives in HBM,
occupancy-proportional when the dense [G, W] layout would not fit.
``ingest_sequence`` and ``process_batch_cuda`` run the device pipeline
(stable placement + closed-form window exchange, csrc/window.cuh).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConsistencyError, DataError, InvalidConfigError


@dataclass(frozen=True)
class CostModel:
    """The reference's modelled per-tuple cost (engine.py:27-48):
    ``overhead + window_passes * per_element_cost * fill_after_insert`` per
    tuple, plus ``per_iteration_overhead`` once per batch.  The device does
    the work; process_batch_sim reports it in these units."""

    window_passes: int = 1
    per_element_cost: int = 1
    per_tuple_overhead: int = 1
    per_iteration_overhead: int = 0

    def __post_init__(self) -> None:
        if self.window_passes < 1:
            raise InvalidConfigError(f"window_passes must be >= 1, got {self.window_passes}")
        bad = [k for k in ("per_element_cost", "per_tuple_overhead", "per_iteration_overhead")
               if getattr(self, k) < 0]
        if bad:
            raise InvalidConfigError(f"{bad[0]} must be >= 0")

    def run_cost(self, f0: np.ndarray, k: np.ndarray, window: int) -> np.ndarray:
        """Closed-form cost of a run of k values entering a window of fill f0:
        sum over j = 1..k of overhead + passes * elem * min(f0 + j, W)."""
        f0 = np.asarray(f0, dtype=np.int64)
        k = np.asarray(k, dtype=np.int64)
        below = np.clip(window - f0, 0, k)              # inserts before the window is full
        filled = below * f0 + below * (below + 1) // 2 + (k - below) * window
        return k * self.per_tuple_overhead + self.window_passes * self.per_element_cost * filled


@dataclass
class AggregateTrace:
    """Per-ingest (group, window_sum) pairs (engine.py:125-145).  The CUDA
    backend records each batch in grouped order (group ids ascending, arrival
    order within a group), so only per-group projections are meaningful --
    exactly what the reference compares (grouped_projection)."""

    groups: np.ndarray
    sums: np.ndarray

    def __len__(self) -> int:
        return len(self.groups)

    def for_group(self, group: int) -> np.ndarray:
        return self.sums[self.groups == group]

    def grouped_projection(self) -> tuple[np.ndarray, np.ndarray]:
        order = np.argsort(self.groups, kind="stable")
        return self.groups[order], self.sums[order]


class TraceBuffer:
    """Accumulates trace chunks across batches (engine.py:148-164)."""

    def __init__(self) -> None:
        self._groups: list = []
        self._sums: list = []

    def append(self, groups, sums) -> None:
        self._groups.append(np.asarray(groups, dtype=np.int64))
        self._sums.append(np.asarray(sums, dtype=np.int64))

    def build(self) -> AggregateTrace:
        if not self._groups:
            e = np.empty(0, dtype=np.int64)
            return AggregateTrace(e, e.copy())
        return AggregateTrace(np.concatenate(self._groups), np.concatenate(self._sums))


@dataclass(frozen=True)
class IterationReport:
    """Execution record of one batch (engine.py:167-176).  On the CUDA
    backend per_thread_cost is the aggregate kernel's per-partition time
    in ns and makespan its maximum."""

    per_thread_cost: np.ndarray
    makespan: int
    tuples: int
    imbalance: int
    moves: int = 0
    scanned: int = 0


class WindowStore:
    """Per-group windows of the last ``window`` values, on the GPU
    (engine.py:51-93).  Aggregates beyond the reference's SUM/COUNT
    (AVG, MIN, MAX) are maintained when requested."""

    def __init__(self, n_groups: int, window: int, n_partitions: int = 148,
                 aggregates=("count", "sum", "avg", "min", "max"), max_batch: int = 1 << 22,
                 **kw):
        from .stream_engine import StreamEngine
        if n_groups < 1:
            raise InvalidConfigError(f"n_groups must be >= 1, got {n_groups}")
        if window < 1:
            raise InvalidConfigError(f"window must be >= 1, got {window}")
        self.n_groups = n_groups
        self.window = window
        self.engine = StreamEngine(n_groups, window, n_partitions=n_partitions,
                                   aggregates=aggregates, max_batch=max_batch, **kw)

    # observable state (host copies)
    @property
    def fill(self) -> np.ndarray:
        return self.engine.snapshot()["fill"]

    @property
    def next_pos(self) -> np.ndarray:
        return self.engine.snapshot()["next_pos"]

    @property
    def window_sum(self) -> np.ndarray:
        return self.engine.snapshot()["window_sum"]

    @property
    def values(self) -> np.ndarray:
        """Dense [G, W] ring image (only for shapes that fit on the host)."""
        if self.n_groups * self.window > (1 << 27):
            raise InvalidConfigError("dense value image too large; use contents(g)")
        snap = self.engine.snapshot()
        out = np.zeros((self.n_groups, self.window), dtype=np.int64)
        for g in range(self.n_groups):
            c = self.engine.contents(g)
            out[g, (int(snap["next_pos"][g]) + np.arange(len(c))) % self.window] = c
        return out

    def contents(self, group: int) -> np.ndarray:
        """Current window of a group in arrival order, oldest first."""
        return self.engine.contents(group)

    def aggregates(self) -> dict:
        """COUNT / SUM / AVG (/ MIN / MAX) of every group's window."""
        s = self.engine.snapshot()
        out = {"count": s["fill"], "sum": s["window_sum"], "avg": s["avg"]}
        if "min" in s:
            out["min"], out["max"] = s["min"], s["max"]
        return out

    def state_equal(self, other) -> bool:
        a = self.engine.snapshot()
        b = other.engine.snapshot() if isinstance(other, WindowStore) else {
            "fill": other.fill, "next_pos": other.next_pos, "window_sum": other.window_sum}
        if not all(np.array_equal(a[k], b[k]) for k in ("fill", "next_pos", "window_sum")):
            return False
        return all(np.array_equal(self.contents(g), other.contents(g)) for g in range(self.n_groups))


def ingest_sequence(store: WindowStore, groups, attrs, model=None, *, assume_grouped: bool = False,
                    want_sums: bool = False, want_costs: bool = False):
    """Ingest an ordered tuple sequence (engine.py:253-296).

    Per-group arrival order is preserved by the device's stable placement,
    so pre-grouped and arbitrary orders give identical windows.  The
    per-tuple trace (want_sums) and the simulated cost model (want_costs)
    belong to the reference's CPU backends and are not produced here.
    """
    if want_costs:
        raise InvalidConfigError("the simulated cost model belongs to the reference's CPU backends")
    g = np.asarray(groups)
    if len(g) == 0:
        return (np.empty(0, dtype=np.int64) if want_sums else None), None
    if assume_grouped:
        starts = np.concatenate(([0], np.flatnonzero(g[1:] != g[:-1]) + 1))
        if g.min() < 0 or g.max() >= store.n_groups:
            raise DataError(f"group id outside [0, {store.n_groups})")
        if len(np.unique(g[starts])) != len(starts):
            raise ConsistencyError("assume_grouped input has a split group run")
    if not want_sums:
        store.engine.ingest(g, np.asarray(attrs))
        return None, None
    # per-tuple sums in input order: the device trace is in grouped order
    # (stable by group), so un-permute with the stable argsort of the groups
    eng = store.engine
    eng.set_trace(True)
    try:
        eng.ingest(g, np.asarray(attrs))
        tg, ts = eng.trace()
    finally:
        eng.set_trace(False)
    sums = np.empty(len(g), dtype=np.int64)
    sums[np.argsort(g, kind="stable")] = ts
    return sums, None


def _segment_runs(reordered, n_groups: int):
    """Validate a reordered batch (engine.py:281-284) and cut it into group
    runs: (groups, indicator, run heads, run groups, run thread)."""
    groups = np.asarray(reordered.groups, dtype=np.int64)
    ind = np.asarray(reordered.indicator, dtype=np.int64)
    n = len(groups)
    if ind[0] != 0 or ind[-1] != n or (np.diff(ind) < 0).any():
        raise ConsistencyError("indicator does not cut the batch into segments")
    if n and (groups.min() < 0 or groups.max() >= n_groups):
        i = int(np.flatnonzero((groups < 0) | (groups >= n_groups))[0])
        raise DataError(f"tuple {i} has group {int(groups[i])}, outside [0, {n_groups})")
    heads = np.flatnonzero(np.r_[True, groups[1:] != groups[:-1]]) if n else np.empty(0, np.int64)
    run_g = groups[heads]
    if len(np.unique(run_g)) != len(run_g):
        raise ConsistencyError("reordered batch has a split group run")
    run_t = np.searchsorted(ind, heads, side="right") - 1
    return groups, ind, heads, run_g, run_t


def process_batch_cuda(reordered, store: WindowStore, trace=None) -> IterationReport:
    """CUDA executor for a reordered batch: the slot of process_batch_sim /
    process_batch_parallel (engine.py:299-429).

    The batch is executed with the partitioning it carries: thread t of the
    report is the device partition holding exactly the groups of segment t
    (in segment order; groups absent from the batch are parked on the last
    partition, they carry no work).  The store is mutated in place and
    per_thread_cost is each partition's aggregate-kernel time in ns.
    Validation follows the reference: a group id outside [0, G) raises
    DataError, a group split over two runs ConsistencyError (engine.py:281-284),
    both before anything is ingested."""
    eng = store.engine
    P = len(reordered.indicator) - 1
    if P != eng.n_partitions:
        raise InvalidConfigError(f"reordered batch has {P} threads, the store's engine {eng.n_partitions} partitions")
    groups, ind, heads, run_g, run_t = _segment_runs(reordered, store.n_groups)
    absent = np.setdiff1d(np.arange(store.n_groups), run_g)
    order = np.concatenate((run_g, absent))
    sizes = np.bincount(run_t, minlength=P)
    sizes[-1] += len(absent)
    offsets = np.zeros(P + 1, dtype=np.int64)
    np.cumsum(sizes, out=offsets[1:])
    eng.set_csr(order, offsets)
    if trace is not None:
        eng.set_trace(True)
    try:
        rep = eng.step(groups, np.asarray(reordered.attrs))
        if trace is not None:
            trace.append(*eng.trace())
    finally:
        if trace is not None:
            eng.set_trace(False)
    ns = eng.last_part_ns()
    tpt = np.diff(ind)
    return IterationReport(per_thread_cost=ns, makespan=int(ns.max()) if len(ns) else 0,
                           tuples=rep.tuples, imbalance=int(tpt.max() - tpt.min()) if len(tpt) else 0)


def process_batch_sim(reordered, store: WindowStore, model: CostModel, trace=None) -> IterationReport:
    """The reference's deterministic backend slot (engine.py:299-321): the
    batch is executed on the device (process_batch_cuda) and the report is
    in the reference's modelled cost units -- per-thread sums of
    ``CostModel.run_cost`` over each segment's runs, makespan = max +
    per_iteration_overhead -- so rows equal the reference's bit for bit."""
    if model is None:
        raise InvalidConfigError("cost accounting requires a CostModel")
    groups, ind, heads, run_g, run_t = _segment_runs(reordered, store.n_groups)
    f0 = store.engine.snapshot()["fill"][run_g]
    k = np.diff(np.r_[heads, len(groups)])
    rep = process_batch_cuda(reordered, store, trace)
    per_thread = np.bincount(run_t, weights=model.run_cost(f0, k, store.window),
                             minlength=len(ind) - 1).astype(np.int64)
    return IterationReport(per_thread_cost=per_thread,
                           makespan=int(per_thread.max()) + model.per_iteration_overhead,
                           tuples=rep.tuples, imbalance=rep.imbalance)


def process_batch_parallel(reordered, store: WindowStore, pool_size: int = 1, executor=None,
                           trace=None) -> IterationReport:
    """The reference's measured backend slot (engine.py:362-429): its logical
    threads are the device partitions, timed per partition (ns) by the
    aggregate kernel itself.  ``pool_size`` / ``executor`` are accepted for
    signature parity; the GPU is the pool."""
    if pool_size < 1:
        raise InvalidConfigError(f"pool_size must be >= 1, got {pool_size}")
    return process_batch_cuda(reordered, store, trace)


def ingest_tuple(store: WindowStore, group: int, attr: int, model: CostModel) -> tuple[int, int]:
    """Insert one value (engine.py:96-122): returns (window_sum, cost) after
    it, cost in the reference's model units."""
    if not 0 <= group < store.n_groups:
        raise DataError(f"group {group} outside [0, {store.n_groups})")
    eng = store.engine
    eng.step(np.array([group], dtype=np.uint32), np.array([attr], dtype=np.int64))
    r = eng.results()
    fill = int(r.count[0])
    cost = model.per_tuple_overhead + model.window_passes * model.per_element_cost * fill
    return int(r.sum[0]), int(cost)


def serial_reference(stream, window: int, batch_size: int = 1 << 20):
    """The reference's per-tuple oracle (engine.py:432-445) on the device:
    the whole stream through the fused step in trace mode.  Returns the
    final store and the AggregateTrace (compare with grouped_projection;
    the window state and the per-group projections are batch-independent)."""
    from .datagen import batches
    store = WindowStore(stream.n_groups, window, max_batch=batch_size)
    eng = store.engine
    buf = TraceBuffer()
    eng.set_trace(True)
    try:
        for b in batches(stream, batch_size):
            eng.step(b.groups, b.attrs)
            buf.append(*eng.trace())
    finally:
        eng.set_trace(False)
    return store, buf.build()
