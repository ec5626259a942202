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


def process_batch_cuda(reordered, store: WindowStore, trace=None) -> IterationReport:
    """CUDA executor for a reordered batch: the slot of process_batch_sim /
    process_batch_parallel (engine.py:299-429)."""
    eng = store.engine
    if trace is not None:
        eng.set_trace(True)
    try:
        rep = eng.step(np.asarray(reordered.groups), np.asarray(reordered.attrs))
        if trace is not None:
            trace.append(*eng.trace())
    finally:
        if trace is not None:
            eng.set_trace(False)
    ns = eng.last_part_ns()
    tpt = np.diff(np.asarray(reordered.indicator))
    return IterationReport(per_thread_cost=ns, makespan=int(ns.max()) if len(ns) else 0,
                           tuples=rep.tuples, imbalance=int(tpt.max() - tpt.min()) if len(tpt) else 0)


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
