"""StreamEngine: the device-resident operator behind every public call.

One ``StreamEngine`` owns one ``ss_engine`` handle (include/ss_b200.h): the
per-group windows, the group -> partition assignment and the pipeline
scratch of one GPU.  Inputs may be numpy arrays (host) or torch tensors
(host or CUDA); host inputs are staged by the engine itself.  Every
computation runs in the CUDA library -- this module only marshals
pointers and maps status codes onto the reference's exception types
(errors.py).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .datagen import REPLAY_DTYPE
from .errors import DataError, InvalidConfigError

AGG_NAMES = {"count": L.AGG_COUNT, "sum": L.AGG_SUM, "avg": L.AGG_AVG,
             "min": L.AGG_MIN, "max": L.AGG_MAX}


@dataclass(frozen=True)
class WindowSpec:
    """Sliding window of the last ``rows`` values.

    scope='group' (default): each group's last ``rows`` values -- the
    reference's per-group ring (engine.py:51-70).  scope='stream': the last
    ``rows`` tuples of the whole stream, grouped (``[ROWS W]``; SURVEY 7.3's
    D1 alternative, 8(f) 4); COUNT / SUM / AVG / MIN / MAX per group over it.
    """

    rows: int
    scope: str = "group"

    def __post_init__(self):
        if self.rows < 1:
            raise InvalidConfigError(f"window must be >= 1, got {self.rows}")
        if self.scope not in ("group", "stream"):
            raise InvalidConfigError(f"scope must be 'group' or 'stream', got {self.scope!r}")


@dataclass(frozen=True)
class Aggregates:
    """Aggregate functions maintained per group (COUNT/SUM are the
    reference's own state, engine.py:67-70; AVG/MIN/MAX derive from it)."""

    names: tuple = ("count", "sum", "avg")

    def __post_init__(self):
        for n in self.names:
            if n not in AGG_NAMES:
                raise InvalidConfigError(f"unknown aggregate {n!r}")

    @property
    def mask(self) -> int:
        m = L.AGG_COUNT | L.AGG_SUM
        for n in self.names:
            m |= AGG_NAMES[n]
        return m


@dataclass
class StepReport:
    """Per-batch record (the fields of IterationReport, engine.py:167-176,
    plus the load-monitor outputs)."""

    tuples: int
    imbalance: int
    moves: int
    moves_applied_before: int
    scanned: int
    max_load: int
    touched: int
    split_groups: int
    mean_load: float
    load_ratio: float


@dataclass
class Results:
    """Per-batch emission: one row per group touched by the batch."""

    groups: np.ndarray
    count: np.ndarray
    sum: np.ndarray
    avg: np.ndarray
    min: np.ndarray | None = None
    max: np.ndarray | None = None


def _ptr(x):
    """(pointer, keepalive) of a numpy array or torch tensor."""
    if x is None:
        return None, None
    if isinstance(x, np.ndarray):
        x = np.ascontiguousarray(x)
        return x.ctypes.data_as(C.c_void_p), x
    # torch tensor
    if not x.is_contiguous():
        x = x.contiguous()
    return C.c_void_p(x.data_ptr()), x


def _first_bad_group(g, n_groups: int):
    bad = np.flatnonzero((g < 0) | (g >= n_groups))
    i = int(bad[0])
    return DataError(f"tuple {i} has group {int(g[i])}, outside [0, {n_groups})")


def _keys_u32(groups, n_groups: int):
    """Group ids as u32 for the device.  Ids the u32 view cannot carry (< 0 or
    >= 2^32) raise DataError here, before anything is staged; ids in
    [G, 2^32) are caught on the device (count_batch, partition.py:119-126)."""
    if isinstance(groups, np.ndarray):
        g = groups
        if g.dtype != np.uint32:
            if g.size and (g.min() < 0 or g.max() > 0xFFFFFFFF):
                raise _first_bad_group(g, n_groups)
            g = g.astype(np.uint32)
        return g
    import torch
    if groups.dtype == torch.int32 or groups.dtype == torch.uint32:
        return groups
    if groups.dtype == torch.int64:
        if groups.numel():
            lo, hi = torch.aminmax(groups)
            if int(lo) < 0 or int(hi) > 0xFFFFFFFF:      # would wrap into range as u32
                raise _first_bad_group(groups.cpu().numpy(), n_groups)
        return groups.to(torch.int32)
    raise InvalidConfigError(f"unsupported group dtype {groups.dtype}")


_I32_LO, _I32_HI = -(1 << 31), (1 << 31) - 1


def _attrs_i32(attrs):
    """Attribute values as int32 (the device ring width).  The reference
    stream's values are int32 (datagen.py:24-26); a wider value cannot be
    stored exactly and raises DataError before any state changes."""
    if isinstance(attrs, np.ndarray):
        if attrs.dtype == np.int32:
            return attrs
        if attrs.size and np.issubdtype(attrs.dtype, np.integer) and attrs.dtype.itemsize >= 4:
            lo, hi = attrs.min(), attrs.max()
            if lo < _I32_LO or hi > _I32_HI:
                i = int(np.flatnonzero((attrs < _I32_LO) | (attrs > _I32_HI))[0])
                raise DataError(f"tuple {i} has attr {int(attrs[i])}, outside the int32 range of the window store")
        elif attrs.size and not np.issubdtype(attrs.dtype, np.integer):
            raise DataError(f"attrs must be integers, got {attrs.dtype}")
        return attrs.astype(np.int32)
    import torch
    if attrs.dtype == torch.int32:
        return attrs
    if attrs.is_floating_point():
        raise DataError(f"attrs must be integers, got {attrs.dtype}")
    if attrs.dtype == torch.int64 and attrs.numel():
        lo, hi = torch.aminmax(attrs)
        if int(lo) < _I32_LO or int(hi) > _I32_HI:
            a = attrs.cpu().numpy()
            i = int(np.flatnonzero((a < _I32_LO) | (a > _I32_HI))[0])
            raise DataError(f"tuple {i} has attr {int(a[i])}, outside the int32 range of the window store")
    return attrs.to(torch.int32)


def hash_lists(n_groups: int, n_partitions: int, block: int | None = None):
    """Static hash partitioning: group g -> mix(g // block) mod P, ids
    ascending inside each partition (BASELINE C1 "static hash partitioning").

    Large domains hash blocks of 8 consecutive ids (one 32-byte sector of
    every per-group int32 array) instead of single ids, so the window
    update's per-member state reads of a partition come 8 to a sector; small
    domains (fewer than 64 groups per partition) hash single ids to keep
    every partition populated."""
    if block is None:
        import os
        block = 8 if n_groups >= 64 * n_partitions else 1
        block = int(os.environ.get("SS_B200_HASH_BLOCK", block))     # A/B measurement only
    g = np.arange(n_groups, dtype=np.uint64) // np.uint64(block)
    with np.errstate(over="ignore"):
        x = (g + np.uint64(0x9E3779B97F4A7C15)) * np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(31)
    part = (x % np.uint64(n_partitions)).astype(np.int64)
    order = np.lexsort((np.arange(n_groups), part))
    cuts = np.searchsorted(part[order], np.arange(n_partitions + 1))
    return [order[cuts[i]:cuts[i + 1]].tolist() for i in range(n_partitions)]


class StreamEngine:
    """Device-resident sliding-window GROUP BY with partitioned execution.

    ``n_partitions`` is the number of processing units (the aggregate
    kernel's CTAs); the reference's logical threads (harness.py:53-55).
    """

    def __init__(self, n_groups: int, window, n_partitions: int = 148,
                 aggregates=("count", "sum", "avg"), device: int = 0,
                 max_batch: int = 1 << 24, sub_batch: int = 0, pool_values: int = 0,
                 stream=None, key_bits: int = 32, initial: str = "contiguous"):
        self._lib = L.load()
        if key_bits not in (32, 64):
            raise InvalidConfigError("key_bits must be 32 or 64")
        self.key_bits = key_bits
        spec = window if isinstance(window, WindowSpec) else WindowSpec(int(window))
        aggs = aggregates if isinstance(aggregates, Aggregates) else Aggregates(tuple(aggregates))
        if n_groups < 1:
            raise InvalidConfigError(f"n_groups must be >= 1, got {n_groups}")
        if n_partitions < 1:
            raise InvalidConfigError(f"n_partitions must be >= 1, got {n_partitions}")
        self.n_groups = int(n_groups)
        self.window = spec.rows
        self.scope = spec.scope
        self.n_partitions = int(n_partitions)
        self.aggregates = aggs
        self.minmax = bool(aggs.mask & (L.AGG_MIN | L.AGG_MAX))
        cfg = L.Config(n_groups=self.n_groups, window=self.window,
                       n_partitions=self.n_partitions, key_bits=key_bits, agg_mask=aggs.mask,
                       scope=1 if spec.scope == "stream" else 0, device=device, reserved=0,
                       max_batch=int(max_batch),
                       sub_batch=int(sub_batch), pool_values=int(pool_values))
        h = C.c_void_p()
        rc = self._lib.ss_create(C.byref(cfg), C.byref(h))
        self._h = h
        if rc:
            msg = self._lib.ss_last_error(h) if h else b"ss_create failed"
            if h:
                self._lib.ss_destroy(h)
            self._h = None
            from .errors import raise_for_status
            raise_for_status(rc, msg.decode())
        if initial == "hash":
            self.set_lists(hash_lists(self.n_groups, self.n_partitions))
        elif initial != "contiguous":
            raise InvalidConfigError(f"unknown initial assignment {initial!r}")
        if stream is not None:
            self.set_stream(stream)
        self.sub_batch = int(self._lib.ss_sub_batch(self._h))

    # -- lifecycle ---------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._lib.ss_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        L.check(self._h, rc)

    def set_stream(self, stream):
        """Enqueue on a torch.cuda.Stream (or a raw cudaStream_t int)."""
        raw = getattr(stream, "cuda_stream", stream)
        self._check(self._lib.ss_set_stream(self._h, C.c_void_p(int(raw))))

    def sync(self):
        self._check(self._lib.ss_sync(self._h))

    # -- assignment --------------------------------------------------------
    def set_lists(self, lists):
        sizes = [len(x) for x in lists]
        offs = np.zeros(len(lists) + 1, dtype=np.int64)
        np.cumsum(sizes, out=offs[1:])
        self.set_csr(np.fromiter((g for lst in lists for g in lst), dtype=np.int64, count=int(offs[-1])), offs)

    def set_csr(self, order, offsets):
        """Load an assignment as concatenated ordered lists + offsets[P+1]."""
        offs = np.ascontiguousarray(offsets, dtype=np.int64)
        if len(offs) != self.n_partitions + 1:
            raise InvalidConfigError("assignment has a different number of partitions")
        order = np.ascontiguousarray(order, dtype=np.int32)
        po, _k1 = _ptr(order)
        pf, _k2 = _ptr(offs)
        self._check(self._lib.ss_set_assignment(self._h, po, pf))

    def get_csr(self):
        """(group_to_thread, order, offsets) of the device assignment."""
        g2t = np.empty(self.n_groups, dtype=np.int32)
        order = np.empty(self.n_groups, dtype=np.int32)
        offs = np.empty(self.n_partitions + 1, dtype=np.int64)
        self._check(self._lib.ss_get_assignment(self._h, _ptr(g2t)[0], _ptr(order)[0], _ptr(offs)[0]))
        return g2t.astype(np.int64), order.astype(np.int64), offs

    def get_lists(self):
        g2t, order, offs = self.get_csr()
        flat = order.tolist()
        return g2t, [flat[offs[p]:offs[p + 1]] for p in range(self.n_partitions)]

    def apply_moves(self, moves):
        """moves: iterable of (group, src, dst, placement) with placement
        'front'/'back' (partition.py:181-203)."""
        arr = (L.MoveC * max(1, len(moves)))()
        for i, (g, s, d, pl) in enumerate(moves):
            if pl not in ("front", "back"):
                raise InvalidConfigError(f"unknown placement {pl!r}")
            arr[i] = L.MoveC(int(g), int(s), int(d), L.BACK_CODE if pl == "back" else L.FRONT_CODE)
        self._check(self._lib.ss_apply_moves(self._h, arr, len(moves)))

    # -- partition step ----------------------------------------------------
    def count(self, groups):
        g = _keys_u32(groups, self.n_groups)
        n = len(g)
        counts = np.empty(self.n_groups, dtype=np.int64)
        tpt = np.empty(self.n_partitions, dtype=np.int64)
        pg, _k = _ptr(g)
        self._check(self._lib.ss_count(self._h, pg, n, _ptr(counts)[0], _ptr(tpt)[0]))
        return counts, tpt

    def reorder(self, groups, attrs):
        g = _keys_u32(groups, self.n_groups)
        a = _attrs_i32(attrs)
        n = len(g)
        og = np.empty(n, dtype=np.uint32)
        oa = np.empty(n, dtype=np.int32)
        ind = np.empty(self.n_partitions + 1, dtype=np.int64)
        pg, _k1 = _ptr(g)
        pa, _k2 = _ptr(a)
        self._check(self._lib.ss_reorder(self._h, pg, pa, n, _ptr(og)[0], _ptr(oa)[0], _ptr(ind)[0]))
        return og.astype(np.int64), oa.astype(np.int64), ind

    # -- aggregate update ----------------------------------------------------
    def ingest(self, groups, attrs):
        g = _keys_u32(groups, self.n_groups)
        a = _attrs_i32(attrs)
        pg, _k1 = _ptr(g)
        pa, _k2 = _ptr(a)
        self._check(self._lib.ss_ingest(self._h, pg, pa, len(g)))

    # -- balancer ------------------------------------------------------------
    @staticmethod
    def balancer_struct(policy="no", thread_threshold=1000, pot=0.5, max_moves=None,
                        split=False, split_target=1.2, split_max=0):
        if policy not in L.POLICY_CODES:
            raise InvalidConfigError(f"unknown policy {policy!r}")
        return L.Balancer(policy=L.POLICY_CODES[policy], reserved=0,
                          thread_threshold=int(thread_threshold), pot=float(pot),
                          max_moves=int(max_moves or 0), split=int(bool(split)),
                          split_max=int(split_max), split_target=float(split_target))

    def balance(self, groups, bal: "L.Balancer"):
        g = _keys_u32(groups, self.n_groups)
        cap = 4 * self.n_partitions if bal.max_moves <= 0 else int(bal.max_moves)
        cap = max(cap, 1)
        moves = (L.MoveC * cap)()
        nm = C.c_int64()
        sc = C.c_int64()
        ft = np.empty(self.n_partitions, dtype=np.int64)
        pg, _k = _ptr(g)
        self._check(self._lib.ss_balance(self._h, pg, len(g), C.byref(bal), moves, C.byref(nm),
                                         C.byref(sc), _ptr(ft)[0]))
        out = [(m.group, m.src, m.dst, "back" if m.placement == L.BACK_CODE else "front")
               for m in moves[:nm.value]]
        return out, sc.value, ft

    def balance_counts(self, counts, bal: "L.Balancer"):
        """The policy on given per-group counts (no recount); nothing applied."""
        c = np.ascontiguousarray(counts, dtype=np.int32)
        cap = 4 * self.n_partitions if bal.max_moves <= 0 else int(bal.max_moves)
        moves = (L.MoveC * max(cap, 1))()
        nm, sc = C.c_int64(), C.c_int64()
        ft = np.empty(self.n_partitions, dtype=np.int64)
        self._check(self._lib.ss_balance_counts(self._h, _ptr(c)[0], C.byref(bal), moves, C.byref(nm),
                                                C.byref(sc), _ptr(ft)[0]))
        out = [(m.group, m.src, m.dst, "back" if m.placement == L.BACK_CODE else "front")
               for m in moves[:nm.value]]
        return out, sc.value, ft

    # -- fused per-batch step --------------------------------------------------
    def step(self, groups, attrs, balancer=None, sync: bool = True):
        if self.key_bits == 64:
            return self._step64(groups, attrs, balancer, sync)
        g = _keys_u32(groups, self.n_groups)
        a = _attrs_i32(attrs)
        pg, _k1 = _ptr(g)
        pa, _k2 = _ptr(a)
        bal = balancer if balancer is not None else self.balancer_struct()
        rep = L.StepReport()
        self._check(self._lib.ss_step(self._h, pg, pa, len(g), C.byref(bal),
                                      C.byref(rep) if sync else None))
        # host inputs are copied asynchronously: keep the last two alive
        self._keep = (getattr(self, "_keep", (None, None))[-1], (_k1, _k2))
        return self._report(rep) if sync else None

    def step_records(self, records, balancer=None, sync: bool = True):
        """One batch given as replay records (datagen.REPLAY_DTYPE: u32 group,
        i32 attr), host (pinned for overlap) or device; SURVEY 8(f) 3."""
        if isinstance(records, np.ndarray):
            rec = np.ascontiguousarray(records)
            n = len(rec) if rec.dtype == REPLAY_DTYPE else rec.nbytes // 8
        else:
            rec = records.contiguous()
            n = rec.numel() * rec.element_size() // 8
        pr, _k = _ptr(rec)
        bal = balancer if balancer is not None else self.balancer_struct()
        rep = L.StepReport()
        self._check(self._lib.ss_step_records(self._h, pr, n, C.byref(bal), C.byref(rep) if sync else None))
        self._keep = (getattr(self, "_keep", (None, None))[-1], (_k,))
        return self._report(rep) if sync else None

    def _step64(self, keys, attrs, balancer, sync):
        if isinstance(keys, np.ndarray):
            k = np.ascontiguousarray(keys, dtype=np.int64)
        else:
            import torch
            k = keys.to(torch.int64).contiguous()
        a = _attrs_i32(attrs)
        pk, _k1 = _ptr(k)
        pa, _k2 = _ptr(a)
        bal = balancer if balancer is not None else self.balancer_struct()
        rep = L.StepReport()
        self._check(self._lib.ss_step_keys64(self._h, pk, pa, len(k), C.byref(bal),
                                             C.byref(rep) if sync else None))
        self._keep = (getattr(self, "_keep", (None, None))[-1], (_k1, _k2))
        return self._report(rep) if sync else None

    def slot_keys(self) -> np.ndarray:
        """int64 key of every assigned group slot (slots follow first appearance)."""
        n = C.c_int64()
        self._check(self._lib.ss_slot_keys(self._h, None, C.byref(n)))
        out = np.empty(max(1, n.value), dtype=np.int64)
        self._check(self._lib.ss_slot_keys(self._h, _ptr(out)[0], C.byref(n)))
        return out[:n.value]

    def set_key_pipeline(self, ready_inputs: bool = True):
        """int64 keys: declare device key inputs complete when step() is
        called, so the next batch's key probe may overlap this one (host
        inputs always do)."""
        self._check(self._lib.ss_set_key_pipeline(self._h, int(bool(ready_inputs))))

    def set_trace(self, enable: bool = True):
        """Per-tuple trace mode: every batch keeps all tuples
        and records (group, window sum after the tuple) per tuple."""
        self._check(self._lib.ss_set_trace(self._h, int(bool(enable))))

    def trace(self):
        """The last batch's trace in grouped-projection order (group ids
        ascending, arrival order within a group): (groups, sums) int64."""
        n = C.c_int64()
        self._check(self._lib.ss_trace(self._h, 0, None, None, C.byref(n)))
        g = np.empty(max(1, n.value), dtype=np.int32)
        sm = np.empty(max(1, n.value), dtype=np.int64)
        self._check(self._lib.ss_trace(self._h, n.value, _ptr(g)[0], _ptr(sm)[0], C.byref(n)))
        return g[:n.value].astype(np.int64), sm[:n.value]

    def set_graphs(self, enable: bool = True):
        """Replay the fused step as cached CUDA graphs (default on)."""
        self._check(self._lib.ss_set_graphs(self._h, int(bool(enable))))

    # -- streaming emission ---------------------------------
    def set_host_emit(self, enable: bool = True):
        """Every step writes its rows (group + the configured aggregates) into
        pinned host memory; results_pull() returns the oldest batch not yet
        pulled."""
        self._check(self._lib.ss_set_host_emit(self._h, int(bool(enable))))
        G = self.n_groups
        names = set(self.aggregates.names) | {"count", "sum"}
        self._pull = {
            "groups": np.empty(G, dtype=np.int32),
            "count": np.empty(G, dtype=np.int64) if "count" in names else None,
            "sum": np.empty(G, dtype=np.int64) if "sum" in names else None,
            "avg": np.empty(G, dtype=np.float64) if "avg" in names else None,
            "min": np.empty(G, dtype=np.int32) if self.minmax and "min" in names else None,
            "max": np.empty(G, dtype=np.int32) if self.minmax and "max" in names else None,
        }

    def results_pull(self) -> Results:
        """Rows of the oldest unpulled batch: groups plus the configured
        aggregate columns (None when not configured).  The arrays are views
        into reused buffers: copy them to keep them.  A batch the device
        rejected raises DataError here (it and the batches issued after it
        were not applied)."""
        n = C.c_int64()
        b = self._pull
        ptr = lambda k: (_ptr(b[k])[0] if b[k] is not None else None)
        self._check(self._lib.ss_results_pull(self._h, self.n_groups, ptr("groups"), ptr("count"), ptr("sum"),
                                              ptr("avg"), ptr("min"), ptr("max"), C.byref(n)))
        k = n.value
        cut = lambda a: None if a is None else a[:k]
        return Results(b["groups"][:k], cut(b["count"]), cut(b["sum"]), cut(b["avg"]), cut(b["min"]),
                       cut(b["max"]))

    def pulled_row_bytes(self) -> int:
        """Bytes per emitted row that results_pull moves device -> host."""
        wire = {"groups": 4, "count": 4, "sum": 8, "avg": 8, "min": 4, "max": 4}   # device column widths
        return sum(wire[k] for k, a in self._pull.items() if a is not None)

    def last_report(self) -> StepReport:
        rep = L.StepReport()
        self._check(self._lib.ss_last_report(self._h, C.byref(rep)))
        return self._report(rep)

    @staticmethod
    def _report(r) -> StepReport:
        return StepReport(r.tuples, r.imbalance, r.moves, r.moves_applied_before, r.scanned,
                          r.max_load, r.touched, r.split_groups, r.mean_load, r.load_ratio)

    def last_loads(self) -> np.ndarray:
        out = np.empty(self.n_partitions, dtype=np.int64)
        self._check(self._lib.ss_last_loads(self._h, _ptr(out)[0]))
        return out

    def last_part_work(self) -> np.ndarray:
        """Values stored by each partition's window update in the last batch."""
        out = np.empty(self.n_partitions, dtype=np.int64)
        self._check(self._lib.ss_last_part_work(self._h, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out

    def last_part_ns(self) -> np.ndarray:
        out = np.empty(self.n_partitions, dtype=np.int64)
        self._check(self._lib.ss_last_part_ns(self._h, _ptr(out)[0]))
        return out

    def last_moves(self):
        cap = 4 * self.n_partitions
        arr = (L.MoveC * cap)()
        n = C.c_int64()
        self._check(self._lib.ss_last_moves(self._h, arr, cap, C.byref(n)))
        return [(m.group, m.src, m.dst, "back" if m.placement == L.BACK_CODE else "front")
                for m in arr[:min(n.value, cap)]]

    # -- state export ----------------------------------------------------------
    def snapshot(self):
        G = self.n_groups
        out = {k: np.empty(G, dtype=np.int64) for k in ("fill", "next_pos", "window_sum")}
        mn = np.empty(G, dtype=np.int32)
        mx = np.empty(G, dtype=np.int32)
        avg = np.empty(G, dtype=np.float64)
        self._check(self._lib.ss_snapshot(self._h, _ptr(out["fill"])[0], _ptr(out["next_pos"])[0],
                                          _ptr(out["window_sum"])[0], _ptr(mn)[0], _ptr(mx)[0],
                                          _ptr(avg)[0]))
        out["avg"] = avg
        if self.minmax:
            out["min"] = mn.astype(np.int64)
            out["max"] = mx.astype(np.int64)
        return out

    def contents(self, group: int) -> np.ndarray:
        out = np.empty(self.window if self.window < (1 << 22) else 1, dtype=np.int64)
        n = C.c_int64()
        self._check(self._lib.ss_export_values(self._h, int(group), None, 0, C.byref(n)))
        out = np.empty(max(1, n.value), dtype=np.int64)
        self._check(self._lib.ss_export_values(self._h, int(group), _ptr(out)[0], n.value, C.byref(n)))
        return out[:n.value]

    def results(self) -> Results:
        n = C.c_int64()
        self._check(self._lib.ss_results(self._h, 0, None, None, None, None, None, None, C.byref(n)))
        k = n.value
        g = np.empty(k, dtype=np.int32)
        cnt = np.empty(k, dtype=np.int64)
        sm = np.empty(k, dtype=np.int64)
        avg = np.empty(k, dtype=np.float64)
        mn = np.empty(k, dtype=np.int32)
        mx = np.empty(k, dtype=np.int32)
        self._check(self._lib.ss_results(self._h, k, _ptr(g)[0], _ptr(cnt)[0], _ptr(sm)[0], _ptr(avg)[0],
                                         _ptr(mn)[0], _ptr(mx)[0], C.byref(n)))
        r = Results(g.astype(np.int64), cnt, sm, avg)
        if self.minmax:
            r.min = mn.astype(np.int64)
            r.max = mx.astype(np.int64)
        return r
