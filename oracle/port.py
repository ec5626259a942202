"""CPU oracle: a numpy restatement of the reference hot path.

TEST INFRASTRUCTURE ONLY.  Nothing under ``paper_1309_0634_b200/`` may
import this module; only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` use it, and
there only as the checker or the timed CPU baseline, never as product.

Every function restates the behaviour of the reference package
``skewstream`` (``/root/reference/pkg/src/skewstream``) and cites the
lines it follows.  The restatement is *pinned*: ``tests/golden/`` holds
fixtures produced by importing the reference itself
(``tests/golden/make_golden.py``) and ``tests/test_oracle.py`` checks this
module against every one of them.

Differences from the reference that do not change results:

* the window store is occupancy-proportional (per-group regions in one
  flat pool, capacity doubling up to W) instead of a dense ``[G, W]``
  matrix, so the C3/C4 shapes (W = 1e6 / 1e7) fit in memory;
* the store also derives MIN / MAX / AVG from the exact window contents
  (the reference computes SUM only; COUNT is its ``fill``);
* balancer extreme lookups use linear argmax/argmin (first index on ties)
  instead of lazy heaps -- the same lowest-id tie rule.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

FRONT = "front"
BACK = "back"

POLICY_NAMES = ("no", "first", "all", "prob", "best", "shift", "shiftlocal")


class OracleError(Exception):
    """Base for oracle-side precondition failures (mirrors errors.py:4-29)."""

    kind = "error"


class OracleDataError(OracleError):
    kind = "data"


class OracleConfigError(OracleError):
    kind = "config"


class OracleConsistencyError(OracleError):
    kind = "consistency"


class OracleStaleMoveError(OracleError):
    kind = "stale"


# --------------------------------------------------------------------------
# L1 partitioning  (partition.py)
# --------------------------------------------------------------------------

@dataclass
class OAssignment:
    """group->thread map plus ordered per-thread group lists (partition.py:45-94)."""

    g2t: np.ndarray
    lists: list

    @property
    def n_groups(self) -> int:
        return len(self.g2t)

    @property
    def n_threads(self) -> int:
        return len(self.lists)

    def clone(self) -> "OAssignment":
        return OAssignment(self.g2t.copy(), [list(x) for x in self.lists])

    def rank(self) -> np.ndarray:
        """Position of every group in concatenated list order (partition.py:63-70)."""
        flat = np.asarray([g for lst in self.lists for g in lst], dtype=np.int64)
        out = np.empty(self.n_groups, dtype=np.int64)
        out[flat] = np.arange(self.n_groups, dtype=np.int64)
        return out

    def csr(self) -> tuple[np.ndarray, np.ndarray]:
        order = np.asarray([g for lst in self.lists for g in lst], dtype=np.int64)
        off = np.zeros(self.n_threads + 1, dtype=np.int64)
        np.cumsum([len(x) for x in self.lists], out=off[1:])
        return order, off


def contiguous_assignment(n_groups: int, n_threads: int) -> OAssignment:
    """Consecutive id ranges, sizes differing by at most one (partition.py:97-114)."""
    if n_groups < 1 or n_threads < 1:
        raise OracleConfigError("need n_groups >= 1 and n_threads >= 1")
    q, r = divmod(n_groups, n_threads)
    sizes = [q + (t < r) for t in range(n_threads)]
    lists, g2t, lo = [], np.empty(n_groups, dtype=np.int64), 0
    for t, s in enumerate(sizes):
        lists.append(list(range(lo, lo + s)))
        g2t[lo:lo + s] = t
        lo += s
    return OAssignment(g2t, lists)


def histogram(groups: np.ndarray, asg: OAssignment) -> tuple[np.ndarray, np.ndarray]:
    """Per-group counts and per-thread tpt; DataError names the first bad tuple
    (partition.py:117-130)."""
    g = np.asarray(groups, dtype=np.int64)
    if g.size:
        bad = np.flatnonzero((g < 0) | (g >= asg.n_groups))
        if bad.size:
            i = int(bad[0])
            raise OracleDataError(f"tuple {i} has group {int(g[i])}, outside "
                                  f"[0, {asg.n_groups})")
    counts = np.bincount(g, minlength=asg.n_groups).astype(np.int64)
    tpt = np.bincount(asg.g2t[g], minlength=asg.n_threads).astype(np.int64)
    return counts, tpt


def place(groups, attrs, asg: OAssignment, counts, tpt):
    """Stable thread-major, group-contiguous placement (partition.py:161-178).

    Returns (groups', attrs', indicator[P+1]).
    """
    n = len(groups)
    if int(np.sum(tpt)) != n or int(np.sum(counts)) != n:
        raise OracleConsistencyError("stats do not sum to the batch size")
    key = asg.rank()[np.asarray(groups, dtype=np.int64)]
    perm = np.argsort(key, kind="stable")
    ind = np.zeros(asg.n_threads + 1, dtype=np.int64)
    ind[1:] = np.cumsum(tpt)
    return (np.asarray(groups, dtype=np.int64)[perm],
            np.asarray(attrs, dtype=np.int64)[perm], ind)


def apply_move_list(asg: OAssignment, moves) -> OAssignment:
    """Sequential application on a copy (partition.py:181-203).

    ``moves`` is a list of (group, src, dst, placement) tuples.
    """
    out = asg.clone()
    for g, s, d, pl in moves:
        if pl not in (FRONT, BACK):
            raise OracleConfigError(f"unknown placement {pl!r}")
        if not (0 <= s < out.n_threads and 0 <= d < out.n_threads):
            raise OracleConfigError("thread out of range")
        if not (0 <= g < out.n_groups):
            raise OracleConfigError("group out of range")
        if int(out.g2t[g]) != s:
            raise OracleStaleMoveError(f"group {g} is on {int(out.g2t[g])}, not {s}")
        out.lists[s].remove(g)
        if pl == BACK:
            out.lists[d].append(g)
        else:
            out.lists[d].insert(0, g)
        out.g2t[g] = d
    return out


# --------------------------------------------------------------------------
# L3 window store + closed-form ingest  (engine.py)
# --------------------------------------------------------------------------

class OStore:
    """Per-group windows of the last W values, occupancy-proportional.

    Same observable state as the reference ``WindowStore`` (engine.py:51-93):
    ``fill``, ``next_pos``, ``window_sum`` and ring slot contents; slot
    ``s`` of group ``g`` lives at ``pool[off[g] + s]``.  A region grows by
    doubling while the window fills; a filling window is linear
    (next_pos == 0, engine.py:54-57), so growth copies ``fill`` values.
    """

    def __init__(self, n_groups: int, window: int, dense_limit: int = 1 << 24):
        if n_groups < 1 or window < 1:
            raise OracleConfigError("n_groups and window must be >= 1")
        self.n_groups = n_groups
        self.window = window
        self.fill = np.zeros(n_groups, dtype=np.int64)
        self.next_pos = np.zeros(n_groups, dtype=np.int64)
        self.window_sum = np.zeros(n_groups, dtype=np.int64)
        if n_groups * window <= dense_limit:
            self.cap = np.full(n_groups, window, dtype=np.int64)
            self.off = np.arange(n_groups, dtype=np.int64) * window
            self.pool = np.zeros(n_groups * window, dtype=np.int64)
            self._top = n_groups * window
        else:
            self.cap = np.zeros(n_groups, dtype=np.int64)
            self.off = np.zeros(n_groups, dtype=np.int64)
            self.pool = np.zeros(1 << 16, dtype=np.int64)
            self._top = 0

    # -- storage management -------------------------------------------------
    def _reserve(self, groups: np.ndarray, need: np.ndarray) -> None:
        w = self.window
        grow = need > self.cap[groups]
        if not grow.any():
            return
        gs, nd = groups[grow], need[grow]
        new_cap = np.minimum(w, np.maximum(np.maximum(nd, 2 * self.cap[gs]), 8))
        total = int(new_cap.sum())
        if self._top + total > len(self.pool):
            size = max(2 * len(self.pool), self._top + total)
            pool = np.zeros(size, dtype=np.int64)
            pool[:self._top] = self.pool[:self._top]
            self.pool = pool
        starts = self._top + np.concatenate(([0], np.cumsum(new_cap)[:-1]))
        for g, st in zip(gs.tolist(), starts.tolist()):
            f = int(self.fill[g])
            if f:
                o = int(self.off[g])
                self.pool[st:st + f] = self.pool[o:o + f]
        self.off[gs] = starts
        self.cap[gs] = new_cap
        self._top += total

    def contents(self, g: int) -> np.ndarray:
        """Window of group g, oldest first (engine.py:72-77)."""
        f, p = int(self.fill[g]), int(self.next_pos[g])
        idx = (p + np.arange(f)) % self.window
        return self.pool[int(self.off[g]) + idx].copy()

    # -- closed-form batch update (engine.py:185-250) ------------------------
    def ingest_runs(self, rg: np.ndarray, starts: np.ndarray, lens: np.ndarray,
                    vals: np.ndarray, want_sums: bool = False):
        """One contiguous run of values per group, applied in closed form.

        For a group with prior (f0, p0, S0) receiving k values the new
        timeline is old-window ++ run; the final state and the ring slots
        of the last min(k, W) values follow directly.
        """
        w = self.window
        r = len(rg)
        if r == 0:
            return np.empty(0, dtype=np.int64) if want_sums else None
        f0 = self.fill[rg].copy()
        p0 = self.next_pos[rg].copy()
        s0 = self.window_sum[rg].copy()
        self._reserve(rg, np.minimum(f0 + lens, w))
        base = self.off[rg]
        run_of = np.repeat(np.arange(r), lens)           # run id per value
        j = np.arange(len(vals), dtype=np.int64) - starts[run_of]

        sums = None
        if want_sums:
            # timeline = prior window ++ run; per-tuple sum = window over it
            plen = f0
            pcum = np.concatenate(([0], np.cumsum(plen)))
            prun = np.repeat(np.arange(r), plen)
            pj = np.arange(int(pcum[-1]), dtype=np.int64) - pcum[:-1][prun]
            prior = self.pool[base[prun] + (p0[prun] + pj) % w]
            tl_len = f0 + lens
            tcum = np.concatenate(([0], np.cumsum(tl_len)))
            tl = np.empty(int(tcum[-1]), dtype=np.int64)
            tl[tcum[:-1][prun] + pj] = prior
            tl[tcum[:-1][run_of] + f0[run_of] + j] = vals
            cs = np.concatenate(([0], np.cumsum(tl)))
            hi = f0[run_of] + j + 1
            lo = np.maximum(hi - w, 0)
            b = tcum[:-1][run_of]
            sums = cs[b + hi] - cs[b + lo]

        total = f0 + lens
        # evicted prior values: the first max(0, f0+k-W) old entries when k < W
        full_replace = lens >= w
        n_evict = np.where(full_replace, 0, np.maximum(total - w, 0))
        ecum = np.concatenate(([0], np.cumsum(n_evict)))
        erun = np.repeat(np.arange(r), n_evict)
        ej = np.arange(int(ecum[-1]), dtype=np.int64) - ecum[:-1][erun]
        evicted = self.pool[base[erun] + (p0[erun] + ej) % w]
        ev_sum = np.zeros(r, dtype=np.int64)
        np.add.at(ev_sum, erun, evicted)

        kept = np.minimum(lens, w)
        kcum = np.concatenate(([0], np.cumsum(kept)))
        krun = np.repeat(np.arange(r), kept)
        kj = np.arange(int(kcum[-1]), dtype=np.int64) - kcum[:-1][krun]
        t_idx = (lens - kept)[krun] + kj                 # index inside the run
        kv = vals[starts[krun] + t_idx]
        kept_sum = np.zeros(r, dtype=np.int64)
        np.add.at(kept_sum, krun, kv)
        all_sum = np.zeros(r, dtype=np.int64)
        np.add.at(all_sum, run_of, vals)

        new_sum = np.where(full_replace, kept_sum, s0 + all_sum - ev_sum)
        slot = (p0[krun] + f0[krun] + t_idx) % w
        self.pool[base[krun] + slot] = kv
        self.fill[rg] = np.minimum(total, w)
        self.next_pos[rg] = (p0 + np.maximum(total - w, 0)) % w
        self.window_sum[rg] = new_sum
        return sums

    def ingest(self, groups, attrs, assume_grouped: bool = False,
               want_sums: bool = False):
        """Ordered sequence ingest (engine.py:253-296)."""
        g = np.asarray(groups, dtype=np.int64)
        a = np.asarray(attrs, dtype=np.int64)
        n = len(g)
        if n == 0:
            return np.empty(0, dtype=np.int64) if want_sums else None
        order = None
        if not assume_grouped:
            order = np.argsort(g, kind="stable")
            g, a = g[order], a[order]
        edge = np.flatnonzero(g[1:] != g[:-1]) + 1
        starts = np.concatenate(([0], edge)).astype(np.int64)
        lens = np.diff(np.concatenate((starts, [n]))).astype(np.int64)
        rg = g[starts]
        if rg.min() < 0 or rg.max() >= self.n_groups:
            raise OracleDataError(f"group id outside [0, {self.n_groups})")
        if assume_grouped and len(np.unique(rg)) != len(rg):
            raise OracleConsistencyError("assume_grouped input has a split group run")
        sums = self.ingest_runs(rg, starts, lens, a, want_sums)
        if order is not None and sums is not None:
            out = np.empty_like(sums)
            out[order] = sums
            sums = out
        return sums

    # -- aggregates (north-star additions over the reference) ----------------
    def aggregates(self, groups=None):
        """COUNT, SUM, AVG, MIN, MAX of the current windows.

        COUNT = fill, SUM = window_sum (engine.py:67-70); AVG is the
        correctly rounded float64 quotient; MIN/MAX scan contents().
        Empty windows report MIN = MAX = 0 and AVG = 0.0.
        """
        gs = np.arange(self.n_groups) if groups is None else np.asarray(groups)
        cnt = self.fill[gs].copy()
        sm = self.window_sum[gs].copy()
        avg = np.where(cnt > 0, sm.astype(np.float64) / np.maximum(cnt, 1), 0.0)
        mn = np.zeros(len(gs), dtype=np.int64)
        mx = np.zeros(len(gs), dtype=np.int64)
        for i, g in enumerate(np.asarray(gs).tolist()):
            c = self.contents(g)
            if len(c):
                mn[i] = c.min()
                mx[i] = c.max()
        return cnt, sm, avg, mn, mx


# --------------------------------------------------------------------------
# L2 balancing  (balance.py)
# --------------------------------------------------------------------------

@dataclass
class OVerdict:
    moves: list = field(default_factory=list)     # (g, src, dst, placement)
    scanned: int = 0
    final_tpt: np.ndarray | None = None


class _Lists:
    """Lazily copied working per-thread lists (balance.py:116-134)."""

    def __init__(self, lists):
        self.base = lists
        self.mut = {}

    def get(self, t):
        return self.mut.get(t, self.base[t])

    def own(self, t):
        if t not in self.mut:
            self.mut[t] = list(self.base[t])
        return self.mut[t]


def _cap(cfg, n_threads):
    mm = cfg.get("max_moves")
    return mm if mm is not None else 4 * n_threads    # balance.py:64-65


def _extremes(counts, tpt, asg, cfg, choose):
    """Hottest->coolest greedy loop shared by four policies (balance.py:141-172)."""
    loads = [int(x) for x in tpt]
    cap = _cap(cfg, asg.n_threads)
    thr = cfg["thread_threshold"]
    work = _Lists(asg.lists)
    moved: set = set()
    out = OVerdict()
    while len(out.moves) < cap:
        hi = max(range(len(loads)), key=lambda t: (loads[t], -t))
        lo = min(range(len(loads)), key=lambda t: (loads[t], t))
        if loads[hi] - loads[lo] <= thr:
            break
        got = choose(loads, work, moved, hi, lo)
        if got is None:
            break
        g, scanned = got
        out.scanned += scanned
        c = int(counts[g])
        work.own(hi).remove(g)
        work.own(lo).append(g)
        out.moves.append((g, hi, lo, BACK))
        moved.add(g)
        loads[hi] -= c
        loads[lo] += c
    out.final_tpt = np.asarray(loads, dtype=np.int64)
    return out


def policy_no(counts, tpt, asg, rgroups, ind, cfg):
    """balance.py:175-178."""
    return OVerdict([], 0, np.asarray(tpt, dtype=np.int64).copy())


def policy_first(counts, tpt, asg, rgroups, ind, cfg):
    """Donor's current first group, unless moved or empty (balance.py:181-200)."""
    def choose(loads, work, moved, hi, lo):
        lst = work.get(hi)
        if not lst:
            return None
        g = lst[0]
        if g in moved or int(counts[g]) == 0:
            return None
        return g, 0
    return _extremes(counts, tpt, asg, cfg, choose)


def policy_all(counts, tpt, asg, rgroups, ind, cfg):
    """Heaviest non-moved donor group; charges the entry segment (balance.py:203-227)."""
    def choose(loads, work, moved, hi, lo):
        best = None
        for g in work.get(hi):
            if g in moved:
                continue
            key = (int(counts[g]), -g)
            if best is None or key > best[0]:
                best = (key, g)
        if best is None or best[0][0] <= 0:
            return None
        return best[1], int(ind[hi + 1] - ind[hi])
    return _extremes(counts, tpt, asg, cfg, choose)


def policy_prob(counts, tpt, asg, rgroups, ind, cfg):
    """Scan the donor's entry segment until a count reaches the limit
    (balance.py:230-264)."""
    pot = cfg["pot"]

    def choose(loads, work, moved, hi, lo):
        owned = work.get(hi)
        if not owned:
            return None
        limit = math.ceil(pot * loads[hi] / len(owned))
        seg = rgroups[int(ind[hi]):int(ind[hi + 1])].tolist()
        seen = {}
        for pos, g in enumerate(seg, start=1):
            seen[g] = seen.get(g, 0) + 1
            if seen[g] >= limit and g not in moved:
                return g, pos
        best_g, best_c = -1, 0
        for g, c in seen.items():
            if g in moved:
                continue
            if c > best_c or (c == best_c and g < best_g):
                best_g, best_c = g, c
        if best_c <= 0:
            return None
        return best_g, len(seg)
    return _extremes(counts, tpt, asg, cfg, choose)


def policy_best(counts, tpt, asg, rgroups, ind, cfg):
    """Group minimising the post-move pair gap; strict improvement only
    (balance.py:267-293)."""
    def choose(loads, work, moved, hi, lo):
        dmax, dmin = loads[hi], loads[lo]
        best = None
        for g in work.get(hi):
            if g in moved:
                continue
            c = int(counts[g])
            key = (abs((dmax - c) - (dmin + c)), g)
            if best is None or key < best:
                best = key
        if best is None or best[0] >= dmax - dmin:
            return None
        return best[1], 0
    return _extremes(counts, tpt, asg, cfg, choose)


def policy_shift(counts, tpt, asg, rgroups, ind, cfg):
    """Neighbour cascades between the extremes (balance.py:296-342)."""
    loads = [int(x) for x in tpt]
    cap = _cap(cfg, asg.n_threads)
    thr = cfg["thread_threshold"]
    work = _Lists(asg.lists)
    moved: set = set()
    moves = []
    while len(moves) < cap:
        hi = loads.index(max(loads))
        lo = loads.index(min(loads))
        if loads[hi] - loads[lo] <= thr:
            break
        down = hi > lo
        span = range(lo + 1, hi + 1) if down else range(hi, lo)
        emitted = 0
        for i in span:
            if len(moves) >= cap:
                break
            lst = work.get(i)
            if not lst:
                continue
            g = lst[0] if down else lst[-1]
            if g in moved:
                continue
            dst = i - 1 if down else i + 1
            work.own(i).remove(g)
            if down:
                work.own(dst).append(g)
            else:
                work.own(dst).insert(0, g)
            c = int(counts[g])
            loads[i] -= c
            loads[dst] += c
            moves.append((g, i, dst, BACK if down else FRONT))
            moved.add(g)
            emitted += 1
        if emitted == 0:
            break
    return OVerdict(moves, 0, np.asarray(loads, dtype=np.int64))


def policy_shiftlocal(counts, tpt, asg, rgroups, ind, cfg):
    """One sweep over adjacent pairs with immediate updates (balance.py:345-385)."""
    loads = [int(x) for x in tpt]
    cap = _cap(cfg, asg.n_threads)
    thr = cfg["thread_threshold"]
    work = _Lists(asg.lists)
    moved: set = set()
    moves = []
    for i in range(asg.n_threads - 1):
        if len(moves) >= cap:
            break
        if loads[i] - loads[i + 1] > thr:
            src, dst, last = i, i + 1, True
        elif loads[i + 1] - loads[i] > thr:
            src, dst, last = i + 1, i, False
        else:
            continue
        lst = work.get(src)
        if not lst:
            continue
        g = lst[-1] if last else lst[0]
        if g in moved:
            continue
        work.own(src).remove(g)
        if last:
            work.own(dst).insert(0, g)
        else:
            work.own(dst).append(g)
        c = int(counts[g])
        loads[src] -= c
        loads[dst] += c
        moves.append((g, src, dst, FRONT if last else BACK))
        moved.add(g)
    return OVerdict(moves, 0, np.asarray(loads, dtype=np.int64))


POLICY_FNS = {
    "no": policy_no, "first": policy_first, "all": policy_all,
    "prob": policy_prob, "best": policy_best, "shift": policy_shift,
    "shiftlocal": policy_shiftlocal,
}


def balancer_cfg(policy="no", thread_threshold=1000, pot=0.5, max_moves=None):
    """Validated knobs (balance.py:38-65)."""
    if policy not in POLICY_FNS:
        raise OracleConfigError(f"unknown policy {policy!r}")
    if thread_threshold < 1 or not (0 < pot <= 1) or (
            max_moves is not None and max_moves < 1):
        raise OracleConfigError("bad balancer config")
    return {"policy": policy, "thread_threshold": int(thread_threshold),
            "pot": float(pot), "max_moves": max_moves}


# --------------------------------------------------------------------------
# L4 pipeline  (harness.py:85-140)
# --------------------------------------------------------------------------

@dataclass
class ORow:
    tuples: int
    tpt: np.ndarray
    imbalance: int
    moves_applied_before: int
    scanned: int
    moves: list


def run_batches(batch_iter, n_groups: int, window: int, n_threads: int,
                cfg: dict | None = None, want_rows: bool = True,
                asg: OAssignment | None = None):
    """count -> place -> policy -> ingest -> apply, moves delayed one batch.

    ``batch_iter`` yields (groups, attrs) arrays.  Returns (store, final
    assignment, rows).  Mirrors the loop body of harness.run (99-117).
    """
    cfg = cfg or balancer_cfg()
    asg = asg or contiguous_assignment(n_groups, n_threads)
    store = OStore(n_groups, window)
    fn = POLICY_FNS[cfg["policy"]]
    rows, prev = [], 0
    for groups, attrs in batch_iter:
        counts, tpt = histogram(groups, asg)
        rg, ra, ind = place(groups, attrs, asg, counts, tpt)
        verdict = fn(counts, tpt, asg, rg, ind, cfg)
        store.ingest(rg, ra, assume_grouped=True)
        if want_rows:
            rows.append(ORow(len(rg), tpt, int(tpt.max() - tpt.min()) if len(tpt) else 0,
                             prev, verdict.scanned, list(verdict.moves)))
        asg = apply_move_list(asg, verdict.moves)
        prev = len(verdict.moves)
    return store, asg, rows
