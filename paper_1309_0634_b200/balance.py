"""Load-balancing policies, drop-in for the reference ``skewstream.balance``
(balance.py:1-405).

Every policy runs on the GPU (k_balance in csrc/balance.cuh via ss_balance):
the same greedy loops, tie rules, anti-ping-pong set, move cap and
MoveList (moves, scanned_tuples, final_tpt) as the reference.  Policy
functions keep the reference signature ``(stats, assignment, reordered,
cfg) -> MoveList`` and are pure: nothing is applied.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import ConsistencyError, InvalidConfigError
from .partition import Assignment, BatchStats, Move, ReorderedBatch, device_for


class Policy(Enum):
    NO_BALANCE = "no"
    GET_FIRST = "first"
    CHECK_ALL = "all"
    PROB_CHECK = "prob"
    BEST_BALANCE = "best"
    SHIFT = "shift"
    SHIFT_LOCAL = "shiftlocal"


@dataclass(frozen=True)
class BalancerConfig:
    """Tuning knobs shared by every policy (balance.py:38-65).

    ``split`` (new, not in the reference) turns on hot-key splitting across
    blocks with a final combine in the fused CUDA step.
    """

    policy: Policy = Policy.NO_BALANCE
    thread_threshold: int = 1000
    pot: float = 0.5
    max_moves: int | None = None
    split: bool = False

    def __post_init__(self) -> None:
        if not isinstance(self.policy, Policy):
            object.__setattr__(self, "policy", Policy(self.policy))
        if self.thread_threshold < 1:
            raise InvalidConfigError(f"thread_threshold must be >= 1, got {self.thread_threshold}")
        if not 0 < self.pot <= 1:
            raise InvalidConfigError(f"pot must be in (0, 1], got {self.pot}")
        if self.max_moves is not None and self.max_moves < 1:
            raise InvalidConfigError(f"max_moves must be >= 1, got {self.max_moves}")

    def resolved_max_moves(self, n_threads: int) -> int:
        return self.max_moves if self.max_moves is not None else 4 * n_threads

    def to_c(self, policy: Policy | None = None):
        from .stream_engine import StreamEngine
        p = (policy or self.policy).value
        return StreamEngine.balancer_struct(p, self.thread_threshold, self.pot, self.max_moves,
                                            split=self.split)


@dataclass(frozen=True)
class MoveList:
    """A policy's verdict for one batch (balance.py:68-80)."""

    moves: list
    scanned_tuples: int
    final_tpt: np.ndarray


def _device_policy(policy: Policy):
    def fn(stats: BatchStats, assignment: Assignment, reordered: ReorderedBatch,
           cfg: BalancerConfig) -> MoveList:
        # the policy reads the caller's BatchStats (balance.py:149-151):
        # group_counts drive the moves, tpt the loads.  The device derives the
        # loads from the counts and the assignment, and walks each donor's
        # entry segment in list order (the layout reorder_batch produced), so
        # stats / assignment / reordered must describe the same batch
        counts = np.asarray(stats.group_counts, dtype=np.int64)
        if len(counts) != assignment.n_groups:
            raise ConsistencyError(f"stats cover {len(counts)} groups, the assignment {assignment.n_groups}")
        tpt = np.bincount(assignment.group_to_thread, weights=counts,
                          minlength=assignment.n_threads).astype(np.int64)
        if not np.array_equal(tpt, np.asarray(stats.tpt, dtype=np.int64)):
            raise ConsistencyError("stats.tpt disagrees with group_counts under this assignment")
        if not np.array_equal(np.diff(np.asarray(reordered.indicator, dtype=np.int64)), tpt):
            raise ConsistencyError("reordered.indicator disagrees with stats.tpt")
        eng = device_for(assignment, 1)
        mv, scanned, final = eng.balance_counts(counts, cfg.to_c(policy))
        return MoveList([Move(g, s, d, pl) for g, s, d, pl in mv], int(scanned), final)
    fn.__name__ = policy.name.lower()
    fn.__doc__ = f"{policy.value!r} policy, executed by k_balance on the GPU."
    return fn


no_balance = _device_policy(Policy.NO_BALANCE)
get_first = _device_policy(Policy.GET_FIRST)
check_all = _device_policy(Policy.CHECK_ALL)
prob_check = _device_policy(Policy.PROB_CHECK)
best_balance = _device_policy(Policy.BEST_BALANCE)
shift = _device_policy(Policy.SHIFT)
shift_local = _device_policy(Policy.SHIFT_LOCAL)

POLICIES = {
    Policy.NO_BALANCE: no_balance, Policy.GET_FIRST: get_first, Policy.CHECK_ALL: check_all,
    Policy.PROB_CHECK: prob_check, Policy.BEST_BALANCE: best_balance, Policy.SHIFT: shift,
    Policy.SHIFT_LOCAL: shift_local,
}


def get_policy(policy) -> callable:
    if not isinstance(policy, Policy):
        try:
            policy = Policy(policy)
        except ValueError as exc:
            raise InvalidConfigError(f"unknown policy {policy!r}") from exc
    return POLICIES[policy]
