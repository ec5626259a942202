"""Replay-file ingest.

A replay file holds 8-byte records (u32 group, i32 attr) -- the reference's
`write_replay` / `read_replay` format (datagen.py:29,250-296).  `ReplayIngest`
streams one through a `StreamEngine`: batch i+1 is copied from the
memory-mapped file into one of two pinned host buffers while batch i runs
on the device (its H2D overlaps the previous batch's compute inside the
engine), records are split into keys / values on the device, and each
batch's rows (group + configured aggregates) are pulled one batch late
from pinned memory.
"""

from __future__ import annotations

import os
from typing import Callable, Iterator

import numpy as np

from .datagen import REPLAY_DTYPE
from .errors import InvalidSpecError


class ReplayIngest:
    def __init__(self, engine, path: str | os.PathLike, batch_size: int):
        import torch
        if batch_size < 1:
            raise InvalidSpecError(f"batch_size must be >= 1, got {batch_size}")
        size = os.path.getsize(path)
        if size % REPLAY_DTYPE.itemsize:
            raise InvalidSpecError(f"replay file size {size} is not a multiple of {REPLAY_DTYPE.itemsize} bytes")
        self.engine = engine
        self.batch_size = int(batch_size)
        self.n_tuples = size // REPLAY_DTYPE.itemsize
        self._rec = np.memmap(path, dtype=np.int64, mode="r") if self.n_tuples else np.empty(0, np.int64)
        self._pinned = [torch.empty(self.batch_size, dtype=torch.int64).pin_memory() for _ in range(2)]

    def __len__(self) -> int:
        return -(-self.n_tuples // self.batch_size)

    def batches(self, balancer=None, on_rows: Callable[[int, object], None] | None = None
                ) -> Iterator[int]:
        """Run every batch; yields the batch index after issuing it.  `on_rows(i,
        rows)` receives batch i's emitted rows (a stream_engine.Results: groups
        and the configured aggregates), one batch late.  A record whose group
        is outside [0, G) raises DataError at the pull of its batch
        (count_batch, partition.py:119-126)."""
        eng = self.engine
        eng.set_host_emit(True)
        for i in range(len(self)):
            lo = i * self.batch_size
            hi = min(self.n_tuples, lo + self.batch_size)
            buf = self._pinned[i % 2]
            # the buffer used two batches ago: its H2D was issued before the
            # previous batch, whose rows were pulled below, so it has landed
            buf[: hi - lo].numpy()[:] = self._rec[lo:hi]
            eng.step_records(buf[: hi - lo], balancer, sync=False)
            if i > 0:
                rows = eng.results_pull()
                if on_rows is not None:
                    on_rows(i - 1, rows)
            yield i
        if len(self):
            rows = eng.results_pull()
            if on_rows is not None:
                on_rows(len(self) - 1, rows)
