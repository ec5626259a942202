"""Key-sharded multi-GPU execution: one process per GPU.

Every rank owns the groups whose owner is its rank.  The group -> GPU map
is the assignment of a GPU-level engine whose "threads" are the GPUs; it
starts as a key hash (``initial="hash"``: group g on GPU hash(g) mod N, the
partitioner's hash option, stream_engine.hash_lists) or as contiguous id
ranges (initial_assignment with threads = GPUs, partition.py:97-114).

Per global batch, on the device and stream-ordered on ONE CUDA stream that
the engines and NCCL share:

  1. each rank takes its contiguous slice of the global batch (rank r's
     tuples all arrived before rank r+1's);
  2. ``ss_route_records`` stably splits the slice by owner into 8-byte
     (group, attr) records -- one message per tuple;
  3. a [world, 3] control block (tuples to each peer, this rank's bad-tuple
     status, migration words to each peer) is exchanged with one small
     all-to-all and read back ONCE -- the only host read of the step:
     NCCL's all-to-all takes its split sizes from the host;
  4. window state of the groups the previous batch's GPU-level policy moved
     travels as per-destination blobs (one all-to-all) and is imported on
     the device (``ss_import_blob_dev``);
  5. the records travel in one all-to-all (NCCL over NVLink/NVSwitch;
     gloo in the CPU tests); received chunks are concatenated in source-rank
     order, so every group's tuples arrive in global arrival order -- the
     only thing the windows depend on -- and the local
     fused step runs on them directly (``ss_step_records``);
  6. GPU-level balancing: the batch's per-group counts are all-reduced on
     the device, every rank runs the same device policy (k_balance,
     "threads" = GPUs) on identical inputs -- so every rank derives the same
     moves without a broadcast -- and applies them to its GPU-level
     assignment (``ss_balance_apply_dev``); the owner map is refreshed from
     that assignment on the device and the moved groups' state is exported
     into the blobs step 4 ships before the next batch.  Moves decided on
     batch t therefore take effect from batch t+1, the reference's
     one-iteration delay (harness.py:115-116).

int64 keys (``key_bits=64``) shard by a 16-bit key-hash bucket: the GPU-level
engine's groups are the 2^16 buckets, the route ships 12-byte (key, attr)
records, every GPU keeps its own key table, and moving a bucket migrates
all of its keys (each claims a slot on its new GPU at import).

The collectives are plumbing; all compute runs in libss_b200.so.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .errors import DataError, ExecutionError, InvalidConfigError
from .stream_engine import StreamEngine, _ptr



def _is_gloo(group) -> bool:
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def _coll_in(t, group):
    """Tensor as the collective backend wants it (gloo: host copy)."""
    return t.cpu() if _is_gloo(group) else t


def exchange_control(ctrl, group=None):
    """all-to-all of the [world, k] control block -> (sent, received) on the
    host; the one host read of a sharded step."""
    import torch
    import torch.distributed as dist
    send = _coll_in(ctrl.contiguous(), group)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    both = torch.stack([send, recv]).cpu().numpy()
    return both[0], both[1]


def exchange_records(rec, send_counts, recv_counts, group=None):
    """One all-to-all of 8-byte (group, attr) records (int64 view); output
    in source-rank order, on the input's device."""
    import torch
    import torch.distributed as dist
    src = _coll_in(rec, group)
    out = torch.empty(int(np.sum(recv_counts)), dtype=torch.int64, device=src.device)
    dist.all_to_all_single(out, src, [int(x) for x in recv_counts], [int(x) for x in send_counts], group=group)
    return out.to(rec.device, non_blocking=True)


def exchange_words(buf, send_words, recv_words, group=None):
    """All-to-all of int32 word segments (the migration blobs)."""
    import torch
    import torch.distributed as dist
    src = _coll_in(buf[:int(np.sum(send_words))], group)
    out = torch.empty(int(np.sum(recv_words)), dtype=torch.int32, device=src.device)
    dist.all_to_all_single(out, src, [int(x) for x in recv_words], [int(x) for x in send_words], group=group)
    return out.to(buf.device, non_blocking=True)


def allreduce_counts(counts, group=None):
    """Sum of per-group counts over the ranks, in place on the device
    (through the host for gloo)."""
    import torch.distributed as dist
    if _is_gloo(group):
        h = counts.cpu()
        dist.all_reduce(h, group=group)
        counts.copy_(h)
    else:
        dist.all_reduce(counts, group=group)
    return counts


class ShardedEngine:
    """One rank of a key-sharded engine (torch.distributed process group)."""

    KEY_BUCKETS = 1 << 16        # int64 keys: GPU-level "groups" are key-hash buckets (keys.cuh)

    def __init__(self, n_groups: int, window, n_partitions: int = 148, aggregates=("count", "sum", "avg"),
                 device: int = 0, max_batch: int = 1 << 24, sub_batch: int = 0, pool_values: int = 0,
                 group=None, initial: str = "hash", stream=None, key_bits: int = 32):
        import torch
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.world > 16:
            raise InvalidConfigError("at most 16 GPUs per sharded engine")
        self.n_groups = int(n_groups)
        self.dev = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.dev)
        self.key_bits = int(key_bits)
        self.local = StreamEngine(n_groups, window, n_partitions=n_partitions, aggregates=aggregates,
                                  device=device, max_batch=max_batch, sub_batch=sub_batch,
                                  pool_values=pool_values, stream=self.stream, key_bits=self.key_bits)
        self.window = self.local.window
        # the exchanged batch arrives in fresh buffers of varying size every
        # step: graph replay would recapture every time
        self.local.set_graphs(False)
        # GPU-level assignment + policy engine ("threads" = GPUs); its groups
        # are the group ids (u32) or the key-hash buckets (int64 keys)
        self.n_units = self.n_groups if self.key_bits == 32 else self.KEY_BUCKETS
        self.gpu = StreamEngine(self.n_units, 1, n_partitions=self.world, aggregates=("count", "sum"),
                                device=device, max_batch=1 << 16, initial=initial, stream=self.stream)
        owner, _ = self.gpu.get_lists()
        o = np.ascontiguousarray(owner, dtype=np.int32)
        lib = self.local._lib
        if self.key_bits == 32:
            self.local._check(lib.ss_set_owner(self.local._h, _ptr(o)[0], self.world))
        else:
            self.local._check(lib.ss_set_bucket_owner(self.local._h, _ptr(o)[0], self.world))
        i32, i64 = torch.int32, torch.int64
        self._route_cnt = torch.zeros(self.world + 1, dtype=i64, device=self.dev)
        self._counts = torch.zeros(self.n_units, dtype=i32, device=self.dev)
        self._owner = torch.as_tensor(o).to(self.dev)
        self._mig_words = torch.zeros(self.world, dtype=i64, device=self.dev)
        self._moves = None
        self._n_moves = torch.zeros(1, dtype=i32, device=self.dev)
        self._blob = None
        self._rec = None
        self._keep = None

    # -- device buffers ------------------------------------------------------
    def _move_buffers(self, bal):
        import torch
        cap = 4 * self.world if bal.max_moves <= 0 else int(bal.max_moves)
        if self._moves is None or self._moves.numel() < 4 * cap:
            self._moves = torch.zeros(4 * cap, dtype=torch.int32, device=self.dev)
        if self._blob is None:
            # every exported group carries <= W ring values plus its record;
            # int64 keys: a moved bucket carries ~G / 2^16 keys (at most 2^28
            # words in all -- a larger migration raises ExecutionError)
            per_unit = 1 if self.key_bits == 32 else self.n_groups // self.KEY_BUCKETS + 4
            words = min(1 << 28, min(cap, 256) * per_unit * (self.window + 9) + self.world)
            self._blob = torch.empty(words, dtype=torch.int32, device=self.dev)
        return cap

    def route(self, groups, attrs):
        """Stable split of this rank's slice by owner into 8-byte records
        (device int64 view; int64 keys: 12-byte records as int32 words) +
        counts[world + 1] (device; the last entry is the first bad tuple
        index or -1)."""
        import torch
        n = len(groups)
        if self.key_bits == 64:
            k = torch.as_tensor(groups).to(self.dev, torch.int64).contiguous()
            a = torch.as_tensor(attrs).to(self.dev, torch.int32).contiguous()
            if self._rec is None or self._rec.numel() < max(1, 3 * n):
                self._rec = torch.empty(max(1, 3 * n), dtype=torch.int32, device=self.dev)
            self._keep = (k, a)
            self.local._check(self.local._lib.ss_route_records64(self.local._h, _ptr(k)[0], _ptr(a)[0], n,
                                                                 _ptr(self._rec)[0], _ptr(self._route_cnt)[0]))
            return self._rec[:3 * n], self._route_cnt
        if self._rec is None or self._rec.numel() < max(1, n):
            self._rec = torch.empty(max(1, n), dtype=torch.int64, device=self.dev)
        pg, k1 = _ptr(groups)
        pa, k2 = _ptr(attrs)
        self._keep = (k1, k2, groups, attrs)
        self.local._check(self.local._lib.ss_route_records(self.local._h, pg, pa, n, _ptr(self._rec)[0],
                                                           _ptr(self._route_cnt)[0]))
        return self._rec[:n], self._route_cnt

    def _migrate(self, send_w, recv_w):
        """Ship and import the window state of the groups the last GPU-level
        policy moved (sizes from the control exchange)."""
        if (send_w < 0).any() or (recv_w < 0).any():
            raise ExecutionError("migration blob too small")
        if not (recv_w.any() or send_w.any()):
            return
        blob_in = exchange_words(self._blob, send_w, recv_w, self.group)
        if recv_w.any():
            seg = np.zeros(self.world + 1, dtype=np.int64)
            np.cumsum(recv_w, out=seg[1:])
            lib, h = self.local._lib, self.local._h
            if self.key_bits == 64:
                self.local._check(lib.ss_import_blob64_dev(h, _ptr(blob_in)[0], _ptr(seg)[0], self.world))
            else:
                self.local._check(lib.ss_import_blob_dev(h, _ptr(blob_in)[0], _ptr(seg)[0], self.world,
                                                         min(256, self._moves.numel() // 4)))
        self._mig_words.zero_()
        self._keep_blob = blob_in

    def settle(self):
        """Complete the migration the last batch's GPU-level moves started
        (a collective: every rank calls it).  Needed only to read the window
        state between batches -- the next step does it on its own."""
        import torch
        z = torch.zeros(self.world, dtype=torch.int64, device=self.dev)
        ctrl = torch.stack([z, z - 1, self._mig_words], dim=1)
        sent, got = exchange_control(ctrl, self.group)
        self._migrate(sent[:, 2], got[:, 2])

    # -- one global batch ------------------------------------------------------
    def step(self, groups, attrs, balancer=None, gpu_balancer=None):
        """groups/attrs: this rank's contiguous slice of the global batch
        (u32 group ids, or int64 keys with key_bits=64; host or device).
        Returns the tuples this rank ingested."""
        import torch
        n = len(groups)
        rec, cnt = self.route(groups, attrs)
        ctrl = torch.stack([cnt[:self.world], cnt[self.world].expand(self.world), self._mig_words], dim=1)
        sent, got = exchange_control(ctrl, self.group)
        bad = got[:, 1]
        if (bad >= 0).any():
            if sent[0, 1] >= 0:
                i = int(sent[0, 1])
                g = int(groups[i])
                raise DataError(f"tuple {i} has group {g}, outside [0, {self.n_groups})")
            r = int(np.flatnonzero(bad >= 0)[0])
            raise DataError(f"rank {r} rejected this batch (a tuple outside [0, {self.n_groups}))")
        self._migrate(sent[:, 2], got[:, 2])
        send_c, recv_c = sent[:, 0], got[:, 0]
        lib, h = self.local._lib, self.local._h
        if self.key_bits == 64:
            mine = exchange_words(rec, 3 * send_c, 3 * recv_c, self.group)
            self._keep_recv = mine
            bal = balancer if balancer is not None else self.local.balancer_struct()
            self.local._check(lib.ss_step_records64(h, _ptr(mine)[0], int(np.sum(recv_c)), C.byref(bal), None))
        else:
            mine = exchange_records(rec, send_c, recv_c, self.group)
            self._keep_recv = mine
            self.local.step_records(mine, balancer, sync=False)
        if gpu_balancer is not None and gpu_balancer.policy != L.POLICY_CODES["no"]:
            self._move_buffers(gpu_balancer)
            if self.key_bits == 64:
                self.local._check(lib.ss_bucket_counts_dev(h, _ptr(self._counts)[0]))
            else:
                self.local._check(lib.ss_group_counts(h, _ptr(self._counts)[0]))
            allreduce_counts(self._counts, self.group)
            self.gpu._check(lib.ss_balance_apply_dev(self.gpu._h, _ptr(self._counts)[0], C.byref(gpu_balancer),
                                                     _ptr(self._moves)[0], _ptr(self._n_moves)[0],
                                                     _ptr(self._owner)[0]))
            if self.key_bits == 64:
                self.local._check(lib.ss_set_bucket_owner(h, _ptr(self._owner)[0], self.world))
                self.local._check(lib.ss_export_moves64_dev(h, _ptr(self._moves)[0], _ptr(self._n_moves)[0],
                                                            self.rank, _ptr(self._blob)[0], self._blob.numel(),
                                                            _ptr(self._mig_words)[0]))
            else:
                self.local._check(lib.ss_set_owner_dev(h, _ptr(self._owner)[0], self.world))
                self.local._check(lib.ss_export_moves_dev(h, _ptr(self._moves)[0], _ptr(self._n_moves)[0],
                                                          self.rank, _ptr(self._blob)[0], self._blob.numel(),
                                                          _ptr(self._mig_words)[0]))
        return int(np.sum(recv_c))

    # -- inspection (synchronising; tests and reports only) --------------------
    @property
    def owner(self) -> np.ndarray:
        return self._owner.cpu().numpy().astype(np.int64)

    @property
    def last_gpu_moves(self):
        """Moves of the last step's GPU-level policy: (group, src, dst, placement)."""
        if self._moves is None:
            return []
        nm = int(self._n_moves.cpu()[0])
        m = self._moves[:4 * nm].cpu().numpy().reshape(-1, 4)
        return [(int(g), int(s), int(d), "back" if int(p) == L.BACK_CODE else "front") for g, s, d, p in m]

    def close(self):
        self.local.close()
        self.gpu.close()
