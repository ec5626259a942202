"""Key-sharded multi-GPU execution: one process per GPU.

Every rank owns the groups whose owner is its rank (a group -> GPU map that
starts as contiguous id ranges, like initial_assignment with threads =
GPUs, partition.py:97-114).  Per batch:

  1. each rank takes its contiguous slice of the global batch (so rank r's
     tuples all arrived before rank r+1's);
  2. ``ss_route`` stably splits the slice by owner on the device;
  3. counts, then tuples, are exchanged with all-to-all (NCCL over
     NVLink/NVSwitch; gloo for CPU tests); received chunks are concatenated
     in source-rank order, so every group's tuples arrive in global arrival
     order -- the only thing the windows depend on;
  4. the local StreamEngine runs the fused step on its share;
  5. GPU-level balancing: per-group counts are all-reduced and the same
     device policy (k_balance, "threads" = GPUs) runs on every rank on
     identical inputs, so every rank derives the same moves without a
     broadcast; moved groups' windows migrate from the old to the new
     owner (exact ring images, next_pos included) before the next batch.

The collectives are plumbing; all compute runs in libss_b200.so.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .stream_engine import StreamEngine, _ptr


def _coll_device(group):
    import torch.distributed as dist
    return "cpu" if dist.get_backend(group) == "gloo" else "cuda"


def exchange_counts(counts, group=None):
    """all-to-all of the per-destination counts -> per-source counts."""
    import torch
    import torch.distributed as dist
    dev = _coll_device(group)
    send = torch.as_tensor(np.asarray(counts, dtype=np.int64)).to(dev)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    return recv.cpu().numpy()


def exchange_tuples(send_g, send_a, send_counts, recv_counts, group=None):
    """all-to-all of the routed tuples; output is source-rank ordered."""
    import torch
    import torch.distributed as dist
    dev = _coll_device(group)
    out_dev = send_g.device
    sg, sa = send_g.to(dev), send_a.to(dev)
    n = int(np.sum(recv_counts))
    rg = torch.empty(n, dtype=send_g.dtype, device=dev)
    ra = torch.empty(n, dtype=send_a.dtype, device=dev)
    ins, outs = [int(x) for x in send_counts], [int(x) for x in recv_counts]
    dist.all_to_all_single(rg, sg, outs, ins, group=group)
    dist.all_to_all_single(ra, sa, outs, ins, group=group)
    return rg.to(out_dev), ra.to(out_dev)


def allreduce_counts(counts: np.ndarray, group=None) -> np.ndarray:
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(np.ascontiguousarray(counts, dtype=np.int32)).to(_coll_device(group))
    dist.all_reduce(t, group=group)
    return t.cpu().numpy()


def migrate(moves, rank, world, export_fn, import_fn, group=None):
    """Ship the window state of moved groups from their old to their new
    owner.  ``moves`` is identical on every rank; export_fn(groups) ->
    (meta int64[n,5], values int32[...]); import_fn(groups, meta, values)."""
    import torch
    import torch.distributed as dist
    dev = _coll_device(group)
    out = [[] for _ in range(world)]
    for g, src, dst, _ in moves:
        if src == rank and dst != rank:
            out[dst].append(g)
    payload, sizes = [], np.zeros(world, dtype=np.int64)
    for d in range(world):
        if not out[d]:
            continue
        gs = np.asarray(out[d], dtype=np.int32)
        meta, vals = export_fn(gs)
        blob = np.concatenate([np.asarray([len(gs), len(vals)], dtype=np.int64),
                               gs.astype(np.int64), meta.reshape(-1).astype(np.int64),
                               vals.astype(np.int64)])
        payload.append(blob)
        sizes[d] = len(blob)
    recv_sizes = exchange_counts(sizes, group)
    send = torch.as_tensor(np.concatenate(payload) if payload else np.zeros(0, np.int64)).to(dev)
    recv = torch.empty(int(recv_sizes.sum()), dtype=torch.int64, device=dev)
    dist.all_to_all_single(recv, send, [int(x) for x in recv_sizes], [int(x) for x in sizes], group=group)
    buf = recv.cpu().numpy()
    pos = 0
    for s in range(world):
        end = pos + int(recv_sizes[s])
        while pos < end:
            ng, nv = int(buf[pos]), int(buf[pos + 1])
            pos += 2
            gs = buf[pos:pos + ng].astype(np.int32)
            pos += ng
            meta = buf[pos:pos + 5 * ng].reshape(ng, 5)
            pos += 5 * ng
            vals = buf[pos:pos + nv].astype(np.int32)
            pos += nv
            import_fn(gs, meta, vals)


class ShardedEngine:
    """One rank of a key-sharded engine (torch.distributed process group)."""

    def __init__(self, n_groups: int, window, n_partitions: int = 148, aggregates=("count", "sum", "avg"),
                 device: int = 0, max_batch: int = 1 << 24, sub_batch: int = 0, pool_values: int = 0,
                 group=None):
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.n_groups = n_groups
        self.local = StreamEngine(n_groups, window, n_partitions=n_partitions, aggregates=aggregates,
                                  device=device, max_batch=max_batch, sub_batch=sub_batch,
                                  pool_values=pool_values)
        # the exchanged batch arrives in fresh buffers of varying size every
        # step: graph replay would recapture every time
        self.local.set_graphs(False)
        # GPU-level assignment + policy engine ("threads" = GPUs)
        self.gpu = StreamEngine(n_groups, 1, n_partitions=self.world, aggregates=("count", "sum"),
                                device=device, max_batch=1 << 16)
        self.owner, _ = self.gpu.get_lists()
        self._set_owner()
        self.last_gpu_moves = []

    def _set_owner(self):
        o = np.ascontiguousarray(self.owner, dtype=np.int32)
        self.local._check(self.local._lib.ss_set_owner(self.local._h, _ptr(o)[0], self.world))

    # -- device route --------------------------------------------------------
    def route(self, groups, attrs):
        import torch
        n = len(groups)
        dev = groups.device if isinstance(groups, torch.Tensor) else None
        if dev is not None and dev.type == "cuda":
            og = torch.empty(n, dtype=torch.int32, device=dev)
            oa = torch.empty(n, dtype=torch.int32, device=dev)
        else:
            og = torch.empty(n, dtype=torch.int32)
            oa = torch.empty(n, dtype=torch.int32)
        counts = np.zeros(self.world, dtype=np.int64)
        pg, _k1 = _ptr(groups)
        pa, _k2 = _ptr(attrs)
        self.local._check(self.local._lib.ss_route(self.local._h, pg, pa, n, _ptr(og)[0], _ptr(oa)[0],
                                                   _ptr(counts)[0]))
        return og, oa, counts

    # -- state migration -----------------------------------------------------
    def export_state(self, groups):
        g = np.ascontiguousarray(groups, dtype=np.int32)
        meta = np.zeros((len(g), 5), dtype=np.int64)
        nv = C.c_int64()
        lib, h = self.local._lib, self.local._h
        self.local._check(lib.ss_export_state(h, _ptr(g)[0], len(g), _ptr(meta)[0], None, 0, C.byref(nv)))
        vals = np.zeros(max(1, nv.value), dtype=np.int32)
        self.local._check(lib.ss_export_state(h, _ptr(g)[0], len(g), _ptr(meta)[0], _ptr(vals)[0],
                                              nv.value, C.byref(nv)))
        return meta, vals[:nv.value]

    def import_state(self, groups, meta, values):
        g = np.ascontiguousarray(groups, dtype=np.int32)
        m = np.ascontiguousarray(meta, dtype=np.int64)
        v = np.ascontiguousarray(values, dtype=np.int32)
        self.local._check(self.local._lib.ss_import_state(self.local._h, _ptr(g)[0], len(g), _ptr(m)[0],
                                                          _ptr(v)[0]))

    # -- one global batch ------------------------------------------------------
    def step(self, groups, attrs, balancer=None, gpu_balancer=None):
        """groups/attrs: this rank's contiguous slice of the global batch."""
        send_g, send_a, counts = self.route(groups, attrs)
        recv_counts = exchange_counts(counts, self.group)
        rg, ra = exchange_tuples(send_g, send_a, counts, recv_counts, self.group)
        rep = self.local.step(rg, ra, balancer)
        self.last_gpu_moves = []
        if gpu_balancer is not None and gpu_balancer.policy != L.POLICY_CODES["no"]:
            c = np.zeros(self.n_groups, dtype=np.int32)
            self.local._check(self.local._lib.ss_group_counts(self.local._h, _ptr(c)[0]))
            total = allreduce_counts(c, self.group)
            moves, _, _ = self.gpu.balance_counts(total, gpu_balancer)
            if moves:
                migrate(moves, self.rank, self.world, self.export_state, self.import_state, self.group)
                self.gpu.apply_moves(moves)
                self.owner, _ = self.gpu.get_lists()
                self._set_owner()
            self.last_gpu_moves = moves
        return rep, int(np.sum(recv_counts))

    def close(self):
        self.local.close()
        self.gpu.close()
