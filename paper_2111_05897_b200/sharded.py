"""Hash-sharded embedding worker over N GPUs.

One process per GPU. Every rank holds the rows it owns -- rank ``route_shard(id, S) %
world`` (``ShardSet::shard_of``, embedding_ps.hpp:521-523, with the S logical shards
spread round-robin over the ranks) -- in a local ``hps.ShardSet`` created with all S
shard salts, and runs one embedding worker over its own batch. A step is the reference's
E embedding workers in front of a sharded parameter server
(``EmbeddingWorker::fetch_rows`` embedding_worker.hpp:677-704, ``serve_pull`` :523-571,
``push_to_shards`` :726-775, ``PsShardService`` :185-290), with the per-frame RPCs
replaced by three NCCL all-to-alls:

  forward   route (distinct ids grouped by owner) -> ids to owners -> owner lookup
            (find_or_init + gather + versions) -> rows back -> fp64 pooling
  backward  pairs (one fp64 chain-rule contribution per (sample, distinct id), grouped
            by owner) -> (position, contribution) to owners -> owner applies them in
            (source rank, sample) order = ascending SampleId (rank << 56 | counter,
            core.hpp:98-125; flush order embedding_worker.hpp:788-790)

Two transports move the payloads:
  "p2p"   (default on GPUs) the kernels write every payload once, straight into the
          consumer's HBM over NVLink (CUDA IPC peer mappings of a per-rank arena), with
          device-side barriers -- no collective on the data path, one host round trip per
          step (hps_exchange_forward / _pool / _backward in libhps.so).
  "nccl"  torch.distributed all-to-alls between the local kernels (hps_exchange_route /
          _pool / _pairs, hps_table_gather / hps_table_apply_pairs); ``ops`` is injectable
          so this sequencing is testable with gloo on CPU (tests/test_sharded.py checks it
          against the reference's multi-worker semantics with an oracle-backed ops).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import hps


class DeviceOps:
    """The local steps of a sharded step on this rank's GPU (libhps.so)."""

    def __init__(self, table: hps.ShardSet, world: int, aggregation: int):
        import torch

        self.torch = torch
        self.table = table
        self.world = world
        self.D = table.embedding_dim
        self.device = torch.device("cuda", torch.cuda.current_device())
        h = hps.vp()
        hps.check(hps.lib().hps_exchange_create(world, table.shard_count, aggregation, -1,
                                                C.byref(h)), "exchange")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            hps.lib().hps_exchange_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _s(self):
        return self.torch.cuda.current_stream().cuda_stream

    def route(self, ids, offsets, B: int, F: int):
        """-> (send_ids buffer [>= U], per-owner counts as a device tensor [world])."""
        t = self.torch
        n = ids.numel()
        send = t.empty(max(n, 1), dtype=t.int64, device=self.device)
        counts = t.empty(self.world, dtype=t.int64, device=self.device)
        hps.check(hps.lib().hps_exchange_route(self.h, ids.data_ptr(), n, offsets.data_ptr(), B,
                                               F, send.data_ptr(), counts.data_ptr(), self._s()),
                  "exchange_route")
        return send, counts

    def lookup(self, recv_ids):
        t = self.torch
        n = recv_ids.numel()
        rows = t.empty((n, self.D), dtype=t.float32, device=self.device)
        ver = t.empty(n, dtype=t.int64, device=self.device)
        if n:
            hps.check(hps.lib().hps_table_gather(self.table.h, recv_ids.data_ptr(), n,
                                                 rows.data_ptr(), ver.data_ptr(), hps.ASYNC,
                                                 self._s()), "owner lookup")
        return rows, ver

    def pool(self, rows, B: int, F: int, out=None):
        t = self.torch
        if out is None:
            out = t.empty((B, F, self.D), dtype=t.float32, device=self.device)
        hps.check(hps.lib().hps_exchange_pool(self.h, rows.data_ptr() if rows.numel() else None,
                                              self.D, out.data_ptr(), self._s()), "exchange_pool")
        return out

    def pairs(self, grads, n_ids: int):
        """-> (pair_pos buffer, contribution buffer, per-owner pair counts on the device)."""
        t = self.torch
        grads = grads.contiguous()
        pos = t.empty(max(n_ids, 1), dtype=t.int32, device=self.device)
        con = t.empty((max(n_ids, 1), self.D), dtype=t.float32, device=self.device)
        counts = t.empty(self.world, dtype=t.int64, device=self.device)
        hps.check(hps.lib().hps_exchange_pairs(self.h, grads.data_ptr(), self.D, pos.data_ptr(),
                                               con.data_ptr(), counts.data_ptr(), self._s()),
                  "exchange_pairs")
        return pos, con, counts

    def apply_pairs(self, recv_ids, recv_versions, id_counts, pair_pos, contrib, pair_counts,
                    lr: float, step_tag: int, epoch: int, flags: int = 0) -> bool:
        W = self.world
        ic = (C.c_uint64 * W)(*id_counts)
        pc = (C.c_uint64 * W)(*pair_counts)
        acc = C.c_int(0)
        hps.check(hps.lib().hps_table_apply_pairs(
            self.table.h, recv_ids.data_ptr() if recv_ids.numel() else None,
            recv_versions.data_ptr() if recv_versions is not None and recv_versions.numel()
            else None, ic, pair_pos.data_ptr() if pair_pos.numel() else None,
            contrib.data_ptr() if contrib.numel() else None, pc, W, lr, step_tag, epoch,
            C.byref(acc), flags, self._s()), "apply_pairs")
        return bool(acc.value)


class _DeviceArray:
    """A raw device float32 buffer for torch.as_tensor (zero-copy)."""

    def __init__(self, ptr: int, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4",
                                         "data": (ptr, False), "version": 3, "strides": None}


class PeerExchange:
    """The NVLink peer transport (libhps.so hps_exchange_arena/connect/forward/backward)."""

    def __init__(self, ops: DeviceOps, dist, group, rank: int, max_ids: int, max_groups: int,
                 kappa: float = 0.0):
        import torch

        self.ops = ops
        self.max_ids = max_ids
        handle = (C.c_uint8 * 64)()
        if kappa:
            hps.check(hps.lib().hps_exchange_set_codec(ops.h, kappa), "exchange codec")
        hps.check(hps.lib().hps_exchange_arena(ops.h, max_ids, max_groups, ops.D, handle),
                  "exchange arena")
        ptr = hps.vp()
        hps.check(hps.lib().hps_exchange_pooled(ops.h, C.byref(ptr)), "exchange pooled")
        self.pooled_ptr = ptr.value
        mine = bytes(handle)
        world = ops.world
        if world > 1:
            got = [None] * world
            dist.all_gather_object(got, mine, group=group)
        else:
            got = [mine]
        allh = (C.c_uint8 * (64 * world)).from_buffer_copy(b"".join(got))
        hps.check(hps.lib().hps_exchange_connect(ops.h, rank, allh), "exchange connect")
        torch.cuda.synchronize()

    def forward(self, ids, offsets, B, F):
        o = self.ops
        hps.check(hps.lib().hps_exchange_forward(o.h, o.table.h, ids.data_ptr(), ids.numel(),
                                                 offsets.data_ptr(), B, F, o._s()),
                  "exchange forward")

    def prefetch(self, ids, offsets, B, F):
        o = self.ops
        hps.check(hps.lib().hps_exchange_prefetch(o.h, o.table.h, ids.data_ptr(), ids.numel(),
                                                  offsets.data_ptr(), B, F, o._s()),
                  "exchange prefetch")

    def forward_prefetched(self):
        o = self.ops
        hps.check(hps.lib().hps_exchange_forward_prefetched(o.h, o.table.h, o._s()),
                  "exchange forward (prefetched)")

    def pool(self, B, F, out=None):
        """Pooled [B, F, D]: a zero-copy view of the arena's pooled buffer (valid until the
        next forward) when out is None, else copied into out."""
        o = self.ops
        hps.check(hps.lib().hps_exchange_pool(o.h, None, o.D,
                                              out.data_ptr() if out is not None else None,
                                              o._s()), "exchange pool")
        if out is not None:
            return out
        return o.torch.as_tensor(_DeviceArray(self.pooled_ptr, (B, F, o.D)), device=o.device)

    def backward(self, grads, lr, step_tag, epoch, flags):
        o = self.ops
        acc = C.c_int(0)
        hps.check(hps.lib().hps_exchange_backward(o.h, o.table.h, grads.contiguous().data_ptr(),
                                                  lr, step_tag, epoch, C.byref(acc), flags,
                                                  o._s()), "exchange backward")
        return bool(acc.value)


class ShardedEmbeddingWorker:
    """``register_batch`` / ``serve_pull`` / ``apply_backward`` of one rank's embedding
    worker over the hash-sharded table (sync order; one batch in flight).

    transport: "p2p" (NVLink peer writes; needs ``max_ids`` >= listings per batch) or
    "nccl" (all-to-alls); default "p2p" unless ``ops`` is injected."""

    def __init__(self, table: hps.ShardSet, aggregation: int = hps.MEAN, group=None, ops=None,
                 transport: str | None = None, max_ids: int | None = None,
                 max_groups: int | None = None, codec_kappa: float = 0.0):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        self.table = table
        self.aggregation = aggregation
        self.transport = transport or ("nccl" if ops is not None else "p2p")
        self.ops = ops if ops is not None else DeviceOps(table, self.world, aggregation)
        self.B = self.F = 0
        self.peer = None
        self.max_ids = max_ids
        self.max_groups = max_groups
        # kappa > 0: rows and contributions cross NVLink as kappa-scaled binary16 (the
        # reference's compress_values codec, opt-in and lossy; p2p transport)
        self.codec_kappa = codec_kappa

    # -- collectives ------------------------------------------------------------------
    def _exchange_counts(self, counts):
        """counts[d] = what this rank sends to d (list or tensor) -> (send counts, what each
        source sends to this rank), both host lists; one device->host copy."""
        import torch

        if self.world == 1:
            c = [int(x) for x in (counts.tolist() if torch.is_tensor(counts) else counts)]
            return c, c
        dev = self._comm_device()
        send = counts.to(dev) if torch.is_tensor(counts) else \
            torch.tensor(counts, dtype=torch.int64, device=dev)
        recv = torch.empty_like(send)
        self.dist.all_to_all_single(recv, send, group=self.group)
        both = torch.cat([send, recv]).tolist()
        return [int(x) for x in both[:self.world]], [int(x) for x in both[self.world:]]

    def _a2a(self, inp, send_counts, recv_counts):
        if self.world == 1:
            return inp
        import torch

        out = torch.empty((sum(recv_counts),) + tuple(inp.shape[1:]), dtype=inp.dtype,
                          device=inp.device)
        self.dist.all_to_all_single(out, inp.contiguous(), output_split_sizes=list(recv_counts),
                                    input_split_sizes=list(send_counts), group=self.group)
        return out

    def _comm_device(self):
        import torch

        backend = self.dist.get_backend(self.group)
        return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"

    # -- the worker surface ---------------------------------------------------------------
    def register_batch(self, ids, offsets, B: int, F: int):
        """Route the batch's ids to their owners and fetch the rows (fetch_rows)."""
        self.B, self.F, self.n_ids = B, F, ids.numel()
        if self.transport == "p2p":
            if self.peer is None:
                self.peer = PeerExchange(self.ops, self.dist, self.group, self.rank,
                                         self.max_ids or max(ids.numel(), 1),
                                         max(self.max_groups or 0, B * F), self.codec_kappa)
            self.peer.forward(ids, offsets, B, F)
            return
        send_ids, counts = self.ops.route(ids, offsets, B, F)
        self.send_counts, self.recv_counts = self._exchange_counts(counts)
        self.recv_ids = self._a2a(send_ids[:sum(self.send_counts)], self.send_counts,
                                  self.recv_counts)
        rows, self.recv_versions = self.ops.lookup(self.recv_ids)
        self.rows = self._a2a(rows, self.recv_counts, self.send_counts)

    def prefetch(self, ids, offsets, B: int, F: int):
        """Phase 1 of register_batch (p2p): route the batch and plan its backward pairs --
        no barrier and no table access, so it may run on a stream beside the previous
        batch's backward. Complete it with register_prefetched() after that backward."""
        if self.transport != "p2p":
            raise hps.PreconditionError("prefetch needs the p2p transport")
        if self.peer is None:
            self.peer = PeerExchange(self.ops, self.dist, self.group, self.rank,
                                     self.max_ids or max(ids.numel(), 1),
                                     max(self.max_groups or 0, B * F), self.codec_kappa)
        self._pending = (B, F, ids.numel())
        self.peer.prefetch(ids, offsets, B, F)

    def register_prefetched(self):
        """Phase 2: owner lookup and row delivery of the prefetched batch (fetch_rows)."""
        self.B, self.F, self.n_ids = self._pending
        self.peer.forward_prefetched()

    def serve_pull(self, out_pooled=None):
        """Pooled embeddings [B, F, D] of the registered batch (serve_pull)."""
        if self.transport == "p2p":
            return self.peer.pool(self.B, self.F, out_pooled)
        return self.ops.pool(self.rows, self.B, self.F, out_pooled)

    def apply_backward(self, grads, lr: float, step_tag: int, epoch: int | None = None,
                       flags: int = hps.ASYNC) -> bool:
        """Per-sample gradients [B, F, D] -> owners, applied in ascending SampleId.
        Data-dependent errors (non-finite contributions, capacity) surface from
        ``table.sync()`` unless flags = 0."""
        if self.transport == "p2p":
            e = self.table.epoch() if epoch is None else epoch
            return self.peer.backward(grads, lr, step_tag, e, flags)
        pos, con, counts = self.ops.pairs(grads, self.n_ids)
        self.pair_counts, recv_pair_counts = self._exchange_counts(counts)
        P = sum(self.pair_counts)
        rpos = self._a2a(pos[:P], self.pair_counts, recv_pair_counts)
        rcon = self._a2a(con[:P], self.pair_counts, recv_pair_counts)
        e = self.table.epoch() if epoch is None else epoch
        return self.ops.apply_pairs(self.recv_ids, self.recv_versions, self.recv_counts, rpos,
                                    rcon, recv_pair_counts, lr, step_tag, e, flags)


def owner_of(ids: np.ndarray, shard_count: int, world: int) -> np.ndarray:
    """Owner rank of each id (host helper for tests and tools)."""
    return np.array([hps.route_shard(int(i), shard_count) % world for i in ids], np.int64)
