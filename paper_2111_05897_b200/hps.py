"""Python host mirror of the reference's embedding PS / embedding-worker operator API.

Thin ctypes layer over the C ABI in ``include/hps_c.h`` (``libhps.so``, built for
sm_100a). Names and error behaviour follow the reference
(``/root/reference/proj/include/hybridps``):

* ``ShardSet``  ~ ``ShardSet`` / ``PsShard`` (embedding_ps.hpp:56-553): ``lookup``,
  ``apply_gradients`` (tracked), ``apply_gradients_map`` (untracked), counters,
  epochs.
* ``EmbeddingWorker`` ~ ``EmbeddingWorker`` (embedding_worker.hpp:470-905) at
  batch granularity: ``register_batch`` / ``serve_pull`` / ``apply_backward``.
* ``compress_indices`` / ``dedup`` ~ codec.hpp:123-182; ``mix64`` /
  ``route_shard`` ~ core.hpp:36-44, 145-150.

Arrays may be numpy (host) or torch CUDA tensors (device); the library detects
the pointer kind. There is no CPU fallback: importing this module without the
built library raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# HPS_LIB: an alternative build of the same library (profiling experiments only)
LIB_PATH = os.environ.get("HPS_LIB") or os.path.join(_HERE, "libhps.so")

# ---- errors (errors.hpp:22-107) ------------------------------------------------------


class Error(RuntimeError):
    code = -1


class PreconditionError(Error):
    code = 1


class ConfigError(Error):
    code = 2


class ProtocolError(Error):
    code = 3


class TransportError(Error):
    code = 4


class CheckpointCorruptError(Error):
    code = 5


class DivergenceError(Error):
    code = 6


class ConsistencyError(Error):
    code = 7


class UndefinedMetricError(Error):
    code = 8


class StaleSampleError(Error):
    code = 9


class BackpressureError(Error):
    code = 10


class ClockError(Error):
    code = 11


class SyncFailureError(Error):
    code = 12


class UnrecoverableRunError(Error):
    code = 13


class CudaError(Error):
    code = 100


_ERRORS = {c.code: c for c in (PreconditionError, ConfigError, ProtocolError, TransportError,
                               CheckpointCorruptError, DivergenceError, ConsistencyError,
                               UndefinedMetricError, StaleSampleError, BackpressureError,
                               ClockError, SyncFailureError, UnrecoverableRunError, CudaError)}

ADAGRAD, SGD = 0, 1
MEAN, SUM = 0, 1
ASYNC = 1
DEVICE_STEP = 2
TABLE_TAG_RING = 1  # hps_table_cfg.flags
TABLE_LRU = 2

# ---- library loading -----------------------------------------------------------------

_lib = None

vp = C.c_void_p


class Counters(C.Structure):
    _fields_ = [("misses", C.c_uint64), ("evictions", C.c_uint64), ("clock_resets", C.c_uint64),
                ("stale_epoch_drops", C.c_uint64), ("size", C.c_uint64), ("capacity", C.c_uint64),
                ("epoch", C.c_uint32), ("max_delay", C.c_uint32),
                ("delay_hist", C.c_uint64 * 17)]


class TableCfg(C.Structure):
    _fields_ = [("shard_count", C.c_uint32), ("shard_salts", C.POINTER(C.c_uint64)),
                ("capacity", C.c_uint64), ("embedding_dim", C.c_uint32),
                ("optimizer", C.c_int32), ("device", C.c_int32), ("owner_rank", C.c_uint32),
                ("world_size", C.c_uint32), ("flags", C.c_uint32), ("reserved0", C.c_uint32),
                ("shard_capacity", C.c_uint64)]


def lib():
    """Loads libhps.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    st = C.c_int
    sz = C.c_size_t
    u32, u64, f32, i32 = C.c_uint32, C.c_uint64, C.c_float, C.c_int32
    sig = {
        "hps_last_error": (C.c_char_p, []),
        "hps_abi_version": (C.c_int, []),
        "hps_mix64": (u64, [u64]),
        "hps_route_shard": (u32, [u64, u32]),
        "hps_route": (st, [vp, sz, u32, vp, vp]),
        "hps_table_create": (st, [C.POINTER(TableCfg), C.POINTER(vp)]),
        "hps_table_destroy": (st, [vp]),
        "hps_table_counters": (st, [vp, C.POINTER(Counters)]),
        "hps_table_sync": (st, [vp]),
        "hps_table_epoch": (u32, [vp]),
        "hps_table_device_step": (st, [vp, C.POINTER(u32)]),
        "hps_table_advance_epoch": (u32, [vp]),
        "hps_table_reset": (st, [vp]),
        "hps_compress_values": (st, [vp, u64, u32, f32, vp, vp, vp]),
        "hps_decompress_values": (st, [vp, vp, u64, u32, vp, vp]),
        "hps_table_checkpoint_save": (st, [vp, u32, u32, vp, u64, C.POINTER(u64)]),
        "hps_table_checkpoint_load": (st, [vp, C.POINTER(vp), C.POINTER(u64), u32, C.c_int]),
        "hps_lookup": (st, [vp, vp, sz, vp, vp, vp]),
        "hps_table_gather": (st, [vp, vp, sz, vp, vp, u32, vp]),
        "hps_apply": (st, [vp, vp, vp, vp, sz, f32, u32, u32, vp, C.POINTER(C.c_int), u32, vp]),
        "hps_peek": (st, [vp, vp, sz, vp, vp, vp, vp, vp]),
        "hps_batch_create": (st, [vp, i32, C.POINTER(vp)]),
        "hps_batch_destroy": (st, [vp]),
        "hps_batch_register": (st, [vp, vp, sz, vp, u32, u32, vp, vp]),
        "hps_batch_pull": (st, [vp, vp, vp, vp]),
        "hps_batch_defer_plan_join": (st, [vp, C.c_int]),
        "hps_batch_join_plan": (st, [vp, vp]),
        "hps_batch_push": (st, [vp, vp, f32, u32, u32, C.c_int, vp, C.POINTER(C.c_int), u32, vp]),
        "hps_batch_pairs": (st, [vp, C.POINTER(u64)]),
        "hps_pull_batch": (st, [vp, vp, sz, vp, u32, u32, i32, vp, vp, vp]),
        "hps_push_batch": (st, [vp, vp, sz, vp, u32, u32, i32, vp, vp, vp, f32, u32, u32,
                                C.POINTER(C.c_int), vp]),
        "hps_launch_count": (u64, []),
        "hps_profile_enable": (st, [vp, C.c_int]),
        "hps_profile_get": (st, [vp, C.c_char_p, C.POINTER(C.c_double), C.POINTER(u64)]),
        "hps_dedup": (st, [vp, sz, vp, vp, C.POINTER(u64), vp]),
        "hps_compress_indices": (st, [vp, sz, vp, u32, u32, vp, vp, vp, vp, vp]),
        "hps_exchange_create": (st, [u32, u32, i32, i32, C.POINTER(vp)]),
        "hps_exchange_destroy": (st, [vp]),
        "hps_exchange_route": (st, [vp, vp, sz, vp, u32, u32, vp, vp, vp]),
        "hps_exchange_pool": (st, [vp, vp, u32, vp, vp]),
        "hps_exchange_pairs": (st, [vp, vp, u32, vp, vp, vp, vp]),
        "hps_exchange_arena": (st, [vp, u64, u64, u32, vp]),
        "hps_exchange_set_codec": (st, [vp, f32]),
        "hps_exchange_pooled": (st, [vp, C.POINTER(vp)]),
        "hps_exchange_connect": (st, [vp, u32, vp]),
        "hps_exchange_forward": (st, [vp, vp, vp, sz, vp, u32, u32, vp]),
        "hps_exchange_prefetch": (st, [vp, vp, vp, sz, vp, u32, u32, vp]),
        "hps_exchange_forward_prefetched": (st, [vp, vp, vp]),
        "hps_exchange_backward": (st, [vp, vp, vp, f32, u32, u32, C.POINTER(C.c_int), u32, vp]),
        "hps_table_apply_pairs": (st, [vp, vp, vp, C.POINTER(u64), vp, vp, C.POINTER(u64), u32,
                                       f32, u32, u32, C.POINTER(C.c_int), u32, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(rc: int, what: str = ""):
    if rc:
        msg = lib().hps_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, Error)(f"{what}: {msg}" if what else msg)


# ---- buffer helpers ------------------------------------------------------------------


def _ptr(a):
    """Raw pointer of a numpy array or torch tensor (None passes through)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch.Tensor


def _is_np(a):
    return isinstance(a, np.ndarray)


def _host(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream  # torch.cuda.Stream


def _like(x, shape, np_dtype, torch_dtype=None):
    """Output buffer on the same side as x (numpy host or torch device)."""
    if x is None or _is_np(x):
        return np.zeros(shape, np_dtype)
    import torch

    return torch.empty(shape, dtype=torch_dtype, device=x.device)


def _prep(a, np_dtype):
    if a is None:
        return None
    if _is_np(a) or isinstance(a, (list, tuple)):
        return _host(a, np_dtype)
    return a.contiguous()


# ---- free functions ------------------------------------------------------------------


def launch_count() -> int:
    """Kernels libhps.so has launched in this process."""
    return int(lib().hps_launch_count())


def mix64(x: int) -> int:
    return int(lib().hps_mix64(x & 0xFFFFFFFFFFFFFFFF))


def route_shard(id_: int, shard_count: int) -> int:
    if shard_count == 0:
        raise PreconditionError("route_shard: shard_count must be positive")
    return int(lib().hps_route_shard(id_ & 0xFFFFFFFFFFFFFFFF, shard_count))


def route(ids, shard_count: int, stream=None):
    ids = _prep(ids, np.uint64)
    out = _like(ids, (len(ids),), np.uint32, None if _is_np(ids) else __import__("torch").int32)
    check(lib().hps_route(_ptr(ids), len(ids), shard_count, _ptr(out), _stream_ptr(stream)),
          "route")
    return out


def dedup(ids, stream=None):
    """Sorted unique ids + inverse index (compress_indices semantics on a flat list)."""
    ids = _prep(ids, np.uint64)
    n = len(ids)
    if _is_np(ids):
        uniq = np.zeros(max(n, 1), np.uint64)
        inv = np.zeros(max(n, 1), np.uint32)
    else:
        import torch

        uniq = torch.empty(max(n, 1), dtype=torch.int64, device=ids.device)
        inv = torch.empty(max(n, 1), dtype=torch.int32, device=ids.device)
    u = C.c_uint64(0)
    check(lib().hps_dedup(_ptr(ids), n, _ptr(uniq), _ptr(inv), C.byref(u), _stream_ptr(stream)),
          "dedup")
    return uniq[: u.value], inv[:n]


KAPPA = 1024.0  # kDefaultKappa codec.hpp:214


def compress_values(values, kappa: float = KAPPA, stream=None):
    """compress_values (codec.hpp:222-241) per row of a [rows, block_len] f32 array ->
    (scales [rows] f32, payload [rows, block_len] u16 binary16 bits). numpy in -> numpy out;
    a torch CUDA tensor in -> torch outputs on the device."""
    v = _prep(values, np.float32)
    rows, blen = (v.shape[0], int(np.prod(v.shape[1:]))) if v.ndim > 1 else (1, v.shape[0])
    if _is_np(v):
        scales = np.zeros(rows, np.float32)
        payload = np.zeros((rows, blen), np.uint16)
    else:
        import torch

        scales = torch.empty(rows, dtype=torch.float32, device=v.device)
        payload = torch.empty((rows, blen), dtype=torch.int16, device=v.device)
    check(lib().hps_compress_values(_ptr(v), rows, blen, kappa, _ptr(scales), _ptr(payload),
                                    _stream_ptr(stream)), "compress_values")
    return scales, payload


def decompress_values(scales, payload, stream=None):
    """decompress_values (codec.hpp:244-261) -> [rows, block_len] f32."""
    if _is_np(payload):
        payload = np.ascontiguousarray(payload, np.uint16)
        scales = np.ascontiguousarray(scales, np.float32)
        out = np.zeros(payload.shape, np.float32)
    else:
        import torch

        out = torch.empty(payload.shape, dtype=torch.float32, device=payload.device)
    rows = payload.shape[0]
    blen = int(np.prod(payload.shape[1:]))
    check(lib().hps_decompress_values(_ptr(scales), _ptr(payload), rows, blen, _ptr(out),
                                      _stream_ptr(stream)), "decompress_values")
    return out


def compress_indices(ids, offsets, B: int, G: int, stream=None):
    """codec.hpp:123-156. Returns [(unique_ids, [postings...]) per group] (host)."""
    ids = _host(ids, np.uint64)
    offsets = _host(offsets, np.uint32)
    n = len(ids)
    gu = np.zeros(G + 1, np.uint64)
    un = np.zeros(max(n, 1), np.uint64)
    po = np.zeros(n + 1, np.uint64)
    ps = np.zeros(max(n, 1), np.uint16)
    check(lib().hps_compress_indices(_ptr(ids), n, _ptr(offsets), B, G, _ptr(gu), _ptr(un),
                                     _ptr(po), _ptr(ps), _stream_ptr(stream)), "compress_indices")
    out = []
    for g in range(G):
        a, b = int(gu[g]), int(gu[g + 1])
        out.append((un[a:b].copy(), [ps[int(po[k]):int(po[k + 1])].copy() for k in range(a, b)]))
    return out


# ---- the table (ShardSet / PsShard) ---------------------------------------------------


class ShardSet:
    """S logical shards (per-shard init salts) held on one device.

    ``tag_ring`` (default, like PsShard): exact staleness delays for any step-tag order
    (HPS_TABLE_TAG_RING); ``tag_ring=False`` keeps only each row's latest bump tag -- the
    in-order pipelines' choice, one store per row cheaper -- and refuses (ClockError) the
    tracked applies it could not count exactly.

    ``lru_shard_capacity`` > 0: every logical shard holds at most that many rows and evicts
    its least-recently-used one on a miss (PsShardConfig::capacity + LruStore; PS surface
    only, HPS_TABLE_LRU). ``capacity`` is then ignored.

    ``salts`` follows one of the reference's conventions, e.g.
    ``ShardSet(S, base_salt)`` -> ``salts[i] = mix64(base_salt + i)``
    (embedding_ps.hpp:513); pass ``salts=`` to use explicit per-shard salts.
    """

    def __init__(self, shard_count: int, embedding_dim: int, capacity: int,
                 optimizer: int = ADAGRAD, base_salt: int = 0, salts=None, device: int = -1,
                 owner_rank: int = 0, world_size: int = 1, tag_ring: bool = True,
                 lru_shard_capacity: int = 0):
        if salts is None:
            salts = [mix64((base_salt + i) & 0xFFFFFFFFFFFFFFFF) for i in range(shard_count)]
        self._salts = np.ascontiguousarray(salts, dtype=np.uint64)
        cfg = TableCfg(len(self._salts), self._salts.ctypes.data_as(C.POINTER(C.c_uint64)),
                       capacity, embedding_dim, optimizer, device, owner_rank, world_size,
                       (TABLE_TAG_RING if tag_ring else 0) |
                       (TABLE_LRU if lru_shard_capacity else 0), 0, lru_shard_capacity)
        h = vp()
        check(lib().hps_table_create(C.byref(cfg), C.byref(h)), "ShardSet")
        self.h = h
        self.embedding_dim = embedding_dim
        self.shard_count = len(self._salts)
        self.capacity = capacity
        self.optimizer = optimizer

    def close(self):
        if getattr(self, "h", None):
            lib().hps_table_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def shard_of(self, id_: int) -> int:
        return route_shard(id_, self.shard_count)

    # counters / epochs (embedding_ps.hpp:75-98, 193-207)
    def counters(self) -> Counters:
        c = Counters()
        check(lib().hps_table_counters(self.h, C.byref(c)), "counters")
        return c

    def miss_count(self) -> int:
        return self.counters().misses

    def size(self) -> int:
        return self.counters().size

    def stale_epoch_drops(self) -> int:
        return self.counters().stale_epoch_drops

    def eviction_count(self) -> int:
        return self.counters().evictions

    def clock_reset_count(self) -> int:
        return self.counters().clock_resets

    def epoch(self) -> int:
        return int(lib().hps_table_epoch(self.h))

    def device_step(self) -> int:
        """Steps pushed with DEVICE_STEP so far (the table's device step counter)."""
        v = C.c_uint32(0)
        check(lib().hps_table_device_step(self.h, C.byref(v)), "device_step")
        return v.value

    def advance_epoch(self) -> int:
        return int(lib().hps_table_advance_epoch(self.h))

    def reset_for_recovery(self):
        check(lib().hps_table_reset(self.h), "reset_for_recovery")

    def sync(self):
        check(lib().hps_table_sync(self.h), "sync")

    # PsShard::save_checkpoint (embedding_ps.hpp:222-260), per logical shard
    def save_checkpoint(self, shard: int = 0, shard_capacity: int = 0) -> bytes:
        n = C.c_uint64(0)
        check(lib().hps_table_checkpoint_save(self.h, shard, shard_capacity, None, 0,
                                              C.byref(n)), "save_checkpoint")
        buf = (C.c_uint8 * max(n.value, 1))()
        check(lib().hps_table_checkpoint_save(self.h, shard, shard_capacity, buf, n.value,
                                              C.byref(n)), "save_checkpoint")
        return bytes(buf)[:n.value]

    # PsShard::load_checkpoint / recover_from_checkpoint (:262-300) for the whole table
    def load_checkpoint(self, images, recover: bool = False):
        images = [bytes(im) for im in images]
        bufs = [C.create_string_buffer(im, len(im)) for im in images]
        ptrs = (vp * max(len(bufs), 1))(*[C.cast(b, vp) for b in bufs])
        sizes = (C.c_uint64 * max(len(bufs), 1))(*[len(im) for im in images])
        check(lib().hps_table_checkpoint_load(self.h, ptrs, sizes, len(images), int(recover)),
              "load_checkpoint")

    def profile(self, enable: bool = True):
        check(lib().hps_profile_enable(self.h, int(enable)), "profile")

    def profile_get(self, region: str):
        """(total_ms, count) of a named region since profile(True)."""
        ms = C.c_double(0)
        n = C.c_uint64(0)
        check(lib().hps_profile_get(self.h, region.encode(), C.byref(ms), C.byref(n)),
              "profile_get")
        return ms.value, n.value

    # PsShard::lookup
    def lookup(self, ids, out_values=None, out_versions=None, stream=None):
        ids = _prep(ids, np.uint64)
        n = len(ids)
        D = self.embedding_dim
        if out_values is None:
            out_values = _like(ids, (n, D), np.float32,
                               None if _is_np(ids) else __import__("torch").float32)
        if out_versions is None and _is_np(ids):
            out_versions = np.zeros(n, np.uint64)
        check(lib().hps_lookup(self.h, _ptr(ids), n, _ptr(out_values), _ptr(out_versions),
                               _stream_ptr(stream)), "lookup")
        return out_values, out_versions

    def lookup_map(self, ids) -> dict:
        vals, _ = self.lookup(ids)
        return {int(i): vals[k].copy() for k, i in enumerate(np.asarray(ids, np.uint64))}

    # PsShard::apply_gradients (tracked) -> (accepted, delays)
    def apply_gradients(self, ids, grads, read_versions, lr: float, step_tag: int,
                        caller_epoch: int | None = None, want_delays: bool = True, stream=None):
        ids = _prep(ids, np.uint64)
        grads = _prep(grads, np.float32)
        rv = _prep(read_versions, np.uint64)
        n = len(ids)
        delays = np.zeros(n, np.uint32) if want_delays else None
        acc = C.c_int(0)
        epoch = self.epoch() if caller_epoch is None else caller_epoch
        check(lib().hps_apply(self.h, _ptr(ids), _ptr(grads), _ptr(rv), n, lr, step_tag, epoch,
                              _ptr(delays), C.byref(acc), 0, _stream_ptr(stream)),
              "apply_gradients")
        return bool(acc.value), delays

    # PsShard::apply_gradients_map (untracked)
    def apply_gradients_map(self, grads: dict, lr: float):
        ids = np.array(sorted(grads), np.uint64)
        g = np.stack([np.asarray(grads[int(i)], np.float32) for i in ids]) if len(ids) else \
            np.zeros((0, self.embedding_dim), np.float32)
        if g.shape[1:] != (self.embedding_dim,):
            raise PreconditionError("apply_gradients: gradient width mismatch")
        acc = C.c_int(0)
        check(lib().hps_apply(self.h, _ptr(ids), _ptr(np.ascontiguousarray(g)), None, len(ids),
                              lr, 0, self.epoch(), None, C.byref(acc), 0, None),
              "apply_gradients_map")

    def peek(self, ids):
        """(w, acc, versions, present) without initialising or touching rows."""
        ids = _host(ids, np.uint64)
        n = len(ids)
        D = self.embedding_dim
        w = np.zeros((n, D), np.float32)
        a = np.zeros((n, D), np.float32)
        v = np.zeros(n, np.uint64)
        p = np.zeros(n, np.uint8)
        check(lib().hps_peek(self.h, _ptr(ids), n, _ptr(w), _ptr(a), _ptr(v), _ptr(p), None),
              "peek")
        return w, a, v, p.astype(bool)


# ---- the embedding worker (batch granularity) -------------------------------------------


class EmbeddingWorker:
    """EmbeddingWorker (embedding_worker.hpp:470) over one device table, batch-shaped.

    ``register_batch`` buffers a CSR batch (B samples x F groups); ``serve_pull``
    returns pooled embeddings [B, F, D] (+ per-listing read versions);
    ``apply_backward`` applies per-sample gradients [B, F, D] in ascending sample-key
    order (sync / gated-flush semantics).
    """

    def __init__(self, table: ShardSet, aggregation: int = MEAN):
        self.table = table
        self.aggregation = aggregation
        h = vp()
        check(lib().hps_batch_create(table.h, aggregation, C.byref(h)), "EmbeddingWorker")
        self.h = h
        self.B = self.F = self.N = 0

    def close(self):
        if getattr(self, "h", None):
            lib().hps_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def register_batch(self, ids, offsets, B: int, F: int, sample_keys=None, stream=None):
        ids = _prep(ids, np.uint64)
        offsets = _prep(offsets, np.uint32)
        sk = _prep(sample_keys, np.uint64)
        self.B, self.F, self.N = B, F, len(ids)
        self._keep = (ids, offsets, sk)
        check(lib().hps_batch_register(self.h, _ptr(ids), len(ids), _ptr(offsets), B, F, _ptr(sk),
                                       _stream_ptr(stream)), "register_batch")

    def defer_plan_join(self, on: bool = True):
        """Join this batch's plan (its sort) at the push instead of the register / pull
        (hps_batch_defer_plan_join): for pipelines that register the next batch beside
        the current step. Under graph capture, a capture that ends before the push must
        call join_plan on one of its streams."""
        check(lib().hps_batch_defer_plan_join(self.h, int(on)), "defer_plan_join")

    def join_plan(self, stream=None):
        check(lib().hps_batch_join_plan(self.h, _stream_ptr(stream)), "join_plan")

    def serve_pull(self, out_pooled=None, out_read_versions=None, stream=None, like=None):
        D = self.table.embedding_dim
        if out_pooled is None:
            ref = like if like is not None else (self._keep[0] if hasattr(self, "_keep") else None)
            out_pooled = _like(ref, (self.B, self.F, D), np.float32,
                               None if ref is None or _is_np(ref) else __import__("torch").float32)
        check(lib().hps_batch_pull(self.h, _ptr(out_pooled), _ptr(out_read_versions),
                                   _stream_ptr(stream)), "serve_pull")
        return out_pooled

    def apply_backward(self, grads, lr: float, step_tag: int = 0, epoch: int | None = None,
                       untracked: bool = False, flags: int = 0, stream=None) -> bool:
        grads = _prep(grads, np.float32)
        acc = C.c_int(0)
        e = self.table.epoch() if epoch is None else epoch
        check(lib().hps_batch_push(self.h, _ptr(grads), lr, step_tag, e, int(untracked), None,
                                   C.byref(acc), flags, _stream_ptr(stream)), "apply_backward")
        return bool(acc.value)

    def pairs(self) -> int:
        p = C.c_uint64(0)
        check(lib().hps_batch_pairs(self.h, C.byref(p)), "pairs")
        return p.value
