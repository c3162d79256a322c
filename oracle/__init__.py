"""Parity oracle for the embedding hot path -- TEST INFRASTRUCTURE ONLY.

Two CPU implementations live here, both loaded through ctypes:

* ``Restatement`` -- ``build/libhps_oracle.so``, the plain-C restatement of the
  reference algorithm (``hps_oracle.c``; every function cites the reference
  file:line it restates).
* ``Reference`` -- ``_ref/libhps_ref.so``, the UNMODIFIED reference headers
  (``/root/reference/proj/include``) compiled by ``oracle/Makefile`` and driven
  through ``ref_driver.cpp``: S ``PsShard`` behind ``PsShardService`` on a
  ``LocalHub`` with E ``EmbeddingWorker`` in front, sync (staleness-0) order.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference /
cpu_baseline legs may import this package. The product library never does.
"""
from __future__ import annotations

import ctypes as C
import os
import struct

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.environ.get('HPS_ORACLE_SO', os.path.join(HERE, 'build', 'libhps_oracle.so'))
REFERENCE_SO = os.path.join(HERE, "_ref", "libhps_ref.so")

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
u16p = C.POINTER(C.c_uint16)
f32p = C.POINTER(C.c_float)
u8p = C.POINTER(C.c_uint8)
intp = C.POINTER(C.c_int)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _u64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.uint64)


def _f32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float32)


_lib_cache: dict = {}


def _load(path: str):
    if path not in _lib_cache:
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run `make -C oracle` (or __graft_entry__.build())")
        _lib_cache[path] = C.CDLL(path)
    return _lib_cache[path]


def restatement_lib():
    lib = _load(RESTATEMENT_SO)
    if not getattr(lib, "_typed", False):
        lib.orc_mix64.restype = C.c_uint64
        lib.orc_mix64.argtypes = [C.c_uint64]
        lib.orc_route_shard.restype = C.c_uint32
        lib.orc_route_shard.argtypes = [C.c_uint64, C.c_uint32]
        lib.orc_init_row.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, f32p]
        lib.orc_table_create.restype = C.c_void_p
        lib.orc_table_create.argtypes = [C.c_uint32, u64p, C.c_uint32, C.c_int]
        lib.orc_table_destroy.argtypes = [C.c_void_p]
        lib.orc_table_epoch.restype = C.c_uint32
        lib.orc_table_epoch.argtypes = [C.c_void_p]
        lib.orc_table_advance_epoch.restype = C.c_uint32
        lib.orc_table_advance_epoch.argtypes = [C.c_void_p]
        lib.orc_table_counters.argtypes = [C.c_void_p, u64p]
        lib.orc_lookup.argtypes = [C.c_void_p, u64p, C.c_size_t, f32p, u64p]
        lib.orc_peek.argtypes = [C.c_void_p, u64p, C.c_size_t, f32p, f32p, u64p, u8p]
        lib.orc_apply.restype = C.c_int
        lib.orc_apply.argtypes = [C.c_void_p, u64p, f32p, u64p, C.c_size_t, C.c_float,
                                  C.c_uint32, C.c_uint32, u32p, intp]
        lib.orc_apply_map.restype = C.c_int
        lib.orc_apply_map.argtypes = [C.c_void_p, u64p, f32p, C.c_size_t, C.c_float]
        lib.orc_pull_batch.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, u64p, u64p, C.c_int,
                                       f32p, u64p]
        lib.orc_push_batch.restype = C.c_int
        lib.orc_push_batch.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, u64p, u64p, C.c_int,
                                       f32p, u64p, u64p, C.c_float, C.c_uint32, C.c_uint32,
                                       u32p, u64p, intp]
        lib.orc_compress_indices.restype = C.c_int
        lib.orc_compress_indices.argtypes = [C.c_uint32, C.c_uint32, u64p, u64p, u64p, u64p,
                                             u64p, u16p]
        lib._typed = True
    return lib


def reference_lib():
    lib = _load(REFERENCE_SO)
    if not getattr(lib, "_typed", False):
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_mix64.restype = C.c_uint64
        lib.ref_mix64.argtypes = [C.c_uint64]
        lib.ref_route_shard.restype = C.c_uint32
        lib.ref_route_shard.argtypes = [C.c_uint64, C.c_uint32]
        lib.ref_table_create.restype = C.c_void_p
        lib.ref_table_create.argtypes = [C.c_uint32, u64p, C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                                         C.c_uint32, C.c_uint32, C.c_uint64, C.c_int]
        lib.ref_table_destroy.argtypes = [C.c_void_p]
        lib.ref_step.restype = C.c_int
        lib.ref_step.argtypes = [C.c_void_p, C.c_uint32, u64p, u64p, f32p, C.c_float, C.c_uint64,
                                 C.c_int, C.c_int, C.c_int, f32p, u64p, u64p]
        lib.ref_set_epoch.argtypes = [C.c_void_p, C.c_uint32]
        lib.ref_shard_lookup.restype = C.c_int
        lib.ref_shard_lookup.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, u64p, f32p, u64p]
        lib.ref_shard_apply.restype = C.c_int
        lib.ref_shard_apply.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, u64p, f32p, u64p,
                                        C.c_float, C.c_uint32, C.c_uint32, u32p, intp]
        lib.ref_shard_apply_map.restype = C.c_int
        lib.ref_shard_apply_map.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, u64p, f32p,
                                            C.c_float]
        lib.ref_shard_counters.restype = C.c_int
        lib.ref_shard_counters.argtypes = [C.c_void_p, C.c_uint32, u64p]
        lib.ref_shard_advance_epoch.restype = C.c_uint32
        lib.ref_shard_advance_epoch.argtypes = [C.c_void_p, C.c_uint32]
        lib.ref_shard_export.restype = C.c_int64
        lib.ref_shard_export.argtypes = [C.c_void_p, C.c_uint32, u8p, C.c_uint64]
        lib.ref_compress_indices.restype = C.c_int
        lib.ref_compress_indices.argtypes = [C.c_uint32, C.c_uint32, u64p, u64p, u64p, u64p, u64p,
                                             u16p]
        lib.ref_shard_import.restype = C.c_int
        lib.ref_shard_import.argtypes = [C.c_void_p, C.c_uint32, u8p, C.c_uint64, C.c_int]
        lib.ref_compress_values.restype = C.c_int
        lib.ref_compress_values.argtypes = [f32p, C.c_uint64, C.c_uint32, C.c_float, f32p, u16p]
        lib.ref_decompress_values.restype = C.c_int
        lib.ref_decompress_values.argtypes = [f32p, u16p, C.c_uint64, C.c_uint32, f32p]
        lib.ref_dense_init.restype = C.c_int64
        lib.ref_dense_init.argtypes = [u64p, C.c_uint32, C.c_uint64, f32p, C.c_uint64]
        lib.ref_dense_fwd_bwd.restype = C.c_int
        lib.ref_dense_fwd_bwd.argtypes = [u64p, C.c_uint32, f32p, C.c_uint32, f32p, f32p, f32p,
                                          f32p, f32p, f32p]
        lib.ref_allreduce.restype = C.c_int
        lib.ref_allreduce.argtypes = [C.c_uint32, C.c_uint64, f32p, f32p]
        lib.ref_sgd_step.restype = C.c_int
        lib.ref_sgd_step.argtypes = [f32p, f32p, C.c_uint64, C.c_float]
        lib._typed = True
    return lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


# ----------------------------------------------------------------------------- restatement


class Restatement:
    """The C restatement: one table of S logical shards (salts per shard)."""

    def __init__(self, salts, dim: int, optimizer: str = "adagrad"):
        self.lib = restatement_lib()
        self.salts = _u64(salts)
        self.S = len(self.salts)
        self.D = dim
        self.h = self.lib.orc_table_create(self.S, _p(self.salts, u64p), dim,
                                           0 if optimizer == "adagrad" else 1)
        if not self.h:
            raise OracleError(2, "bad config")

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_table_destroy(self.h)
            self.h = None

    @property
    def epoch(self) -> int:
        return self.lib.orc_table_epoch(self.h)

    def advance_epoch(self) -> int:
        return self.lib.orc_table_advance_epoch(self.h)

    def counters(self) -> dict:
        o = np.zeros(4, np.uint64)
        self.lib.orc_table_counters(self.h, _p(o, u64p))
        return dict(misses=int(o[0]), clock_resets=int(o[1]), stale_epoch_drops=int(o[2]),
                    size=int(o[3]))

    def lookup(self, ids):
        ids = _u64(ids)
        out = np.zeros((len(ids), self.D), np.float32)
        ver = np.zeros(len(ids), np.uint64)
        self.lib.orc_lookup(self.h, _p(ids, u64p), len(ids), _p(out, f32p), _p(ver, u64p))
        return out, ver

    def peek(self, ids):
        ids = _u64(ids)
        n = len(ids)
        w = np.zeros((n, self.D), np.float32)
        a = np.zeros((n, self.D), np.float32)
        v = np.zeros(n, np.uint64)
        pr = np.zeros(n, np.uint8)
        self.lib.orc_peek(self.h, _p(ids, u64p), n, _p(w, f32p), _p(a, f32p), _p(v, u64p),
                          _p(pr, u8p))
        return w, a, v, pr.astype(bool)

    def apply(self, ids, grads, read_versions, lr, step_tag, epoch=None):
        ids = _u64(ids)
        grads = _f32(grads)
        rv = _u64(read_versions)
        dl = np.zeros(len(ids), np.uint32)
        acc = C.c_int(0)
        rc = self.lib.orc_apply(self.h, _p(ids, u64p), _p(grads, f32p), _p(rv, u64p), len(ids),
                                lr, step_tag, self.epoch if epoch is None else epoch,
                                _p(dl, u32p), C.byref(acc))
        if rc:
            raise OracleError(rc, "apply")
        return bool(acc.value), dl

    def apply_map(self, ids, grads, lr):
        ids = _u64(ids)
        grads = _f32(grads)
        rc = self.lib.orc_apply_map(self.h, _p(ids, u64p), _p(grads, f32p), len(ids), lr)
        if rc:
            raise OracleError(rc, "apply_map")

    def pull_batch(self, B, F, ids, offsets, agg="mean"):
        ids = _u64(ids)
        offsets = _u64(offsets)
        pooled = np.zeros((B, F, self.D), np.float32)
        rv = np.zeros(len(ids), np.uint64)
        self.lib.orc_pull_batch(self.h, B, F, _p(ids, u64p), _p(offsets, u64p),
                                0 if agg == "mean" else 1, _p(pooled, f32p), _p(rv, u64p))
        return pooled, rv

    def push_batch(self, B, F, ids, offsets, grads, lr, step_tag=0, read_versions=None,
                   sample_keys=None, agg="mean", epoch=None):
        ids = _u64(ids)
        offsets = _u64(offsets)
        grads = _f32(grads)
        rv = _u64(read_versions)
        sk = _u64(sample_keys)
        dl = np.zeros(max(1, len(ids)), np.uint32)
        nd = C.c_uint64(0)
        acc = C.c_int(0)
        rc = self.lib.orc_push_batch(self.h, B, F, _p(ids, u64p), _p(offsets, u64p),
                                     0 if agg == "mean" else 1, _p(grads, f32p), _p(rv, u64p),
                                     _p(sk, u64p), lr, step_tag,
                                     self.epoch if epoch is None else epoch, _p(dl, u32p),
                                     C.byref(nd), C.byref(acc))
        if rc:
            raise OracleError(rc, "push_batch")
        return bool(acc.value), dl[: nd.value]


def mix64(x: int) -> int:
    return int(restatement_lib().orc_mix64(x))


def route_shard(x: int, s: int) -> int:
    return int(restatement_lib().orc_route_shard(x, s))


def init_row(id_: int, salt: int, dim: int) -> np.ndarray:
    out = np.zeros(dim, np.float32)
    restatement_lib().orc_init_row(id_, salt, dim, _p(out, f32p))
    return out


def compress_indices(B, G, ids, offsets, lib: str = "restatement"):
    """Returns list over groups of (unique_ids[u], postings list of arrays)."""
    ids = _u64(ids)
    offsets = _u64(offsets)
    N = max(1, len(ids))
    gu = np.zeros(G + 1, np.uint64)
    un = np.zeros(N, np.uint64)
    po = np.zeros(N + 1, np.uint64)
    ps = np.zeros(N, np.uint16)
    if lib == "restatement":
        rc = restatement_lib().orc_compress_indices(B, G, _p(ids, u64p), _p(offsets, u64p),
                                                    _p(gu, u64p), _p(un, u64p), _p(po, u64p),
                                                    _p(ps, u16p))
    else:
        rc = reference_lib().ref_compress_indices(B, G, _p(ids, u64p), _p(offsets, u64p),
                                                  _p(gu, u64p), _p(un, u64p), _p(po, u64p),
                                                  _p(ps, u16p))
    if rc:
        raise OracleError(rc, "compress_indices")
    return unpack_compressed(G, gu, un, po, ps)


def unpack_compressed(G, gu, un, po, ps):
    out = []
    for g in range(G):
        a, b = int(gu[g]), int(gu[g + 1])
        uniq = np.array(un[a:b], np.uint64)
        posts = [np.array(ps[int(po[k]):int(po[k + 1])], np.uint16) for k in range(a, b)]
        out.append((uniq, posts))
    return out


# ----------------------------------------------------------------------------- reference


class Reference:
    """The reference's own path (headers compiled in oracle/_ref)."""

    def __init__(self, salts, capacity, dim, optimizer="adagrad", agg="mean", groups=1,
                 workers=1, ew_buffer=0, compress=False):
        self.lib = reference_lib()
        self.salts = _u64(salts)
        self.S = len(self.salts)
        self.D = dim
        self.F = groups
        self.h = self.lib.ref_table_create(self.S, _p(self.salts, u64p), capacity, dim,
                                           0 if optimizer == "adagrad" else 1,
                                           0 if agg == "mean" else 1, groups, workers, ew_buffer,
                                           int(compress))
        if not self.h:
            raise OracleError(2, self.lib.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_table_destroy(self.h)
            self.h = None

    def _check(self, rc, what):
        if rc:
            raise OracleError(rc, f"{what}: {self.lib.ref_last_error().decode()}")

    def step(self, B, ids, offsets, grads=None, lr=0.0, step=0, has_step=False, threads=1,
             pull=True, push=True, push_threads=False):
        ids = _u64(ids)
        offsets = _u64(offsets)
        grads = _f32(grads)
        pooled = np.zeros((B, self.F, self.D), np.float32) if pull else None
        rv = np.zeros(max(1, len(ids)), np.uint64) if pull else None
        sids = np.zeros(B, np.uint64) if pull else None
        # push_threads: the hybrid push, apply_backward from `threads` threads at once
        flags = (1 if pull else 0) | ((4 if push_threads else 2) if push else 0)
        rc = self.lib.ref_step(self.h, B, _p(ids, u64p), _p(offsets, u64p), _p(grads, f32p), lr,
                               step, int(has_step), threads, flags, _p(pooled, f32p),
                               _p(rv, u64p), _p(sids, u64p))
        self._check(rc, "step")
        return pooled, (rv[: len(ids)] if rv is not None else None), sids

    def set_epoch(self, e):
        self.lib.ref_set_epoch(self.h, e)

    def shard_lookup(self, s, ids):
        ids = _u64(ids)
        out = np.zeros((len(ids), self.D), np.float32)
        ver = np.zeros(len(ids), np.uint64)
        self._check(self.lib.ref_shard_lookup(self.h, s, len(ids), _p(ids, u64p), _p(out, f32p),
                                              _p(ver, u64p)), "lookup")
        return out, ver

    def shard_apply(self, s, ids, grads, read_versions, lr, step_tag, epoch):
        ids = _u64(ids)
        grads = _f32(grads)
        rv = _u64(read_versions)
        dl = np.zeros(len(ids), np.uint32)
        acc = C.c_int(0)
        self._check(self.lib.ref_shard_apply(self.h, s, len(ids), _p(ids, u64p), _p(grads, f32p),
                                             _p(rv, u64p), lr, step_tag, epoch, _p(dl, u32p),
                                             C.byref(acc)), "apply")
        return bool(acc.value), dl

    def shard_apply_map(self, s, ids, grads, lr):
        ids = _u64(ids)
        grads = _f32(grads)
        self._check(self.lib.ref_shard_apply_map(self.h, s, len(ids), _p(ids, u64p),
                                                 _p(grads, f32p), lr), "apply_map")

    def shard_counters(self, s):
        o = np.zeros(6, np.uint64)
        self._check(self.lib.ref_shard_counters(self.h, s, _p(o, u64p)), "counters")
        return dict(misses=int(o[0]), evictions=int(o[1]), clock_resets=int(o[2]),
                    stale_epoch_drops=int(o[3]), epoch=int(o[4]), size=int(o[5]))

    def shard_export(self, s) -> bytes:
        n = self.lib.ref_shard_export(self.h, s, None, 0)
        if n < 0:
            self._check(-n, "export")
        buf = np.zeros(n, np.uint8)
        self.lib.ref_shard_export(self.h, s, _p(buf, u8p), n)
        return buf.tobytes()

    def shard_import(self, s, image: bytes, validate_only: bool = False):
        """recover_from_checkpoint (embedding_ps.hpp:280-292) of shard s from an HPS1 image
        (validate_only: PsShard::load_checkpoint into a discarded shard)."""
        buf = np.frombuffer(image, np.uint8).copy()
        self._check(self.lib.ref_shard_import(self.h, s, _p(buf, u8p), len(buf),
                                              int(validate_only)), "shard_import")

    def state(self):
        """{id: (w[D], acc[D], version)} over every shard, from HPS1 images."""
        out = {}
        for s in range(self.S):
            out.update(parse_hps1(self.shard_export(s))["rows"])
        return out


def parse_hps1(buf: bytes) -> dict:
    """Parse an HPS1 checkpoint image (embedding_ps.hpp:211-260 layout)."""
    assert buf[:4] == b"HPS1", "bad magic"
    dim, cap = struct.unpack_from("<II", buf, 8)
    (salt,) = struct.unpack_from("<Q", buf, 16)
    hwm, head, tail, free_head, live, epoch = struct.unpack_from("<6I", buf, 24)
    q = 64
    ids = np.frombuffer(buf, np.uint64, hwm, q)
    q += 8 * hwm
    prev = np.frombuffer(buf, np.uint32, hwm, q)
    q += 4 * hwm
    nxt = np.frombuffer(buf, np.uint32, hwm, q)
    q += 4 * hwm
    vers = np.frombuffer(buf, np.uint64, hwm, q)
    q += 8 * hwm
    rows = np.frombuffer(buf, np.float32, hwm * 2 * dim, q).reshape(hwm, 2 * dim)
    # Live slots: walk the recency chain from head.
    live_slots = []
    s = head
    while s != 0xFFFFFFFF and len(live_slots) < hwm:
        live_slots.append(s)
        s = int(nxt[s])
    res = {}
    for s in live_slots:
        res[int(ids[s])] = (rows[s, :dim].copy(), rows[s, dim:].copy(), int(vers[s]))
    return dict(dim=dim, capacity=cap, salt=salt, epoch=epoch, rows=res)


# ---- dense tower (the reference's DenseNet / AllReduceHub, C5) ---------------------------


def _ref_rc(rc, what):
    if rc:
        raise OracleError(rc, f"{what}: {reference_lib().ref_last_error().decode()}")


def ref_dense_init(dims, init_seed: int) -> np.ndarray:
    """DenseNet(dims, Rng(mix64(init_seed))) params (nn_worker.hpp:331-336)."""
    lib = reference_lib()
    d = _u64(np.asarray(dims))
    n = lib.ref_dense_init(_p(d, u64p), len(d), init_seed, None, 0)
    _ref_rc(0 if n >= 0 else -n, "dense_init")
    out = np.zeros(n, np.float32)
    lib.ref_dense_init(_p(d, u64p), len(d), init_seed, _p(out, f32p), n)
    return out


def ref_dense_fwd_bwd(dims, params, inputs, labels):
    """batch_forward_backward (dense_nn.hpp:218-246) -> (loss, probs, dense_grad, input_grads)."""
    lib = reference_lib()
    d = _u64(np.asarray(dims))
    params, inputs, labels = _f32(params), _f32(inputs), _f32(labels)
    B = len(labels)
    loss = C.c_float(0)
    probs = np.zeros(B, np.float32)
    dg = np.zeros(len(params), np.float32)
    ig = np.zeros((B, int(dims[0])), np.float32)
    _ref_rc(lib.ref_dense_fwd_bwd(_p(d, u64p), len(d), _p(params, f32p), B, _p(inputs, f32p),
                                  _p(labels, f32p), C.byref(loss), _p(probs, f32p), _p(dg, f32p),
                                  _p(ig, f32p)), "dense_fwd_bwd")
    return loss.value, probs, dg, ig


def ref_allreduce(parts) -> np.ndarray:
    """AllReduceHub canonical mean (nn_worker.hpp:214-226) of parts[K, n]."""
    parts = _f32(parts)
    K, n = parts.shape
    out = np.zeros(n, np.float32)
    _ref_rc(reference_lib().ref_allreduce(K, n, _p(parts, f32p), _p(out, f32p)), "allreduce")
    return out


def ref_sgd_step(params, grad, lr: float) -> np.ndarray:
    """sgd_step (dense_nn.hpp:263-273) on a copy of params."""
    p = _f32(params).copy()
    g = _f32(grad)
    _ref_rc(reference_lib().ref_sgd_step(_p(p, f32p), _p(g, f32p), len(p), lr), "sgd_step")
    return p


# ---- value codec (codec.hpp:30-103, 208-261) ---------------------------------------------


def ref_compress_values(v, kappa: float = 1024.0):
    """The reference's compress_values per row of v[rows, len] -> (scales, payload u16)."""
    v = _f32(np.atleast_2d(v))
    rows, n = v.shape
    sc = np.zeros(rows, np.float32)
    pl = np.zeros((rows, n), np.uint16)
    _ref_rc(reference_lib().ref_compress_values(_p(v, f32p), rows, n, kappa, _p(sc, f32p),
                                                _p(pl, u16p)), "compress_values")
    return sc, pl


def ref_decompress_values(scales, payload):
    sc = _f32(scales)
    pl = np.ascontiguousarray(np.atleast_2d(payload), np.uint16)
    out = np.zeros(pl.shape, np.float32)
    _ref_rc(reference_lib().ref_decompress_values(_p(sc, f32p), _p(pl, u16p), pl.shape[0],
                                                  pl.shape[1], _p(out, f32p)), "decompress_values")
    return out


def compress_values_np(v, kappa: float = 1024.0):
    """Restatement (numpy): scale = kappa / max|row| (1 for a zero row) in float32, payload =
    binary16 of v*scale (IEEE round-to-nearest-even with subnormals, as float_to_half_bits),
    an all-zero row -> +0 payload."""
    v = np.atleast_2d(np.asarray(v, np.float32))
    m = np.abs(v).max(axis=1)
    zero = m == 0
    scale = np.where(zero, np.float32(1.0), np.float32(kappa) / np.where(zero, 1, m)).astype(np.float32)
    pl = (v * scale[:, None]).astype(np.float16).view(np.uint16)
    pl[zero] = 0
    return scale, pl


def decompress_values_np(scales, payload):
    w = np.asarray(payload, np.uint16).view(np.float16).astype(np.float32)
    return (w / np.asarray(scales, np.float32)[:, None]).astype(np.float32)
