"""Synthetic Criteo-shaped batches for BASELINE.json's configs (host, numpy).

Every random quantity is drawn from the reference's own generator family -- the
splitmix stream of core.hpp:49-63 (draw k of Rng(seed) is mix64(seed + k*gamma)) --
so batches are reproducible bit-for-bit and identical for the GPU path, the oracle
and the reference arm. Feature groups own disjoint id ranges, as in
data.hpp:62-67. IDs are listed sorted and unique within a (sample, group), as
data.hpp:172-176 generates them (one-hot configs trivially satisfy this).

configs (BASELINE.json "configs"):
  c1  batch 1024, 8 one-hot features, 1M rows, D=16, sum, SGD          (parity / CPU run)
  c2  batch 16384, 26 one-hot features, 100M rows, D=64, Adagrad       (single B200 headline)
  c3  c2 shape, multi-hot avg 50 ids/feature (Poisson, clipped [1,100]), Zipf(1.1) ids
  c4  c2 shape per GPU over a 1B-row table hash-sharded across GPUs
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
MASK64 = 0xFFFFFFFFFFFFFFFF


def mix64(x) -> np.ndarray:
    """Vectorised mix64 (core.hpp:36-44)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + GAMMA
        x = x ^ (x >> np.uint64(30))
        x = x * M1
        x = x ^ (x >> np.uint64(27))
        x = x * M2
        x = x ^ (x >> np.uint64(31))
    return x


def mix64_int(x: int) -> int:
    return int(mix64(np.uint64(x & MASK64)))


def rng_stream(seed: int, n: int, start: int = 0) -> np.ndarray:
    """Draws start..start+n-1 of Rng(seed).next_u64() (core.hpp:53-57)."""
    k = np.arange(start, start + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(np.uint64(seed & MASK64) + k * GAMMA)


def uniform01(seed: int, n: int, start: int = 0) -> np.ndarray:
    return (rng_stream(seed, n, start) >> np.uint64(11)).astype(np.float64) * 2.0**-53


@dataclass
class Config:
    name: str
    batch: int
    features: int
    rows: int
    dim: int
    optimizer: str  # "adagrad" | "sgd"
    aggregation: str  # "mean" | "sum"
    multi_hot: float = 0.0  # mean ids per feature (0 = one-hot)
    zipf: float = 0.0  # Zipf exponent (0 = uniform)
    shards: int = 8
    lr: float = 0.05
    seed: int = 7
    grad_scale: float = 0.01
    capacity: int = 0  # 0 = rows

    @property
    def rows_per_feature(self) -> int:
        return self.rows // self.features

    def salts(self) -> list:
        # ShardSet convention (embedding_ps.hpp:513) with base salt = seed.
        return [mix64_int(self.seed + s) for s in range(self.shards)]

    def table_capacity(self) -> int:
        return self.capacity or self.rows_per_feature * self.features


CONFIGS = {
    "c1": Config("c1", 1024, 8, 1_000_000, 16, "sgd", "sum", shards=4,
                 capacity=4 * (1 << 20)),
    "c2": Config("c2", 16384, 26, 100_000_000, 64, "adagrad", "mean"),
    "c3": Config("c3", 16384, 26, 100_000_000, 64, "adagrad", "mean", multi_hot=50.0, zipf=1.1),
    "c4": Config("c4", 16384, 26, 1_000_000_000, 64, "adagrad", "mean"),
    # C5: the C2/C4 embedding shape + the dense tower (hybrid step); 13 Criteo dense
    # features; the reference NN worker's default hidden widths {64, 32}
    # (orchestrator.hpp:94) -> a 3-layer MLP (1677 -> 64 -> 32 -> 1).
    "c5": Config("c5", 16384, 26, 100_000_000, 64, "adagrad", "mean"),
}

C5_NON_ID = 13
C5_HIDDEN = (64, 32)
C5_STALENESS = 4


def sharded_config(world: int) -> Config:
    """C4 at `world` GPUs, weak-scaled: per-GPU batch 16384 of the C2 shape over a table
    of 125M rows per GPU (1B rows at 8 GPUs), S = 8 logical shards per GPU."""
    return Config("c4", 16384, 26, 125_000_000 * world, 64, "adagrad", "mean",
                  shards=8 * world)


@dataclass
class Batch:
    ids: np.ndarray  # uint64 [N]
    offsets: np.ndarray  # uint32 [B*F+1]
    B: int
    F: int
    meta: dict = field(default_factory=dict)

    @property
    def N(self) -> int:
        return int(self.offsets[-1])


def _feature_seed(cfg: Config, f: int) -> int:
    return mix64_int(cfg.seed ^ f)


def _zipf_ranks(seed: int, n: int, s: float, n_items: int, start: int) -> np.ndarray:
    """Rejection-inversion Zipf sampler (Hormann & Derflinger 1996) over ranks
    1..n_items, driven by the splitmix uniform stream; O(1) memory in n_items."""
    one_m_s = 1.0 - s

    def H(x):
        return (np.power(x, one_m_s) - 1.0) / one_m_s

    def H_inv(y):
        return np.power(1.0 + one_m_s * y, 1.0 / one_m_s)

    def h(x):
        return np.power(x, -s)

    hx1 = H(1.5) - 1.0
    hN = H(n_items + 0.5)
    s_thr = 2.0 - H_inv(H(2.5) - h(2.0))
    out = np.zeros(n, np.int64)
    todo = np.arange(n)
    draw = start
    while len(todo):
        u01 = uniform01(seed, len(todo), draw)
        draw += len(todo)
        u = hN + u01 * (hx1 - hN)
        x = H_inv(u)
        k = np.clip(np.floor(x + 0.5), 1, n_items)
        ok = (k - x <= s_thr) | (u >= H(k + 0.5) - h(k))
        out[todo[ok]] = k[ok].astype(np.int64)
        todo = todo[~ok]
    return out


def _scramble(ranks: np.ndarray, R: int) -> np.ndarray:
    """Bijective rank -> local id scramble inside [0, R) so hot ids spread out."""
    P = 2_654_435_761  # prime, coprime with any R < P unless R is a multiple
    if R % P == 0:
        P = 2_246_822_519
    return ((ranks.astype(np.uint64) - np.uint64(1)) * np.uint64(P)) % np.uint64(R)


def make_batch(cfg: Config, step: int = 0, batch: int | None = None) -> Batch:
    """Batch number `step` of the config's stream (same inputs for every arm)."""
    B = batch or cfg.batch
    F = cfg.features
    R = cfg.rows_per_feature
    if cfg.multi_hot <= 0:
        ids = np.empty((B, F), np.uint64)
        for f in range(F):
            fs = _feature_seed(cfg, f)
            local = rng_stream(fs, B, step * B) % np.uint64(R)
            ids[:, f] = np.uint64(f * R) + local
        offsets = np.arange(B * F + 1, dtype=np.uint32)
        return Batch(ids.reshape(-1), offsets, B, F, {"step": step})
    # multi-hot: counts ~ Poisson(mean) clipped to [1, 100] (inverse-CDF on the stream)
    cseed = mix64_int(cfg.seed ^ 0xC0FFEE)
    u = uniform01(cseed, B * F, step * B * F)
    lam = cfg.multi_hot
    kmax = 100
    pmf = np.zeros(kmax + 1)
    pmf[0] = np.exp(-lam)
    for k in range(1, kmax + 1):
        pmf[k] = pmf[k - 1] * lam / k
    cdf = np.cumsum(pmf)
    counts = np.clip(np.searchsorted(cdf, u * cdf[-1], side="right"), 1, kmax).reshape(B, F)
    segs = []
    for f in range(F):
        fs = _feature_seed(cfg, f)
        n = int(counts[:, f].sum())
        start = step * B * kmax  # disjoint draw windows per step
        if cfg.zipf > 0:
            ranks = _zipf_ranks(fs, n, cfg.zipf, R, start * 4)
            local = _scramble(ranks, R)
        else:
            local = rng_stream(fs, n, start) % np.uint64(R)
        segs.append(np.uint64(f * R) + local)
    # assemble sample-major, group-minor; dedupe + sort within each (sample, group)
    seg_id = []
    vals = []
    for f in range(F):
        c = counts[:, f]
        sid = np.repeat(np.arange(B, dtype=np.int64) * F + f, c)
        seg_id.append(sid)
        vals.append(segs[f])
    seg_id = np.concatenate(seg_id)
    vals = np.concatenate(vals)
    order = np.lexsort((vals, seg_id))
    seg_id = seg_id[order]
    vals = vals[order]
    keep = np.ones(len(vals), bool)
    keep[1:] = (seg_id[1:] != seg_id[:-1]) | (vals[1:] != vals[:-1])
    seg_id = seg_id[keep]
    vals = vals[keep]
    cnt = np.bincount(seg_id, minlength=B * F)
    offsets = np.zeros(B * F + 1, np.uint32)
    np.cumsum(cnt, out=offsets[1:])
    return Batch(vals.astype(np.uint64), offsets, B, F, {"step": step})


def make_grads(cfg: Config, B: int, step: int = 0) -> np.ndarray:
    """Per-sample pooled-embedding gradients U(-scale, scale), [B, F, D] f32."""
    n = B * cfg.features * cfg.dim
    u = uniform01(cfg.seed + 1, n, step * n)
    g = (-cfg.grad_scale + (2 * cfg.grad_scale) * u).astype(np.float32)
    return g.reshape(B, cfg.features, cfg.dim)


def random_csr(rng: np.random.Generator, B: int, F: int, max_per_group: int, id_space: int,
               empty_prob: float = 0.1, dup_prob: float = 0.1):
    """Ragged CSR batch for parity tests: empty groups, duplicates within a group and
    across groups, ids from a small space so rows collide across samples."""
    counts = rng.integers(0, max_per_group + 1, size=B * F)
    counts[rng.random(B * F) < empty_prob] = 0
    ids = []
    for c in counts:
        g = rng.integers(0, id_space, size=c).astype(np.uint64)
        if c > 1 and rng.random() < dup_prob:
            g[-1] = g[0]
        ids.append(g)
    offsets = np.zeros(B * F + 1, np.uint32)
    np.cumsum(counts, out=offsets[1:])
    flat = np.concatenate(ids) if ids else np.zeros(0, np.uint64)
    return flat.astype(np.uint64), offsets


def make_dense_inputs(cfg: Config, batch: Batch, non_id_dim: int = C5_NON_ID,
                      teacher_scale: float = 8.0):
    """Non-id features U(-1, 1) and teacher labels for a batch (the reference's synthetic
    CTR stream, data.hpp:105-186, in spirit: a fixed per-id latent and a fixed linear map,
    label ~ Bernoulli(sigmoid(logit))). Returns (non_id [B, nd] f32, labels [B] f32)."""
    B, F = batch.B, batch.F
    step = batch.meta.get("step", 0)
    non_id = (-1.0 + 2.0 * uniform01(cfg.seed ^ 0xD5, B * non_id_dim, step * B * non_id_dim))
    non_id = non_id.reshape(B, non_id_dim)
    # per-id latent in [-1, 1), mean over each group's listings, summed over groups
    lat = (mix64(batch.ids ^ np.uint64(0x7465616368657200)) >> np.uint64(11)).astype(
        np.float64) * 2.0**-53 * 2.0 - 1.0
    offs = batch.offsets.astype(np.int64)
    sums = np.add.reduceat(lat, np.minimum(offs[:-1], len(lat) - 1)) if len(lat) else \
        np.zeros(B * F)
    cnt = np.diff(offs)
    sums = np.where(cnt > 0, sums / np.maximum(cnt, 1), 0.0).reshape(B, F)
    wf = -1.0 + 2.0 * uniform01(cfg.seed ^ 0x7E, F + non_id_dim)
    logit = teacher_scale / np.sqrt(F + non_id_dim) * (sums @ wf[:F] + non_id @ wf[F:])
    u = uniform01(cfg.seed ^ 0x1AB, B, step * B)
    labels = (u < 1.0 / (1.0 + np.exp(-logit))).astype(np.float32)
    return non_id.astype(np.float32), labels
