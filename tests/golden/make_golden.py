"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself.

Run here (needs oracle/_ref/libhps_ref.so, built from /root/reference by
`make -C oracle`):   python tests/golden/make_golden.py

Every array is an output of the unmodified reference headers driven through
oracle/ref_driver.cpp (sync order). The fixtures are committed so the GPU box,
where /root/reference does not exist, can check the CUDA path against them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402
from paper_2111_05897_b200 import workloads as W  # noqa: E402


def state_arrays(ref):
    st = ref.state()
    keys = np.array(sorted(st), np.uint64)
    w = np.stack([st[int(k)][0] for k in keys]) if len(keys) else np.zeros((0, ref.D), np.float32)
    a = np.stack([st[int(k)][1] for k in keys]) if len(keys) else np.zeros((0, ref.D), np.float32)
    v = np.array([st[int(k)][2] for k in keys], np.uint64)
    return keys, w, a, v


def sync_case(name, cfg_kw, batches, grads, lr, E=1, has_step=True):
    D, S, opt, agg, F = cfg_kw["D"], cfg_kw["S"], cfg_kw["opt"], cfg_kw["agg"], cfg_kw["F"]
    salts = cfg_kw["salts"]
    ref = O.Reference(salts, cfg_kw.get("capacity", 1 << 16), D, opt, agg, F, workers=E)
    out = dict(D=D, S=S, F=F, opt=opt, agg=agg, lr=np.float32(lr), E=E, salts=np.array(salts, np.uint64),
               steps=len(batches), has_step=has_step)
    for s, ((ids, offs, B), g) in enumerate(zip(batches, grads)):
        pooled, rv, sids = ref.step(B, ids, offs.astype(np.uint64), g, lr, s + 1, has_step)
        out[f"ids_{s}"] = ids
        out[f"offsets_{s}"] = offs.astype(np.uint32)
        out[f"B_{s}"] = B
        out[f"grads_{s}"] = g
        out[f"pooled_{s}"] = pooled
        out[f"rv_{s}"] = rv
        out[f"sids_{s}"] = sids
    keys, w, a, v = state_arrays(ref)
    out.update(final_ids=keys, final_w=w, final_acc=a, final_ver=v)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k: getattr(v, "shape", v) for k, v in out.items() if k.startswith(("final", "pooled_0"))})


def main():
    # 1) config c1 (BASELINE configs[0]) at its full batch: 1024 x 8 one-hot, D=16, sum, SGD.
    cfg = W.CONFIGS["c1"]
    batches, grads = [], []
    for s in range(2):
        b = W.make_batch(cfg, s)
        batches.append((b.ids, b.offsets, b.B))
        grads.append(W.make_grads(cfg, b.B, s))
    sync_case("c1_two_steps", dict(D=cfg.dim, S=cfg.shards, opt=cfg.optimizer, agg=cfg.aggregation,
                                   F=cfg.features, salts=cfg.salts(), capacity=1 << 20),
              batches, grads, cfg.lr)

    # 2) ragged multi-hot, mean, Adagrad, duplicates within and across groups, empty groups,
    #    hot rows (small id space), two embedding workers (interleaved SampleIds).
    rng = np.random.default_rng(2024)
    batches, grads = [], []
    for s in range(3):
        ids, offs = W.random_csr(rng, 48, 4, 6, 40, empty_prob=0.15, dup_prob=0.3)
        batches.append((ids, offs, 48))
        grads.append((rng.standard_normal((48, 4, 8)) * 0.5).astype(np.float32))
    sync_case("ragged_mean_adagrad_e2", dict(D=8, S=3, opt="adagrad", agg="mean", F=4,
                                             salts=[W.mix64_int(9 + s) for s in range(3)]),
              batches, grads, 0.1, E=2)

    # 3) sum + Adagrad, odd dim (generic kernel path), one worker, no step tags.
    batches, grads = [], []
    for s in range(2):
        ids, offs = W.random_csr(rng, 20, 3, 4, 25, empty_prob=0.2, dup_prob=0.4)
        batches.append((ids, offs, 20))
        grads.append((rng.standard_normal((20, 3, 5)) * 0.5).astype(np.float32))
    sync_case("ragged_sum_adagrad_d5", dict(D=5, S=2, opt="adagrad", agg="sum", F=3,
                                            salts=[W.mix64_int(3 + s) for s in range(2)]),
              batches, grads, 0.05, has_step=False)

    # 4) compress_indices
    ids, offs = W.random_csr(rng, 64, 3, 5, 50, empty_prob=0.2, dup_prob=0.5)
    res = O.compress_indices(64, 3, ids, offs.astype(np.uint64), "reference")
    d = dict(ids=ids, offsets=offs.astype(np.uint32), B=64, G=3)
    for g, (u, posts) in enumerate(res):
        d[f"unique_{g}"] = u
        d[f"post_len_{g}"] = np.array([len(p) for p in posts], np.uint32)
        d[f"postings_{g}"] = np.concatenate(posts) if posts else np.zeros(0, np.uint16)
    np.savez_compressed(os.path.join(HERE, "compress_indices.npz"), **d)

    # 5) mix64 / routing / lazy-init vectors
    xs = np.array([0, 1, 2, 42, 2**63, 2**64 - 2, 2**64 - 1] +
                  list(rng.integers(0, 2**63, 64, dtype=np.int64)), np.uint64)
    lib = O.reference_lib()
    mixed = np.array([lib.ref_mix64(int(x)) for x in xs], np.uint64)
    routes = np.array([[lib.ref_route_shard(int(x), s) for s in (1, 2, 3, 8, 26)] for x in xs],
                      np.uint32)
    init = {}
    for dim in (1, 4, 5, 16, 64):
        ref = O.Reference([77], 256, dim, "adagrad", "mean", 1)
        vals, _ = ref.shard_lookup(0, xs)
        init[f"init_{dim}"] = vals
    np.savez_compressed(os.path.join(HERE, "mix64_init.npz"), x=xs, mix=mixed, routes=routes,
                        route_s=np.array([1, 2, 3, 8, 26], np.uint32), salt=77, **init)
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))


if __name__ == "__main__":
    main()
