"""Pins the C restatement (oracle/hps_oracle.c) to the reference itself.

CPU only. The reference side is oracle/_ref/libhps_ref.so -- the unmodified
reference headers driven through ref_driver.cpp (PsShard behind PsShardService on a
LocalHub, EmbeddingWorker in front, sync order). Every comparison is bit-exact.
"""
import numpy as np
import pytest

import oracle as O
from paper_2111_05897_b200 import workloads as W

pytestmark = pytest.mark.usefixtures("oracle_built")


def test_mix64_known_answers():
    # test_core.cpp:96-108 pins mix64(0); the rest cross-checks restatement vs reference.
    assert O.mix64(0) == 0xE220A8397B1DCDAF
    ref = O.reference_lib()
    rng = np.random.default_rng(1)
    xs = [0, 1, 2**64 - 1, 2**63] + [int(v) for v in rng.integers(0, 2**63, 200, dtype=np.int64)]
    for x in xs:
        assert O.mix64(x) == ref.ref_mix64(x) == W.mix64_int(x)
        for s in (1, 3, 4, 8, 16, 26):
            assert O.route_shard(x, s) == ref.ref_route_shard(x, s) == O.mix64(x) % s
    v = W.mix64(np.array(xs, np.uint64))
    assert [int(a) for a in v] == [O.mix64(x) for x in xs]


@pytest.mark.parametrize("dim", [1, 2, 4, 16, 64, 128])
def test_lazy_init_matches_reference(dim):
    salt = 11
    ref = O.Reference([salt], 4096, dim, "adagrad", "mean", 1)
    ids = np.array([0, 1, 42, 2**63 + 5, 2**64 - 2, 2**64 - 1, 123456789], np.uint64)
    got, ver = ref.shard_lookup(0, ids)
    assert (ver == 0).all()
    for k, i in enumerate(ids):
        mine = O.init_row(int(i), salt, dim)
        assert mine.tobytes() == got[k].tobytes()
    lim = 1.0 / np.sqrt(dim)
    assert np.all(np.abs(got) <= lim)


def _run_both(B, F, D, S, opt, agg, steps, E=1, seed=0, max_per_group=4, id_space=60,
              lr=0.05, has_step=True):
    rng = np.random.default_rng(seed)
    salts = [W.mix64_int(100 + s) for s in range(S)]
    ref = O.Reference(salts, 1 << 14, D, opt, agg, F, workers=E)
    orc = O.Restatement(salts, D, opt)
    for step in range(steps):
        ids, offs = W.random_csr(rng, B, F, max_per_group, id_space)
        grads = (rng.standard_normal((B, F, D)) * 0.3).astype(np.float32)
        pooled_r, rv_r, sids = ref.step(B, ids, offs.astype(np.uint64), grads, lr, step + 1,
                                        has_step, pull=True, push=False)
        pooled_o, rv_o = orc.pull_batch(B, F, ids, offs.astype(np.uint64), agg)
        assert pooled_r.tobytes() == pooled_o.tobytes(), f"pooled differs at step {step}"
        assert (rv_r == rv_o).all()
        ref.step(B, ids, offs.astype(np.uint64), grads, lr, step + 1, has_step, pull=False,
                 push=True)
        ok, _ = orc.push_batch(B, F, ids, offs.astype(np.uint64), grads, lr,
                               step + 1 if has_step else 0, read_versions=rv_o, sample_keys=sids,
                               agg=agg)
        assert ok
    state = ref.state()
    keys = np.array(sorted(state), np.uint64)
    w, a, v, present = orc.peek(keys)
    assert present.all()
    for k, i in enumerate(keys):
        rw, ra, rvv = state[int(i)]
        assert rw.tobytes() == w[k].tobytes(), f"w differs for id {i}"
        assert ra.tobytes() == a[k].tobytes(), f"acc differs for id {i}"
        assert rvv == int(v[k])
    assert orc.counters()["size"] == len(state)
    return ref, orc


@pytest.mark.parametrize("opt", ["adagrad", "sgd"])
@pytest.mark.parametrize("agg", ["mean", "sum"])
def test_sync_steps_bit_exact(opt, agg):
    _run_both(B=24, F=3, D=8, S=4, opt=opt, agg=agg, steps=4, seed=3)


def test_sync_steps_two_workers_interleaved_sids():
    # E=2: sample i -> EW i%2, apply order is ascending SampleId (all of EW0 first).
    _run_both(B=17, F=2, D=4, S=2, opt="adagrad", agg="mean", steps=3, E=2, seed=5)


def test_sync_steps_hot_rows_long_chains():
    # tiny id space -> every row is hit by many samples per step (ordered recurrence)
    _run_both(B=64, F=2, D=16, S=3, opt="adagrad", agg="mean", steps=3, seed=9, id_space=5,
              max_per_group=6)


def test_sync_steps_without_step_tags():
    _run_both(B=12, F=2, D=4, S=1, opt="adagrad", agg="sum", steps=3, seed=11, has_step=False)


def test_c1_config_one_step():
    cfg = W.CONFIGS["c1"]
    b = W.make_batch(cfg, 0, batch=256)
    g = W.make_grads(cfg, 256, 0)
    ref = O.Reference(cfg.salts(), 1 << 16, cfg.dim, cfg.optimizer, cfg.aggregation, cfg.features)
    orc = O.Restatement(cfg.salts(), cfg.dim, cfg.optimizer)
    off = b.offsets.astype(np.uint64)
    pr, rvr, sids = ref.step(b.B, b.ids, off, g, cfg.lr, 1, True, pull=True, push=True)
    po, rvo = orc.pull_batch(b.B, b.F, b.ids, off, cfg.aggregation)
    assert pr.tobytes() == po.tobytes()
    orc.push_batch(b.B, b.F, b.ids, off, g, cfg.lr, 1, read_versions=rvo, sample_keys=sids,
                   agg=cfg.aggregation)
    st = ref.state()
    keys = np.array(sorted(st), np.uint64)
    w, a, v, _ = orc.peek(keys)
    assert np.stack([st[int(k)][0] for k in keys]).tobytes() == w.tobytes()


def test_direct_apply_and_delays_match_reference():
    D = 3
    ref = O.Reference([5], 64, D, "adagrad", "mean", 1)
    orc = O.Restatement([5], D, "adagrad")
    rng = np.random.default_rng(2)
    ids = np.array([1, 2, 1, 3, 1, 2], np.uint64)
    ref.shard_lookup(0, ids)
    orc.lookup(ids)
    for step, rv_shift in [(1, 0), (2, 0), (3, 1), (5, 0), (4, 2)]:
        g = rng.standard_normal((len(ids), D)).astype(np.float32)
        _, vr = ref.shard_lookup(0, ids)
        rvs = np.maximum(vr.astype(np.int64) - rv_shift, 0).astype(np.uint64)
        okr, dr = ref.shard_apply(0, ids, g, rvs, 0.1, step, 0)
        oko, do = orc.apply(ids, g, rvs, 0.1, step)
        assert okr and oko
        assert (dr == do).all()
    st = ref.state()
    keys = np.array(sorted(st), np.uint64)
    w, a, v, _ = orc.peek(keys)
    for k, i in enumerate(keys):
        assert st[int(i)][0].tobytes() == w[k].tobytes()
        assert st[int(i)][1].tobytes() == a[k].tobytes()
        assert st[int(i)][2] == int(v[k])


def test_divergence_rejected_atomically():
    orc = O.Restatement([5], 2, "adagrad")
    before, _ = orc.lookup([1, 2])
    g = np.array([[1, 1], [1, np.nan]], np.float32)
    with pytest.raises(O.OracleError) as e:
        orc.apply([1, 2], g, [0, 0], 0.1, 1)
    assert e.value.code == 6
    after, _ = orc.lookup([1, 2])
    assert before.tobytes() == after.tobytes()


def test_stale_epoch_drops_whole_call():
    orc = O.Restatement([5], 2, "sgd")
    before, _ = orc.lookup([4])
    ok, _ = orc.apply([4], np.ones((1, 2), np.float32), [0], 0.1, 1, epoch=orc.epoch + 1)
    assert not ok
    assert orc.counters()["stale_epoch_drops"] == 1
    assert orc.lookup([4])[0].tobytes() == before.tobytes()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_compress_indices_matches_reference(seed):
    rng = np.random.default_rng(seed)
    B, G = 40, 3
    ids, offs = W.random_csr(rng, B, G, 5, 30, empty_prob=0.2, dup_prob=0.5)
    a = O.compress_indices(B, G, ids, offs.astype(np.uint64), "restatement")
    b = O.compress_indices(B, G, ids, offs.astype(np.uint64), "reference")
    assert len(a) == len(b) == G
    for (ua, pa), (ub, pb) in zip(a, b):
        assert (ua == ub).all()
        assert len(pa) == len(pb)
        for x, y in zip(pa, pb):
            assert (x == y).all()


def test_compress_indices_hand_enumerated():
    # test_codec.cpp:47-60 shape: samples {5,3},{3},{5,5,7}
    ids = np.array([5, 3, 3, 5, 5, 7], np.uint64)
    offs = np.array([0, 2, 3, 6], np.uint64)
    (u, p), = O.compress_indices(3, 1, ids, offs)
    assert list(u) == [3, 5, 7]
    assert [list(x) for x in p] == [[0, 1], [0, 2], [2]]
    with pytest.raises(O.OracleError):
        O.compress_indices(65536, 1, np.zeros(0, np.uint64), np.zeros(65537, np.uint64))


def test_reference_hot_path_gtests_pass():
    """The reference's own six hot-path GTest files, compiled against the reference
    headers with the gtest shim (oracle/Makefile), all pass."""
    import os
    import subprocess

    here = os.path.join(os.path.dirname(O.__file__), "_ref")
    names = ["test_core", "test_codec", "test_lru_store", "test_embedding_ps",
             "test_embedding_worker", "test_staleness"]
    missing = [n for n in names if not os.path.exists(os.path.join(here, n))]
    if missing:
        pytest.skip(f"reference test binaries not built: {missing}")
    for n in names:
        r = subprocess.run([os.path.join(here, n)], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        assert " 0 failed" in r.stdout
