"""CUDA path vs the oracle / reference fixtures, through the C ABI. Needs a B200.

Bar (BASELINE.json north_star): bit-exact for hashing, routing, dedup and inverse
indices; pooled embeddings, updated rows and optimizer state are compared
bit-exactly too (stricter than the 1e-5 relative tolerance the north star allows)
because the kernels replicate the reference's rounding sequence.
"""
import numpy as np
import pytest

import golden_cases as G

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("oracle_built")]


@pytest.fixture(scope="module")
def hps():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2111_05897_b200 import hps as H

    H.lib()
    return H


# ---------------------------------------------------------------- reference fixtures


@pytest.mark.parametrize("case", G.SYNC_CASES)
def test_reference_fixture_host_buffers(hps, case):
    G.replay_gpu(case, device_arrays=False)


@pytest.mark.parametrize("case", G.SYNC_CASES)
def test_reference_fixture_device_buffers(hps, case):
    G.replay_gpu(case, device_arrays=True)


def test_mix64_route_init_vectors(hps):
    d = G.load("mix64_init")
    for x, m in zip(d["x"], d["mix"]):
        assert hps.mix64(int(x)) == int(m)
    for j, s in enumerate(d["route_s"]):
        got = hps.route(d["x"], int(s))
        assert (got == d["routes"][:, j]).all()
    for dim in (1, 4, 5, 16, 64):
        t = hps.ShardSet(1, dim, 1024, hps.ADAGRAD, salts=[int(d["salt"])])
        vals, ver = t.lookup(d["x"])
        assert vals.tobytes() == d[f"init_{dim}"].tobytes()
        assert (ver == 0).all()


def test_route_on_device_tensors(hps):
    import torch

    from paper_2111_05897_b200 import workloads as W

    ids = np.random.default_rng(0).integers(0, 2**63, 100_000, dtype=np.int64).astype(np.uint64)
    t = torch.from_numpy(ids.view(np.int64)).cuda()
    out = hps.route(t, 26).cpu().numpy().view(np.uint32)
    assert (out == (W.mix64(ids) % np.uint64(26)).astype(np.uint32)).all()


# ---------------------------------------------------------------- random sync steps vs oracle


def _sync_vs_oracle(hps, B, F, D, S, opt, agg, steps, E=1, seed=0, max_per_group=4,
                    id_space=60, lr=0.05, capacity=1 << 16, batches=None):
    import oracle as O
    from paper_2111_05897_b200 import workloads as W

    rng = np.random.default_rng(seed)
    salts = [W.mix64_int(100 + s) for s in range(S)]
    orc = O.Restatement(salts, D, opt)
    table = hps.ShardSet(S, D, capacity, hps.ADAGRAD if opt == "adagrad" else hps.SGD, salts=salts)
    ew = hps.EmbeddingWorker(table, hps.MEAN if agg == "mean" else hps.SUM)
    for step in range(steps):
        if batches is None:
            ids, offs = W.random_csr(rng, B, F, max_per_group, id_space)
        else:
            ids, offs = batches[step]
        grads = (rng.standard_normal((B, F, D)) * 0.3).astype(np.float32)
        i = np.arange(B, dtype=np.uint64)
        sids = ((i % np.uint64(E)) << np.uint64(56)) | (i // np.uint64(E))
        po, rvo = orc.pull_batch(B, F, ids, offs.astype(np.uint64), agg)
        ew.register_batch(ids, offs, B, F, sample_keys=sids if E > 1 else None)
        rv = np.zeros(len(ids), np.uint64)
        pg = ew.serve_pull(out_read_versions=rv)
        assert pg.tobytes() == po.tobytes(), f"pooled differs at step {step}"
        assert (rv == rvo).all()
        orc.push_batch(B, F, ids, offs.astype(np.uint64), grads, lr, step + 1, read_versions=rvo,
                       sample_keys=sids, agg=agg)
        assert ew.apply_backward(grads, lr, step + 1)
    st_ids = _touched(orc)
    w, a, v, p = table.peek(st_ids)
    wo, ao, vo, po_ = orc.peek(st_ids)
    assert p.all() and po_.all()
    np.testing.assert_array_equal(w, wo)
    np.testing.assert_array_equal(a, ao)
    np.testing.assert_array_equal(v, vo)
    assert table.size() == orc.counters()["size"]
    return table, orc


def _touched(orc):
    # ids known to the oracle: recover via peek over the id space used by the tests
    space = np.arange(0, 1 << 16, dtype=np.uint64)
    _, _, _, present = orc.peek(space)
    return space[present]


@pytest.mark.parametrize("D", [1, 2, 3, 4, 8, 16, 32, 64, 100, 128])
def test_sync_steps_all_dims(hps, D):
    _sync_vs_oracle(hps, B=32, F=3, D=D, S=4, opt="adagrad", agg="mean", steps=3, seed=D)


@pytest.mark.parametrize("opt", ["adagrad", "sgd"])
@pytest.mark.parametrize("agg", ["mean", "sum"])
def test_sync_steps_opt_agg(hps, opt, agg):
    _sync_vs_oracle(hps, B=64, F=4, D=16, S=3, opt=opt, agg=agg, steps=3, seed=7)


def test_sync_two_workers_sample_keys(hps):
    _sync_vs_oracle(hps, B=33, F=2, D=8, S=2, opt="adagrad", agg="mean", steps=3, E=2, seed=4)


@pytest.mark.parametrize("D,opt,agg", [(64, "adagrad", "mean"), (16, "sgd", "sum"),
                                       (5, "adagrad", "sum"), (128, "adagrad", "mean"),
                                       (200, "sgd", "mean")])
def test_hot_rows_long_chains(hps, D, opt, agg):
    # every row hit by thousands of listings per step: hot rows (update_runs: 32-position
    # batches of contributions staged in shared memory by cp.async, a warp per 32
    # dimensions running the ordered recurrence), odd and > 128 dims included
    _sync_vs_oracle(hps, B=2048, F=2, D=D, S=1, opt=opt, agg=agg, steps=2, seed=5,
                    id_space=4, max_per_group=5)


def test_large_ragged_batch(hps):
    _sync_vs_oracle(hps, B=4096, F=8, D=32, S=8, opt="adagrad", agg="mean", steps=2, seed=6,
                    id_space=50_000, max_per_group=12)


def test_empty_and_all_empty_groups(hps):
    B, F = 8, 3
    ids = np.zeros(0, np.uint64)
    offs = np.zeros(B * F + 1, np.uint32)
    _sync_vs_oracle(hps, B=B, F=F, D=4, S=1, opt="adagrad", agg="mean", steps=1,
                    batches=[(ids, offs)])


# ---------------------------------------------------------------- full-size configs


def test_c2_full_batch_one_step(hps):
    """BASELINE configs[1] shape: 16384 x 26 one-hot over a 100M-id space, D=64, Adagrad."""
    import oracle as O
    from paper_2111_05897_b200 import workloads as W

    cfg = W.CONFIGS["c2"]
    b = W.make_batch(cfg, 0)
    g = W.make_grads(cfg, b.B, 0)
    orc = O.Restatement(cfg.salts(), cfg.dim, cfg.optimizer)
    table = hps.ShardSet(cfg.shards, cfg.dim, 1 << 20, hps.ADAGRAD, salts=cfg.salts())
    ew = hps.EmbeddingWorker(table, hps.MEAN)
    off64 = b.offsets.astype(np.uint64)
    for step in range(2):
        po, rvo = orc.pull_batch(b.B, b.F, b.ids, off64, "mean")
        ew.register_batch(b.ids, b.offsets, b.B, b.F)
        pg = ew.serve_pull()
        assert pg.tobytes() == po.tobytes()
        orc.push_batch(b.B, b.F, b.ids, off64, g, cfg.lr, step + 1, read_versions=rvo, agg="mean")
        ew.apply_backward(g, cfg.lr, step + 1)
    uniq = np.unique(b.ids)
    w, a, v, p = table.peek(uniq)
    wo, ao, vo, _ = orc.peek(uniq)
    assert p.all()
    np.testing.assert_array_equal(w, wo)
    np.testing.assert_array_equal(a, ao)
    np.testing.assert_array_equal(v, vo)
    assert (v == 2).all()


def test_c3_multi_hot_zipf(hps):
    """configs[2] stress shape at reduced batch: multi-hot (avg 50) Zipf(1.1)."""
    from paper_2111_05897_b200 import workloads as W

    cfg = W.CONFIGS["c3"]
    b = W.make_batch(cfg, 0, batch=256)
    assert b.N > 256 * 26 * 20
    _sync_vs_oracle_batch(hps, cfg, b)


@pytest.mark.parametrize("opt,agg", [("sgd", "sum"), ("adagrad", "sum"), ("sgd", "mean")])
def test_multi_hot_large_plan_short_runs(hps, opt, agg):
    """A multi-hot batch (listings >> groups) with > 4096 repeated listings: the large plan
    with per-position metadata, so runs of 2..63 listings take update_short (a warp per row
    from registers) and longer ones update_runs -- for SGD and sum pooling too."""
    from paper_2111_05897_b200 import workloads as W

    rng = np.random.default_rng(41)
    batches = [W.random_csr(rng, 1500, 4, 24, 4000) for _ in range(2)]
    assert int(batches[0][1][-1]) > 2 * 1500 * 4
    _sync_vs_oracle(hps, B=1500, F=4, D=64, S=4, opt=opt, agg=agg, steps=2, batches=batches)


def test_multi_hot_large_plan_stale_reads(hps):
    """Two multi-hot batches pulled before either is pushed: the second push's read
    versions predate the first push (snapshot path), through the large plan's update_short /
    update_runs version accounting -- rows, accumulators, versions and clock resets vs the
    oracle."""
    import oracle as O
    from paper_2111_05897_b200 import workloads as W

    rng = np.random.default_rng(43)
    S, D, B, F = 4, 64, 1200, 4
    salts = [W.mix64_int(100 + s) for s in range(S)]
    orc = O.Restatement(salts, D, "adagrad")
    table = hps.ShardSet(S, D, 1 << 16, hps.ADAGRAD, salts=salts)
    ews = [hps.EmbeddingWorker(table, hps.MEAN) for _ in range(2)]
    bs = [W.random_csr(rng, B, F, 24, 3000) for _ in range(2)]
    gs = [(rng.standard_normal((B, F, D)) * 0.3).astype(np.float32) for _ in range(2)]
    rvos = []
    for k in range(2):
        ids, offs = bs[k]
        po, rvo = orc.pull_batch(B, F, ids, offs.astype(np.uint64), "mean")
        rvos.append(rvo)
        ews[k].register_batch(ids, offs, B, F)
        pg = ews[k].serve_pull()
        assert pg.tobytes() == po.tobytes()
    for k in range(2):
        ids, offs = bs[k]
        orc.push_batch(B, F, ids, offs.astype(np.uint64), gs[k], 0.05, k + 1,
                       read_versions=rvos[k], agg="mean")
        assert ews[k].apply_backward(gs[k], 0.05, k + 1)
    st_ids = _touched(orc)
    w, a, v, p = table.peek(st_ids)
    wo, ao, vo, po_ = orc.peek(st_ids)
    assert w.tobytes() == wo.tobytes()
    assert a.tobytes() == ao.tobytes()
    assert (v == vo).all()
    assert table.counters().clock_resets == orc.counters()["clock_resets"]


def test_c3_full_size_two_steps(hps):
    """configs[2] at full size: 16384 x 26 multi-hot (avg 50) Zipf(1.1) -- 16.9M listings,
    3.8M rows, the hottest row listed ~16k times -- two sync steps through the large plan
    (radix sort, runs lists, warp-per-row updates of hot and multi rows, singles), pooled
    output, rows, accumulators and versions bit-exact vs the oracle."""
    import oracle as O
    from paper_2111_05897_b200 import workloads as W

    cfg = W.CONFIGS["c3"]
    b = W.make_batch(cfg, 0)
    assert b.N > 16_000_000
    orc = O.Restatement(cfg.salts(), cfg.dim, cfg.optimizer)
    table = hps.ShardSet(cfg.shards, cfg.dim, 1 << 22, hps.ADAGRAD, salts=cfg.salts(),
                         tag_ring=False)
    ew = hps.EmbeddingWorker(table, hps.MEAN)
    off64 = b.offsets.astype(np.uint64)
    counts = np.bincount(np.unique(b.ids, return_inverse=True)[1])
    assert counts.max() > 10_000  # the very-hot path is exercised
    for step in range(2):
        g = W.make_grads(cfg, b.B, step)
        po, rvo = orc.pull_batch(b.B, b.F, b.ids, off64, "mean")
        ew.register_batch(b.ids, b.offsets, b.B, b.F)
        pg = ew.serve_pull()
        assert pg.tobytes() == po.tobytes(), f"step {step}: pooled differs"
        orc.push_batch(b.B, b.F, b.ids, off64, g, cfg.lr, step + 1, read_versions=rvo,
                       agg="mean")
        assert ew.apply_backward(g, cfg.lr, step + 1)
    uniq = np.unique(b.ids)
    w, a, v, p = table.peek(uniq)
    wo, ao, vo, _ = orc.peek(uniq)
    assert p.all()
    assert w.tobytes() == wo.tobytes(), "rows differ"
    assert a.tobytes() == ao.tobytes(), "accumulators differ"
    np.testing.assert_array_equal(v, vo)


def _sync_vs_oracle_batch(hps, cfg, b):
    import oracle as O
    from paper_2111_05897_b200 import workloads as W

    g = W.make_grads(cfg, b.B, 0)
    orc = O.Restatement(cfg.salts(), cfg.dim, cfg.optimizer)
    table = hps.ShardSet(cfg.shards, cfg.dim, 1 << 22, hps.ADAGRAD, salts=cfg.salts())
    ew = hps.EmbeddingWorker(table, hps.MEAN)
    off64 = b.offsets.astype(np.uint64)
    po, rvo = orc.pull_batch(b.B, b.F, b.ids, off64, "mean")
    ew.register_batch(b.ids, b.offsets, b.B, b.F)
    pg = ew.serve_pull()
    assert pg.tobytes() == po.tobytes()
    orc.push_batch(b.B, b.F, b.ids, off64, g, cfg.lr, 1, read_versions=rvo, agg="mean")
    ew.apply_backward(g, cfg.lr, 1)
    uniq = np.unique(b.ids)
    w, a, v, _ = table.peek(uniq)
    wo, ao, vo, _ = orc.peek(uniq)
    np.testing.assert_array_equal(w, wo)
    np.testing.assert_array_equal(a, ao)
    np.testing.assert_array_equal(v, vo)


# ---------------------------------------------------------------- PS surface


def test_direct_apply_delays_and_versions(hps):
    import oracle as O

    D = 3
    t = hps.ShardSet(1, D, 64, hps.ADAGRAD, salts=[5])
    orc = O.Restatement([5], D, "adagrad")
    rng = np.random.default_rng(2)
    ids = np.array([1, 2, 1, 3, 1, 2], np.uint64)
    t.lookup(ids)
    orc.lookup(ids)
    for step, shift in [(1, 0), (2, 0), (3, 1), (5, 0), (6, 2), (6, 0), (9, 3)]:
        g = rng.standard_normal((len(ids), D)).astype(np.float32)
        _, vg = t.lookup(ids)
        _, vo = orc.lookup(ids)
        assert (vg == vo).all()
        rv = np.maximum(vo.astype(np.int64) - shift, 0).astype(np.uint64)
        okg, dg = t.apply_gradients(ids, g, rv, 0.1, step)
        oko, do = orc.apply(ids, g, rv, 0.1, step)
        assert okg and oko
        assert (dg == do).all(), (step, dg, do)
    keys = np.array([1, 2, 3], np.uint64)
    w, a, v, _ = t.peek(keys)
    wo, ao, vo, _ = orc.peek(keys)
    np.testing.assert_array_equal(w, wo)
    np.testing.assert_array_equal(a, ao)
    np.testing.assert_array_equal(v, vo)


@pytest.mark.parametrize("D,n,space", [(64, 20000, 5000), (3, 300, 40), (16, 9000, 60)])
def test_direct_apply_without_delays_batch_path(hps, D, n, space):
    """apply_gradients without per-entry delays runs through the batch plan (singles,
    repeated ids in array order, >4096 repeated listings -> sorted path); same rows,
    accumulators and versions as the oracle, and the same delay histogram."""
    import oracle as O

    t = hps.ShardSet(2, D, 1 << 16, hps.ADAGRAD, salts=[5, 6])
    orc = O.Restatement([5, 6], D, "adagrad")
    rng = np.random.default_rng(D)
    for step in range(1, 4):
        ids = rng.integers(0, space, n).astype(np.uint64)
        g = (rng.standard_normal((n, D)) * 0.2).astype(np.float32)
        _, vg = t.lookup(ids)
        _, vo = orc.lookup(ids)
        assert (vg == vo).all()
        rv = np.maximum(vo.astype(np.int64) - (step % 2), 0).astype(np.uint64)
        okg, _ = t.apply_gradients(ids, g, rv, 0.1, step, want_delays=False)
        oko, _ = orc.apply(ids, g, rv, 0.1, step)
        assert okg and oko
    keys = np.arange(space, dtype=np.uint64)
    w, a, v, p = t.peek(keys)
    wo, ao, vo, po = orc.peek(keys)
    assert (p == po).all()
    np.testing.assert_array_equal(w[p], wo[po])
    np.testing.assert_array_equal(a[p], ao[po])
    np.testing.assert_array_equal(v[p], vo[po])


def test_reference_staleness_cases(hps):
    # test_embedding_ps.cpp:171-211 restated through the C ABI.
    t = hps.ShardSet(1, 2, 16, hps.ADAGRAD, salts=[11])

    def one(id_, step, rv):
        ok, d = t.apply_gradients([id_], np.ones((1, 2), np.float32), [rv], 0.01, step)
        assert ok
        return int(d[0])

    _, v = t.lookup([8])
    assert one(8, 1, int(v[0])) == 0
    t2 = hps.ShardSet(1, 2, 16, hps.ADAGRAD, salts=[11])
    _, rv = t2.lookup([8])
    ok, _ = t2.apply_gradients([8], np.ones((1, 2), np.float32), rv, 0.01, 1)
    t2.apply_gradients([8], np.ones((1, 2), np.float32), [1], 0.01, 2)
    _, d = t2.apply_gradients([8], np.ones((1, 2), np.float32), rv, 0.01, 3)
    assert d[0] == 2
    t3 = hps.ShardSet(1, 2, 16, hps.ADAGRAD, salts=[11])
    _, rv = t3.lookup([8])
    t3.apply_gradients([8], np.ones((1, 2), np.float32), rv, 0.01, 1)
    _, rv = t3.lookup([8])
    assert t3.apply_gradients([8], np.ones((1, 2), np.float32), rv, 0.01, 2)[1][0] == 0
    assert t3.apply_gradients([8], np.ones((1, 2), np.float32), rv, 0.01, 2)[1][0] == 0
    t4 = hps.ShardSet(1, 2, 16, hps.ADAGRAD, salts=[11])
    _, rv = t4.lookup([8])
    t4.apply_gradients([8], np.ones((1, 2), np.float32), rv, 0.01, 7)
    assert t4.apply_gradients([8], np.ones((1, 2), np.float32), rv, 0.01, 6)[1][0] == 0


def test_sgd_and_adagrad_arithmetic(hps):
    # test_embedding_ps.cpp:87-109
    t = hps.ShardSet(1, 2, 16, hps.SGD, salts=[11])
    cur = t.lookup_map([7])[7]
    t.apply_gradients_map({7: cur - np.array([1.0, 1.0], np.float32)}, 1.0)
    w = t.lookup_map([7])[7]
    t.apply_gradients_map({7: [2.0, 4.0]}, 0.5)
    got = t.lookup_map([7])[7]
    assert got[0] == np.float32(w[0] - np.float32(0.5) * np.float32(2.0))
    assert got[1] == np.float32(w[1] - np.float32(0.5) * np.float32(4.0))
    a = hps.ShardSet(1, 1, 16, hps.ADAGRAD, salts=[11])
    w0 = a.lookup_map([5])[5][0]
    a.apply_gradients_map({5: [3.0]}, 0.1)
    expect = np.float32(w0 - np.float32(np.float32(0.1) * np.float32(3.0)) /
                        np.float32(np.float32(3.0) + np.float32(1e-10)))
    assert a.lookup_map([5])[5][0] == expect


def test_non_finite_rejected_atomically(hps):
    t = hps.ShardSet(1, 2, 16, hps.ADAGRAD, salts=[11])
    before = t.lookup([1, 2])[0].copy()
    size = t.size()
    g = np.array([[1, 1], [1, np.nan]], np.float32)
    with pytest.raises(hps.DivergenceError):
        t.apply_gradients([1, 2], g, [0, 0], 0.1, 1)
    assert t.lookup([1, 2])[0].tobytes() == before.tobytes()
    with pytest.raises(hps.DivergenceError):
        t.apply_gradients_map({3: [np.inf, 0.0]}, 0.1)
    assert t.size() == size  # the rejected call did not even insert id 3
    # batch surface: a NaN in any non-empty group rejects the whole batch
    ew = hps.EmbeddingWorker(t, hps.MEAN)
    ids = np.array([1, 2, 1], np.uint64)
    offs = np.array([0, 2, 3], np.uint32)
    ew.register_batch(ids, offs, 1, 2)
    ew.serve_pull()
    snap = t.peek([1, 2])
    gb = np.ones((1, 2, 2), np.float32)
    gb[0, 1, 0] = np.inf
    with pytest.raises(hps.DivergenceError):
        ew.apply_backward(gb, 0.1, 1)
    after = t.peek([1, 2])
    assert snap[0].tobytes() == after[0].tobytes() and snap[1].tobytes() == after[1].tobytes()
    # NaN in an EMPTY group is never used, so it is not an error (push_to_shards :731)
    ids = np.array([1], np.uint64)
    offs = np.array([0, 1, 1], np.uint32)
    ew.register_batch(ids, offs, 1, 2)
    ew.serve_pull()
    gb = np.ones((1, 2, 2), np.float32)
    gb[0, 1, :] = np.nan
    assert ew.apply_backward(gb, 0.1, 2)


def test_overflowing_contribution_rejected(hps):
    # finite gradients whose fp64 chain-rule sum overflows float -> non-finite push value
    t = hps.ShardSet(1, 1, 16, hps.SGD, salts=[1])
    ew = hps.EmbeddingWorker(t, hps.SUM)
    ids = np.array([4, 4], np.uint64)
    offs = np.array([0, 1, 2], np.uint32)
    ew.register_batch(ids, offs, 1, 2)
    ew.serve_pull()
    before = t.peek([4])[0].copy()
    g = np.full((1, 2, 1), 3.0e38, np.float32)
    with pytest.raises(hps.DivergenceError):
        ew.apply_backward(g, 0.1, 1)
    assert t.peek([4])[0].tobytes() == before.tobytes()


def test_stale_epoch_drops_whole_call(hps):
    t = hps.ShardSet(1, 2, 16, hps.ADAGRAD, salts=[11])
    before = t.lookup([4])[0].copy()
    ok, _ = t.apply_gradients([4], np.ones((1, 2), np.float32), [0], 0.1, 1,
                              caller_epoch=t.epoch() + 1)
    assert not ok
    assert t.stale_epoch_drops() == 1
    assert t.lookup([4])[0].tobytes() == before.tobytes()
    t.advance_epoch()
    ok, _ = t.apply_gradients([4], np.ones((1, 2), np.float32), [0], 0.1, 1)
    assert ok


def test_capacity_exhaustion_is_reported(hps):
    t = hps.ShardSet(1, 4, 8, hps.ADAGRAD, salts=[1])
    t.lookup(np.arange(8, dtype=np.uint64))
    with pytest.raises(hps.ConfigError):
        t.lookup(np.arange(8, 20, dtype=np.uint64))


def test_reset_for_recovery(hps):
    t = hps.ShardSet(1, 4, 64, hps.ADAGRAD, salts=[1])
    a, _ = t.lookup([1, 2, 3])
    t.apply_gradients_map({1: [1, 1, 1, 1]}, 0.5)
    e = t.epoch()
    t.reset_for_recovery()
    assert t.epoch() == e + 1
    assert t.size() == 0
    b, v = t.lookup([1, 2, 3])
    assert a.tobytes() == b.tobytes() and (v == 0).all()


def test_special_all_ones_id(hps):
    import oracle as O

    t = hps.ShardSet(2, 4, 64, hps.ADAGRAD, salts=[3, 4])
    orc = O.Restatement([3, 4], 4, "adagrad")
    ids = np.array([2**64 - 1, 0, 2**64 - 1], np.uint64)
    g, _ = t.lookup(ids)
    o, _ = orc.lookup(ids)
    assert g.tobytes() == o.tobytes()


# ---------------------------------------------------------------- dedup


@pytest.mark.parametrize("n,space", [(1, 10), (1000, 10), (100_000, 2**63), (300_000, 5000)])
def test_dedup_unique_inverse(hps, n, space):
    rng = np.random.default_rng(n)
    ids = rng.integers(0, space, n, dtype=np.int64).astype(np.uint64)
    if n > 10:
        ids[:3] = [2**64 - 1, 0, 2**64 - 1]
    u, inv = hps.dedup(ids)
    nu, ninv = np.unique(ids, return_inverse=True)
    assert (u == nu).all()
    assert (inv.astype(np.int64) == ninv).all()


def test_dedup_device_tensors(hps):
    import torch

    ids = torch.randint(0, 1000, (50_000,), device="cuda")
    u, inv = hps.dedup(ids)
    nu, ninv = np.unique(ids.cpu().numpy().view(np.uint64), return_inverse=True)
    assert (u.cpu().numpy().view(np.uint64) == nu).all()
    assert (inv.cpu().numpy().astype(np.int64) == ninv).all()


def test_compress_indices_fixture(hps):
    d = G.load("compress_indices")
    res = hps.compress_indices(d["ids"], d["offsets"], int(d["B"]), int(d["G"]))
    for g, (u, posts) in enumerate(res):
        assert (u == d[f"unique_{g}"]).all()
        assert [len(p) for p in posts] == list(d[f"post_len_{g}"])
        flat = np.concatenate(posts) if posts else np.zeros(0, np.uint16)
        assert (flat == d[f"postings_{g}"]).all()


@pytest.mark.parametrize("seed", [0, 1])
def test_compress_indices_vs_oracle_random(hps, seed):
    import oracle as O
    from paper_2111_05897_b200 import workloads as W

    rng = np.random.default_rng(seed)
    B, G_ = 3000, 5
    ids, offs = W.random_csr(rng, B, G_, 6, 2000, empty_prob=0.2, dup_prob=0.5)
    a = hps.compress_indices(ids, offs, B, G_)
    b = O.compress_indices(B, G_, ids, offs.astype(np.uint64))
    for (ua, pa), (ub, pb) in zip(a, b):
        assert (ua == ub).all()
        assert all((x == y).all() for x, y in zip(pa, pb))
    with pytest.raises(hps.PreconditionError):
        hps.compress_indices(np.zeros(0, np.uint64), np.zeros(65537, np.uint32), 65536, 1)


# ---------------------------------------------------------------- pipelined batches


def test_pipelined_batches_read_versions(hps):
    """Two batches pulled before either is pushed (bounded staleness 1): the second
    push must count the first push's bumps as delays (embedding_ps.hpp:454-480). The
    GPU materialises B's pull-time versions only when A's push is about to mutate."""
    import oracle as O
    from paper_2111_05897_b200 import workloads as W

    rng = np.random.default_rng(21)
    B, F, D = 40, 3, 8
    salts = [W.mix64_int(5 + s) for s in range(2)]
    orc = O.Restatement(salts, D, "adagrad")
    t = hps.ShardSet(2, D, 1 << 12, hps.ADAGRAD, salts=salts)
    ew_a = hps.EmbeddingWorker(t, hps.MEAN)
    ew_b = hps.EmbeddingWorker(t, hps.MEAN)
    for rnd in range(3):
        ia, oa = W.random_csr(rng, B, F, 4, 30)
        ib, ob = W.random_csr(rng, B, F, 4, 30)
        ga = (rng.standard_normal((B, F, D)) * 0.3).astype(np.float32)
        gb = (rng.standard_normal((B, F, D)) * 0.3).astype(np.float32)
        pa, rva = orc.pull_batch(B, F, ia, oa.astype(np.uint64), "mean")
        pb, rvb = orc.pull_batch(B, F, ib, ob.astype(np.uint64), "mean")
        ew_a.register_batch(ia, oa, B, F)
        ew_b.register_batch(ib, ob, B, F)
        assert ew_a.serve_pull().tobytes() == pa.tobytes()
        assert ew_b.serve_pull().tobytes() == pb.tobytes()
        _, da = orc.push_batch(B, F, ia, oa.astype(np.uint64), ga, 0.05, 2 * rnd + 1,
                               read_versions=rva, agg="mean")
        _, db = orc.push_batch(B, F, ib, ob.astype(np.uint64), gb, 0.05, 2 * rnd + 2,
                               read_versions=rvb, agg="mean")
        ew_a.apply_backward(ga, 0.05, 2 * rnd + 1)
        ew_b.apply_backward(gb, 0.05, 2 * rnd + 2)
        want = np.bincount(np.minimum(np.concatenate([da, db]), 16), minlength=17)
        if rnd == 0:
            hist0 = np.zeros(17, np.int64)
        got = np.array(t.counters().delay_hist[:], np.int64) - hist0
        hist0 = np.array(t.counters().delay_hist[:], np.int64)
        assert (got == want).all(), (got, want)
        assert want[1:].sum() > 0  # the shared rows really saw a delay
    ids = np.arange(0, 30, dtype=np.uint64)
    w, a, v, p = t.peek(ids)
    wo, ao, vo, po = orc.peek(ids)
    assert (p == po).all()
    np.testing.assert_array_equal(w[p], wo[po])
    np.testing.assert_array_equal(a[p], ao[po])
    np.testing.assert_array_equal(v[p], vo[po])


def test_cuda_graph_replay_matches_oracle(hps):
    """A whole step (register + pull + push with HPS_DEVICE_STEP) captured once in a
    CUDA graph and replayed on fresh inputs copied into the captured buffers is
    bit-exact with eager sync steps (step tags advance on the device)."""
    import torch

    import oracle as O
    from paper_2111_05897_b200 import workloads as W

    rng = np.random.default_rng(31)
    B, F, D = 64, 4, 16
    salts = [W.mix64_int(1 + s) for s in range(3)]
    orc = O.Restatement(salts, D, "adagrad")
    t = hps.ShardSet(3, D, 1 << 14, hps.ADAGRAD, salts=salts)
    ew = hps.EmbeddingWorker(t, hps.MEAN)
    dev = torch.device("cuda:0")
    # fixed shape: one-hot-ish CSR with every group of size 1..2 -> same N each step
    counts = np.ones(B * F, np.uint32)
    counts[::5] = 2
    offs = np.zeros(B * F + 1, np.uint32)
    np.cumsum(counts, out=offs[1:])
    N = int(offs[-1])
    ids_t = torch.zeros(N, dtype=torch.int64, device=dev)
    offs_t = torch.from_numpy(offs.view(np.int32)).to(dev)
    g_t = torch.zeros((B, F, D), dtype=torch.float32, device=dev)
    pooled_t = torch.zeros((B, F, D), dtype=torch.float32, device=dev)

    def step(s):
        ew.register_batch(ids_t, offs_t, B, F, stream=s)
        ew.serve_pull(out_pooled=pooled_t, stream=s)
        ew.apply_backward(g_t, 0.05, flags=hps.ASYNC | hps.DEVICE_STEP, stream=s)

    batches = [(rng.integers(0, 200, N).astype(np.uint64),
                (rng.standard_normal((B, F, D)) * 0.3).astype(np.float32)) for _ in range(4)]
    # eager warm-up step 1, then capture, then replay steps 2..4
    ids_t.copy_(torch.from_numpy(batches[0][0].view(np.int64)))
    g_t.copy_(torch.from_numpy(batches[0][1]))
    step(torch.cuda.current_stream())
    torch.cuda.synchronize()
    po, rvo = orc.pull_batch(B, F, batches[0][0], offs.astype(np.uint64), "mean")
    assert pooled_t.cpu().numpy().tobytes() == po.tobytes()
    orc.push_batch(B, F, batches[0][0], offs.astype(np.uint64), batches[0][1], 0.05, 1,
                   read_versions=rvo, agg="mean")
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, capture_error_mode="thread_local"):
        step(torch.cuda.current_stream())
    for k in range(1, 4):
        ids, g = batches[k]
        ids_t.copy_(torch.from_numpy(ids.view(np.int64)))
        g_t.copy_(torch.from_numpy(g))
        graph.replay()
        torch.cuda.synchronize()
        po, rvo = orc.pull_batch(B, F, ids, offs.astype(np.uint64), "mean")
        assert pooled_t.cpu().numpy().tobytes() == po.tobytes(), f"replay {k}"
        orc.push_batch(B, F, ids, offs.astype(np.uint64), g, 0.05, k + 1, read_versions=rvo,
                       agg="mean")
    t.sync()
    assert t.device_step() == 4
    keys = np.arange(200, dtype=np.uint64)
    w, a, v, p = t.peek(keys)
    wo, ao, vo, po_ = orc.peek(keys)
    assert (p == po_).all()
    np.testing.assert_array_equal(w[p], wo[po_])
    np.testing.assert_array_equal(a[p], ao[po_])
    np.testing.assert_array_equal(v[p], vo[po_])


def _graph_case(hps, B, F, D, space, agg, opt, grad_fn, steps=3, seed=5):
    """Register/pull/push captured once in a CUDA graph and replayed on new inputs copied
    into the captured buffers; bit-exact with the oracle stepping eagerly."""
    import torch

    import oracle as O
    from paper_2111_05897_b200 import workloads as W

    rng = np.random.default_rng(seed)
    salts = [W.mix64_int(3 + s) for s in range(4)]
    orc = O.Restatement(salts, D, "adagrad" if opt == hps.ADAGRAD else "sgd")
    t = hps.ShardSet(4, D, 1 << 16, opt, salts=salts)
    ew = hps.EmbeddingWorker(t, agg)
    dev = torch.device("cuda:0")
    offs = np.arange(B * F + 1, dtype=np.uint32) * 2  # two listings per group
    N = int(offs[-1])
    ids_t = torch.zeros(N, dtype=torch.int64, device=dev)
    offs_t = torch.from_numpy(offs.view(np.int32)).to(dev)
    g_t = torch.zeros((B, F, D), dtype=torch.float32, device=dev)
    pooled_t = torch.zeros((B, F, D), dtype=torch.float32, device=dev)
    aggs = "mean" if agg == hps.MEAN else "sum"

    def step(s):
        ew.register_batch(ids_t, offs_t, B, F, stream=s)
        ew.serve_pull(out_pooled=pooled_t, stream=s)
        ew.apply_backward(g_t, 0.05, flags=hps.ASYNC | hps.DEVICE_STEP, stream=s)

    graph = None
    for k in range(steps):
        ids = rng.integers(0, space, N).astype(np.uint64)
        g = grad_fn(rng, (B, F, D))
        ids_t.copy_(torch.from_numpy(ids.view(np.int64)))
        g_t.copy_(torch.from_numpy(g))
        if k == 0:
            step(torch.cuda.current_stream())
        else:
            if graph is None:
                torch.cuda.synchronize()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, capture_error_mode="thread_local"):
                    step(torch.cuda.current_stream())
            graph.replay()
        torch.cuda.synchronize()
        po, rvo = orc.pull_batch(B, F, ids, offs.astype(np.uint64), aggs)
        assert pooled_t.cpu().numpy().tobytes() == po.tobytes(), f"step {k}"
        orc.push_batch(B, F, ids, offs.astype(np.uint64), g, 0.05, k + 1, read_versions=rvo,
                       agg=aggs)
    t.sync()
    keys = np.arange(space, dtype=np.uint64)
    w, a, v, p = t.peek(keys)
    wo, ao, vo, po_ = orc.peek(keys)
    assert (p == po_).all()
    np.testing.assert_array_equal(w[p], wo[po_])
    np.testing.assert_array_equal(a[p], ao[po_])
    np.testing.assert_array_equal(v[p], vo[po_])


def test_cuda_graph_large_plan_conditional(hps):
    """> 4096 listings of repeated rows: the radix-sort path runs inside a conditional
    graph node on every replay."""
    _graph_case(hps, 1024, 4, 64, 1500, hps.MEAN, hps.ADAGRAD,
                lambda r, sh: (r.standard_normal(sh) * 0.1).astype(np.float32))


def test_cuda_graph_need_exact_conditional(hps):
    """Gradients near the float range make the bound check inconclusive: the exact dry
    run executes inside its conditional graph node (and passes), then the update runs."""
    def huge(r, sh):
        g = (r.standard_normal(sh) * 0.1).astype(np.float32)
        g[:, 0, 0] = np.float32(1e38)
        g[:, 1, 0] = np.float32(-1e38)
        return g
    _graph_case(hps, 64, 4, 16, 40, hps.SUM, hps.SGD, huge)


def test_stale_multi_bits_from_unapplied_batch(hps):
    """A batch registered (rows listed twice) but dropped by the epoch fence leaves its
    plan bits set; a later large-plan batch listing such a row once still applies it."""
    import oracle as O

    D = 16
    t = hps.ShardSet(1, D, 1 << 16, hps.ADAGRAD, salts=[9])
    orc = O.Restatement([9], D, "adagrad")
    ew = hps.EmbeddingWorker(t, hps.SUM)
    rng = np.random.default_rng(4)
    # batch A: ids 0..99 each listed twice; pulled, then pushed with a stale epoch
    idsA = np.repeat(np.arange(100, dtype=np.uint64), 2)
    offA = np.arange(len(idsA) + 1, dtype=np.uint32)
    ew.register_batch(idsA, offA, len(idsA), 1)
    ew.serve_pull()
    t.advance_epoch()
    orc.advance_epoch()
    gA = rng.standard_normal((len(idsA), 1, D)).astype(np.float32)
    assert not ew.apply_backward(gA, 0.1, 1, epoch=0)
    orc.lookup(np.arange(100, dtype=np.uint64))  # the pull's lazy inits
    # batch B: ids 0..99 once each, plus > 4096 listings of repeated ids 1000..1999
    idsB = np.concatenate([np.arange(100, dtype=np.uint64),
                           np.repeat(np.arange(1000, 2000, dtype=np.uint64), 5)])
    offB = np.arange(len(idsB) + 1, dtype=np.uint32)
    gB = rng.standard_normal((len(idsB), 1, D)).astype(np.float32)
    ew.register_batch(idsB, offB, len(idsB), 1)
    pooled = ew.serve_pull()
    po, rvo = orc.pull_batch(len(idsB), 1, idsB, offB.astype(np.uint64), "sum")
    assert pooled.tobytes() == po.tobytes()
    assert ew.apply_backward(gB, 0.1, 2)
    ok, _ = orc.push_batch(len(idsB), 1, idsB, offB.astype(np.uint64), gB, 0.1, 2,
                           read_versions=rvo, agg="sum")
    assert ok
    keys = np.concatenate([np.arange(100), np.arange(1000, 2000)]).astype(np.uint64)
    w, a, v, _ = t.peek(keys)
    wo, ao, vo, _ = orc.peek(keys)
    np.testing.assert_array_equal(w, wo)
    np.testing.assert_array_equal(a, ao)
    np.testing.assert_array_equal(v, vo)


def _pipelined_case(hps, B, F, D, space, steps, graph, seed=41, defer=False):
    """bench.py's pipelined sync schedule: batch s+1 is registered on a second stream
    beside batch s's pull + push (two worker handles alternating, each with its own plan
    bitmaps), and pull(s+1) follows push(s) on the main stream. Pooled outputs and the
    final rows must equal the oracle stepping in plain sync order."""
    import torch

    import oracle as O
    from paper_2111_05897_b200 import workloads as W

    rng = np.random.default_rng(seed)
    salts = [W.mix64_int(5 + s) for s in range(4)]
    orc = O.Restatement(salts, D, "adagrad")
    t = hps.ShardSet(4, D, 1 << 16, hps.ADAGRAD, salts=salts)
    ews = [hps.EmbeddingWorker(t, hps.MEAN) for _ in range(2)]
    for w_ in ews:  # defer: the next batch's plan is joined by its push, not its register
        w_.defer_plan_join(defer)
    dev = torch.device("cuda:0")
    main = torch.cuda.Stream()
    side = torch.cuda.Stream()
    offs = (np.arange(B * F + 1, dtype=np.uint32) * 2)  # two listings per group
    N = int(offs[-1])
    data = []
    for _ in range(steps + 1):
        ids = rng.integers(0, space, N).astype(np.uint64)
        g = (rng.standard_normal((B, F, D)) * 0.2).astype(np.float32)
        data.append((ids, g))
    # device copies (one buffer per batch: the pipeline keeps two batches in flight)
    d_ids = [torch.from_numpy(x[0].view(np.int64)).to(dev) for x in data]
    d_g = [torch.from_numpy(x[1]).to(dev) for x in data]
    offs_t = torch.from_numpy(offs.view(np.int32)).to(dev)
    pooled = [torch.zeros((B, F, D), dtype=torch.float32, device=dev) for _ in range(steps)]

    def pipe_step(i, s):
        side.wait_stream(s)
        if i + 1 < len(data):
            ews[(i + 1) % 2].register_batch(d_ids[i + 1], offs_t, B, F, stream=side)
        ews[i % 2].serve_pull(out_pooled=pooled[i], stream=s)
        ews[i % 2].apply_backward(d_g[i], 0.05, flags=hps.ASYNC | hps.DEVICE_STEP, stream=s)
        s.wait_stream(side)

    torch.cuda.synchronize()
    with torch.cuda.stream(main):
        ews[0].register_batch(d_ids[0], offs_t, B, F, stream=main)
        for i in range(steps):
            if graph and i >= 1:
                g_ = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g_, stream=main, capture_error_mode="thread_local"):
                    pipe_step(i, main)
                    if defer and i + 1 < len(data):  # the capture ends before that push
                        ews[(i + 1) % 2].join_plan(stream=main)
                g_.replay()
                main.synchronize()
            else:
                pipe_step(i, main)
    torch.cuda.synchronize()
    t.sync()
    for i in range(steps):
        ids, g = data[i]
        po, rvo = orc.pull_batch(B, F, ids, offs.astype(np.uint64), "mean")
        assert pooled[i].cpu().numpy().tobytes() == po.tobytes(), f"step {i}: pooled differs"
        orc.push_batch(B, F, ids, offs.astype(np.uint64), g, 0.05, i + 1, read_versions=rvo,
                       agg="mean")
    keys = np.arange(space, dtype=np.uint64)
    w, a, v, p = t.peek(keys)
    wo, ao, vo, po_ = orc.peek(keys)
    # the last registered batch (steps) inserted rows the oracle never pulled: compare
    # the rows both hold
    both = p & po_
    np.testing.assert_array_equal(w[both], wo[both])
    np.testing.assert_array_equal(a[both], ao[both])
    np.testing.assert_array_equal(v[both], vo[both])


@pytest.mark.parametrize("graph", [False, True])
def test_pipelined_register_beside_push(hps, graph):
    _pipelined_case(hps, 64, 4, 16, 300, steps=6, graph=graph)


@pytest.mark.parametrize("graph", [False, True])
def test_pipelined_register_beside_push_large_plan(hps, graph):
    """> 4096 listings of repeated rows: the forked large sort of the next batch runs
    while this batch's update chains run on the same aux stream."""
    _pipelined_case(hps, 1024, 4, 64, 1500, steps=4, graph=graph)


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("B,space", [(64, 300), (1024, 1500)])
def test_pipelined_deferred_plan_join(hps, graph, B, space):
    """hps_batch_defer_plan_join: the next batch's plan (sort) is joined by its push, not
    by its register or pull (bench.py's pipeline); under capture the graph that registers
    a batch joins its plan before it ends (hps_batch_join_plan). Bit-exact either way."""
    _pipelined_case(hps, B, 4, 64 if B > 64 else 16, space, steps=4, graph=graph, defer=True)


# ---------------------------------------------------------------- round 2 semantics


def test_out_of_order_step_tags_count_like_the_reference(hps):
    """count_delay walks the 16-deep tag ring (embedding_ps.hpp:454-480): with step tags
    out of order (bumps 1, 5, 2, then a read-version-0 write at step 4) the reference
    counts 2 distinct earlier tags, not the 3 bumps. Delays, versions and rows equal the
    restatement oracle and the reference itself (oracle/_ref)."""
    import oracle as O

    D = 4
    t = hps.ShardSet(1, D, 64, hps.ADAGRAD, salts=[5])
    orc = O.Restatement([5], D, "adagrad")
    ref = O.Reference([5], 64, D, "adagrad", "mean", 1)
    rng = np.random.default_rng(3)
    ids = np.array([7, 8, 7], np.uint64)
    t.lookup(ids)
    orc.lookup(ids)
    ref.shard_lookup(0, ids)
    seq = [(1, 0), (5, 1), (2, 2), (4, 0), (9, 1), (3, 3), (3, 0), (6, 5), (2, 0)]
    for step, rv0 in seq:
        g = rng.standard_normal((len(ids), D)).astype(np.float32)
        rv = np.full(len(ids), rv0, np.uint64)
        okg, dg = t.apply_gradients(ids, g, rv, 0.1, step)
        oko, do = orc.apply(ids, g, rv, 0.1, step)
        okr, dr = ref.shard_apply(0, ids, g, rv, 0.1, step, 0)
        assert okg and oko and okr
        assert (do == dr).all(), (step, do, dr)
        assert (dg == do).all(), (step, dg, do)
    w, a, v, _ = t.peek(np.array([7, 8], np.uint64))
    wo, ao, vo, _ = orc.peek(np.array([7, 8], np.uint64))
    assert w.tobytes() == wo.tobytes() and a.tobytes() == ao.tobytes()
    assert (v == vo).all()
    assert t.clock_reset_count() == orc.counters()["clock_resets"]


def test_untracked_writes_between_tracked_ones(hps):
    """apply_gradients_map bumps versions without a ring entry (:186); a later tracked
    write's window then holds stale ring slots, which count_delay skips or counts exactly
    as the reference does."""
    import oracle as O

    D = 2
    t = hps.ShardSet(1, D, 64, hps.SGD, salts=[9])
    orc = O.Restatement([9], D, "sgd")
    ids = np.array([3], np.uint64)
    t.lookup(ids)
    orc.lookup(ids)
    g = np.ones((1, D), np.float32)
    for k in range(20):
        if k % 3 == 2:
            t.apply_gradients_map({3: g[0]}, 0.01)
            orc.apply_map(ids, g, 0.01)
            continue
        rv = np.array([max(0, k - 4)], np.uint64)
        okg, dg = t.apply_gradients(ids, g, rv, 0.01, k + 1)
        oko, do = orc.apply(ids, g, rv, 0.01, k + 1)
        assert (dg == do).all(), (k, dg, do)
    w, a, v, _ = t.peek(ids)
    wo, ao, vo, _ = orc.peek(ids)
    assert w.tobytes() == wo.tobytes() and (v == vo).all()


def test_async_rejection_surfaces_at_sync(hps):
    """Two HPS_ASYNC pushes, the first with a non-finite gradient, one table.sync() at the
    end: the sync raises DivergenceError (the rejection is sticky until reported), the
    first push applied nothing and the second applied normally."""
    import oracle as O

    D = 8
    salts = [O.mix64(7 + s) for s in range(2)]
    t = hps.ShardSet(2, D, 1024, hps.ADAGRAD, salts=salts)
    orc = O.Restatement(salts, D, "adagrad")
    ews = [hps.EmbeddingWorker(t, hps.MEAN) for _ in range(2)]
    rng = np.random.default_rng(1)
    B, F = 6, 2
    batches = []
    for k in range(2):
        ids = rng.integers(0, 40, B * F).astype(np.uint64)
        offs = np.arange(B * F + 1, dtype=np.uint32)
        g = (rng.standard_normal((B, F, D)) * 0.1).astype(np.float32)
        batches.append((ids, offs, g))
    batches[0][2][2, 1, 3] = np.nan
    for k, (ids, offs, g) in enumerate(batches):
        ews[k].register_batch(ids, offs, B, F)
        ews[k].serve_pull()
        assert ews[k].apply_backward(g, 0.1, k + 1, flags=hps.ASYNC)
        orc.pull_batch(B, F, ids, offs.astype(np.uint64), "mean")
        if k == 1:
            orc.push_batch(B, F, ids, offs.astype(np.uint64), g, 0.1, k + 1, agg="mean")
    with pytest.raises(hps.DivergenceError):
        t.sync()
    t.sync()  # reported once
    keys = np.arange(40, dtype=np.uint64)
    w, a, v, p = t.peek(keys)
    wo, ao, vo, po = orc.peek(keys)
    assert (p == po).all()
    assert w[p].tobytes() == wo[po].tobytes() and a[p].tobytes() == ao[po].tobytes()
    assert (v[p] == vo[po]).all()


def test_batch_registered_before_reset_is_refused(hps):
    """A batch registered (slots resolved) before reset_for_recovery / a checkpoint load
    may not pull or push through its stale slots: HPS_E_STALE_SAMPLE."""
    D = 4
    t = hps.ShardSet(1, D, 256, hps.ADAGRAD, salts=[3])
    ew = hps.EmbeddingWorker(t, hps.MEAN)
    ids = np.array([1, 2, 3, 4], np.uint64)
    offs = np.arange(5, dtype=np.uint32)
    ew.register_batch(ids, offs, 4, 1)
    ew.serve_pull()
    img = t.save_checkpoint(0)
    t.reset_for_recovery()
    with pytest.raises(hps.StaleSampleError):
        ew.apply_backward(np.ones((4, 1, D), np.float32), 0.1, 1)
    ew.register_batch(ids, offs, 4, 1)
    t.load_checkpoint([img])
    with pytest.raises(hps.StaleSampleError):
        ew.serve_pull()
    ew.register_batch(ids, offs, 4, 1)  # registering again is fine
    ew.serve_pull()
    assert ew.apply_backward(np.ones((4, 1, D), np.float32), 0.1, 1)


def test_batch_push_refuses_out_delays(hps):
    import ctypes as C

    t = hps.ShardSet(1, 4, 64, hps.SGD, salts=[1])
    ew = hps.EmbeddingWorker(t, hps.SUM)
    ew.register_batch(np.array([5], np.uint64), np.array([0, 1], np.uint32), 1, 1)
    ew.serve_pull()
    g = np.ones((1, 1, 4), np.float32)
    dl = np.zeros(1, np.uint32)
    acc = C.c_int(0)
    rc = hps.lib().hps_batch_push(ew.h, g.ctypes.data, 0.1, 1, t.epoch(), 0, dl.ctypes.data,
                                  C.byref(acc), 0, None)
    with pytest.raises(hps.PreconditionError):
        hps.check(rc, "push")


def test_overflow_bound_exact_check_accepts_finite_large_gradients(hps):
    """Gradients so large that the streaming bound is inconclusive (|g| * F >= 2^127) but
    every pair contribution is finite: the last block's exact check accepts the push and
    the update matches the oracle; a pair whose sum overflows is rejected."""
    import oracle as O

    D = 3
    t = hps.ShardSet(1, D, 64, hps.SGD, salts=[4])
    orc = O.Restatement([4], D, "sgd")
    ew = hps.EmbeddingWorker(t, hps.SUM)
    ids = np.array([1, 2, 1, 3], np.uint64)
    offs = np.array([0, 1, 2, 3, 4], np.uint32)  # B=2, F=2, one listing per group
    g = np.zeros((2, 2, D), np.float32)
    g[0, 0] = [2.0e38, -1.0, 0.5]
    g[0, 1] = [1.0, 2.0, 3.0]
    g[1, 0] = [2.0e38, 1.0, 1.0]
    g[1, 1] = [-2.0e38, 0.0, 0.0]
    ew.register_batch(ids, offs, 2, 2)
    ew.serve_pull()
    orc.pull_batch(2, 2, ids, offs.astype(np.uint64), "sum")
    assert ew.apply_backward(g, 1e-40, 1)
    orc.push_batch(2, 2, ids, offs.astype(np.uint64), g, 1e-40, 1, agg="sum")
    keys = np.array([1, 2, 3], np.uint64)
    assert t.peek(keys)[0].tobytes() == orc.peek(keys)[0].tobytes()
    # id 1 twice in one sample, both 2e38 -> the fp64 sum 4e38 overflows float
    ids2 = np.array([1, 1], np.uint64)
    offs2 = np.array([0, 1, 2], np.uint32)
    g2 = np.full((1, 2, D), 2.0e38, np.float32)
    ew.register_batch(ids2, offs2, 1, 2)
    ew.serve_pull()
    before = t.peek(keys)[0].copy()
    with pytest.raises(hps.DivergenceError):
        ew.apply_backward(g2, 1e-40, 2)
    assert t.peek(keys)[0].tobytes() == before.tobytes()


def test_table_without_tag_ring_refuses_what_it_cannot_count(hps):
    """tag_ring=False (the in-order pipelines' tables): in-order tracked applies count
    delays exactly; an out-of-order step tag, or a tracked apply after an untracked write,
    is refused with ClockError before anything mutates."""
    import oracle as O

    D = 2
    t = hps.ShardSet(1, D, 64, hps.ADAGRAD, salts=[11], tag_ring=False)
    orc = O.Restatement([11], D, "adagrad")
    ids = np.array([8, 9], np.uint64)
    _, rv = t.lookup(ids)
    orc.lookup(ids)
    g = np.ones((2, D), np.float32)
    for step in (1, 2, 4):
        okg, dg = t.apply_gradients(ids, g, rv, 0.01, step)
        _, do = orc.apply(ids, g, rv, 0.01, step)
        assert (dg == do).all()
    before = t.peek(ids)
    with pytest.raises(hps.ClockError):
        t.apply_gradients(ids, g, rv, 0.01, 3)
    after = t.peek(ids)
    assert before[0].tobytes() == after[0].tobytes() and (before[2] == after[2]).all()
    t.apply_gradients_map({8: [1.0, 1.0]}, 0.01)
    with pytest.raises(hps.ClockError):
        t.apply_gradients(ids, g, rv, 0.01, 5)
    t.reset_for_recovery()  # a clear forgets both conditions
    _, rv = t.lookup(ids)
    assert t.apply_gradients(ids, g, rv, 0.01, 1)[0]


# ---------------------------------------------------------------- LRU eviction (f3)


def _ref_split(ids, S):
    from paper_2111_05897_b200 import workloads as W

    sh = (W.mix64(np.asarray(ids, np.uint64)) % np.uint64(S)).astype(np.int64)
    return [np.nonzero(sh == s)[0] for s in range(S)]


@pytest.mark.parametrize("D,opt,cap", [(4, "adagrad", 16), (64, "adagrad", 40), (5, "sgd", 7)])
def test_lru_eviction_matches_reference(hps, D, opt, cap):
    """Capacity-bound shards over a cycling working set: every lookup's values and
    versions, every apply's delays, and the eviction / miss / clock-reset counters equal
    the reference's PsShards (LruStore eviction, re-init on re-miss; oracle/_ref). Calls
    mix hits, misses that fit and misses that evict (the sequential path)."""
    import oracle as O

    S = 2
    salts = [O.mix64(7 + s) for s in range(S)]
    t = hps.ShardSet(S, D, 0, hps.ADAGRAD if opt == "adagrad" else hps.SGD, salts=salts,
                     lru_shard_capacity=cap)
    ref = O.Reference(salts, cap, D, opt, "mean", 1)
    rng = np.random.default_rng(D + cap)
    space = 5 * cap
    step = 0
    for it in range(60):
        lo = (it * 3) % space  # a window that drifts over the id space
        n = int(rng.integers(1, 2 * cap))
        ids = ((lo + rng.integers(0, 2 * cap, n)) % space).astype(np.uint64)
        parts = _ref_split(ids, S)
        if it % 3 != 2:
            vals, ver = t.lookup(ids)
            for s, idx in enumerate(parts):
                if len(idx):
                    rv_, rver = ref.shard_lookup(s, ids[idx])
                    assert vals[idx].tobytes() == rv_.tobytes(), (it, s)
                    assert (ver[idx] == rver).all(), (it, s)
        else:
            step += 1
            g = (rng.standard_normal((n, D)) * 0.3).astype(np.float32)
            rv = rng.integers(0, 3, n).astype(np.uint64)
            ok, dl = t.apply_gradients(ids, g, rv, 0.1, step)
            assert ok
            for s, idx in enumerate(parts):
                if len(idx):
                    okr, dr = ref.shard_apply(s, ids[idx], g[idx], rv[idx], 0.1, step, 0)
                    assert (dl[idx] == dr).all(), (it, s, dl[idx], dr)
    cs = [ref.shard_counters(s) for s in range(S)]
    c = t.counters()
    assert c.evictions == sum(x["evictions"] for x in cs) > 0
    assert c.misses == sum(x["misses"] for x in cs)
    assert c.clock_resets == sum(x["clock_resets"] for x in cs)
    assert c.size == sum(x["size"] for x in cs)


def test_lru_reference_eviction_cases(hps):
    """test_embedding_ps.cpp:147-169 (EvictionReinitializesAndCounts) and :214-227
    (EvictionResetIsNotNegative) through the C ABI."""
    t = hps.ShardSet(1, 2, 0, hps.SGD, salts=[11], lru_shard_capacity=2)
    fresh = t.lookup([1])[0].copy()
    t.apply_gradients_map({1: [1.0, 1.0]}, 0.5)
    t.lookup([2])
    t.lookup([3])  # evicts 1
    assert t.eviction_count() == 1
    assert t.lookup([1])[0].tobytes() == fresh.tobytes()  # re-initialised like fresh
    a = hps.ShardSet(1, 2, 0, hps.ADAGRAD, salts=[11], lru_shard_capacity=2)
    g = np.ones((1, 2), np.float32)
    a.lookup([1])
    a.apply_gradients([1], g, [0], 0.01, 1)
    a.apply_gradients([1], g, [1], 0.01, 2)
    _, v = a.lookup([1])
    assert v[0] == 2
    a.lookup([2])
    a.lookup([3])  # evicts id 1, its version restarts
    ok, d = a.apply_gradients([1], g, v, 0.01, 3)
    assert ok and d[0] == 0
    assert a.clock_reset_count() == 1


def test_lru_checkpoint_keeps_recency_and_victim(hps):
    """test_embedding_ps.cpp:272-291 (RoundtripPreservesStateAndVictim): after save and
    load, the next miss evicts the same row as without the round trip; the reference
    loads the image and evicts that row too."""
    import oracle as O

    D, cap = 3, 4
    mk = lambda: hps.ShardSet(1, D, 0, hps.SGD, salts=[11], lru_shard_capacity=cap)
    a = mk()
    for ids in ([1, 2, 3, 4], [2], [1, 3]):  # recency, oldest first: 4, 2, 1, 3
        a.lookup(np.array(ids, np.uint64))
    img = a.save_checkpoint(0)
    b = mk()
    b.load_checkpoint([img])
    ref = O.Reference([11], cap, D, "sgd", "mean", 1)
    ref.shard_import(0, img)
    for t_ in (a, b):
        t_.lookup(np.array([9], np.uint64))  # evicts 4
        assert t_.eviction_count() == 1
    ref.shard_lookup(0, np.array([9], np.uint64))
    for t_ in (a, b):
        _, _, _, present = t_.peek(np.array([1, 2, 3, 4, 9], np.uint64))
        assert present.tolist() == [True, True, True, False, True]
    assert ref.shard_counters(0)["evictions"] == 1
    assert b.save_checkpoint(0) == a.save_checkpoint(0)


def test_lru_checkpoint_save_load_save_byte_identical(hps):
    """test_embedding_ps.cpp:254-270: an image loaded into an LRU table saves back byte
    for byte (rows return to their image slots, the recency chain to its order), and the
    reference loads our image and saves the same bytes."""
    import oracle as O

    D, cap = 3, 8
    a = hps.ShardSet(1, D, 0, hps.ADAGRAD, salts=[5], lru_shard_capacity=cap)
    rng = np.random.default_rng(2)
    for _ in range(50):
        i = int(rng.integers(0, 12))
        a.lookup(np.array([i], np.uint64))
        a.apply_gradients_map({i: rng.uniform(-1, 1, D).astype(np.float32)}, 0.05)
    first = a.save_checkpoint(0)
    b = hps.ShardSet(1, D, 0, hps.ADAGRAD, salts=[5], lru_shard_capacity=cap)
    b.load_checkpoint([first])
    assert b.save_checkpoint(0) == first
    ref = O.Reference([5], cap, D, "adagrad", "mean", 1)
    ref.shard_import(0, first)
    im = O.parse_hps1(ref.shard_export(0))["rows"]
    mine = O.parse_hps1(first)["rows"]
    assert list(im) == list(mine)  # the same recency chain
    for k in mine:
        assert im[k][0].tobytes() == mine[k][0].tobytes()
        assert im[k][1].tobytes() == mine[k][1].tobytes() and im[k][2] == mine[k][2]
