"""The hybrid step: dense tower, synchronous dense
all-reduce and bounded-staleness embedding pipeline.

CPU: the tower's init / forward-backward / SGD against the reference's own DenseNet
(dense_nn.hpp, compiled in oracle/_ref), the canonical all-reduce bit-exact against the
reference's AllReduceHub (nn_worker.hpp:214-226), also across gloo ranks.
GPU: HybridTrainer against an oracle loop (the C restatement's table + the reference's
DenseNet) at staleness 0 and 2, step by step; staleness 4 vs 0 loss curves.
"""
import numpy as np
import pytest

from conftest import cuda_available

import oracle as O
from paper_2111_05897_b200 import dense
from paper_2111_05897_b200 import workloads as W

# Dense forward/backward is cuBLAS/torch fp32 over whole batches vs the reference's
# per-sample loops: same formula, different summation order.
FWD_RTOL = 1e-5
# After several coupled steps (dense params <-> embeddings) the drift compounds.
TRAIN_RTOL = 2e-4


@pytest.mark.parametrize("dims,seed", [([10, 4, 3], 5), ([1677, 64, 32], 0), ([7], 9)])
def test_dense_init_matches_reference(dims, seed):
    assert dense.glorot_params(dims, seed).tobytes() == O.ref_dense_init(dims, seed).tobytes()


@pytest.mark.parametrize("B", [1, 7, 64])
def test_dense_forward_backward_matches_reference(B):
    import torch

    dims = [40, 16, 8]
    rng = np.random.default_rng(B)
    p = O.ref_dense_init(dims, 3)
    x = (rng.random((B, 40)) - 0.5).astype(np.float32)
    y = (rng.random(B) > 0.5).astype(np.float32)
    t = dense.DenseTower(40, (16, 8), 3, device="cpu")
    loss, prob, ig = t.forward_backward(torch.from_numpy(x), torch.from_numpy(y))
    rl, rp, rg, rig = O.ref_dense_fwd_bwd(dims, p, x, y)
    np.testing.assert_allclose(float(loss), rl, rtol=FWD_RTOL)
    np.testing.assert_allclose(prob.numpy(), rp, rtol=FWD_RTOL, atol=1e-7)
    np.testing.assert_allclose(t.grad.numpy(), rg, rtol=FWD_RTOL, atol=1e-7)
    np.testing.assert_allclose(ig.numpy(), rig, rtol=FWD_RTOL, atol=1e-8)
    # embedding slice only (split_group_grads drops the non-id tail)
    _, _, ig2 = t.forward_backward(torch.from_numpy(x), torch.from_numpy(y), input_cols=24)
    assert ig2.shape == (B, 24)
    np.testing.assert_allclose(ig2.numpy(), ig.numpy()[:, :24], rtol=FWD_RTOL, atol=1e-8)
    # the input as column blocks [embeddings | non-id] (the hybrid trainer's form)
    t3 = dense.DenseTower(40, (16, 8), 3, device="cpu")
    l3, p3, ig3 = t3.forward_backward([torch.from_numpy(x[:, :24].copy()),
                                       torch.from_numpy(x[:, 24:].copy())],
                                      torch.from_numpy(y), input_cols=24)
    np.testing.assert_allclose(float(l3), rl, rtol=FWD_RTOL)
    np.testing.assert_allclose(t3.grad.numpy(), rg, rtol=FWD_RTOL, atol=1e-7)
    np.testing.assert_allclose(ig3.numpy(), rig[:, :24], rtol=FWD_RTOL, atol=1e-8)


@pytest.mark.parametrize("K", [1, 2, 3, 5, 8])
def test_canonical_mean_bit_exact(K):
    import torch

    parts = np.random.default_rng(K).standard_normal((K, 1001)).astype(np.float32)
    got = dense.canonical_mean(torch.from_numpy(parts)).numpy()
    assert got.tobytes() == O.ref_allreduce(parts).tobytes()


def test_sgd_step_matches_reference_and_rejects_nonfinite():
    import torch

    from paper_2111_05897_b200.hps import DivergenceError

    t = dense.DenseTower(12, (5,), 1, device="cpu")
    p0 = t.params.numpy().copy()
    g = np.random.default_rng(0).standard_normal(t.param_count).astype(np.float32)
    t.sgd_step(torch.from_numpy(g), 0.05)
    assert t.params.numpy().tobytes() == O.ref_sgd_step(p0, g, 0.05).tobytes()
    p1 = t.params.numpy().copy()
    g[3] = np.nan
    with pytest.raises(DivergenceError):
        t.sgd_step(torch.from_numpy(g), 0.05)
    assert t.params.numpy().tobytes() == p1.tobytes()
    # deferred check: a non-finite gradient applies nothing
    t.sgd_step(torch.from_numpy(g), 0.05, finite=torch.isfinite(torch.from_numpy(g)).all())
    assert t.params.numpy().tobytes() == p1.tobytes()


def _allreduce_rank(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.from_numpy(np.random.default_rng(100 + rank).standard_normal(777).astype(np.float32))
    out = dense.allreduce_mean(g)
    q.put((rank, out.numpy().tobytes()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_allreduce_mean_gloo_bit_exact(world):
    import multiprocessing as mp
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_allreduce_rank, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=30)
    parts = np.stack([np.random.default_rng(100 + r).standard_normal(777).astype(np.float32)
                      for r in range(world)])
    want = O.ref_allreduce(parts).tobytes()
    assert all(res[r] == want for r in range(world))


def test_dense_inputs_deterministic():
    cfg = W.CONFIGS["c5"]
    b = W.make_batch(cfg, 3, 128)
    x1, y1 = W.make_dense_inputs(cfg, b)
    x2, y2 = W.make_dense_inputs(cfg, b)
    assert x1.shape == (128, W.C5_NON_ID) and y1.shape == (128,)
    assert x1.tobytes() == x2.tobytes() and y1.tobytes() == y2.tobytes()
    assert set(np.unique(y1)) <= {0.0, 1.0}


# ---- GPU: the trainer against an oracle loop -------------------------------------------

def _small_stream(steps, B=48, F=4, D=8, nd=3, seed=11):
    rng = np.random.default_rng(seed)
    out = []
    for s in range(steps):
        ids, offs = W.random_csr(rng, B, F, 3, 200)
        x = (rng.random((B, nd)) * 2 - 1).astype(np.float32)
        y = (rng.random(B) > 0.5).astype(np.float32)
        out.append((ids, offs, x, y))
    return out


def _oracle_loop(stream, salts, D, F, nd, hidden, tau, dense_lr, emb_lr, seed):
    """The reference semantics restated: pull(s) after the pushes of steps <= s-1-tau;
    dense step with the reference's DenseNet; SGD; push(s) after pull(s+tau)."""
    orc = O.Restatement(salts, D, "adagrad")
    dims = [F * D + nd] + list(hidden)
    params = O.ref_dense_init(dims, seed)
    losses, pending = [], []
    for s, (ids, offs, x, y) in enumerate(stream):
        B = len(y)
        po, rv = orc.pull_batch(B, F, ids, offs.astype(np.uint64), "mean")
        inp = np.concatenate([po.reshape(B, -1), x], axis=1)
        loss, _, dg, ig = O.ref_dense_fwd_bwd(dims, params, inp, y)
        params = O.ref_sgd_step(params, O.ref_allreduce(dg[None]), dense_lr)
        eg = np.ascontiguousarray(ig[:, :F * D].reshape(B, F, D))
        pending.append((s, ids, offs, eg, rv))
        if len(pending) > tau:
            ps, pids, poffs, peg, prv = pending.pop(0)
            orc.push_batch(len(peg), F, pids, poffs.astype(np.uint64), peg, emb_lr, ps + 1,
                           read_versions=prv, agg="mean")
        losses.append(loss)
    while pending:
        ps, pids, poffs, peg, prv = pending.pop(0)
        orc.push_batch(len(peg), F, pids, poffs.astype(np.uint64), peg, emb_lr, ps + 1,
                       read_versions=prv, agg="mean")
    return np.array(losses), params, orc


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a GPU")
@pytest.mark.parametrize("tau", [0, 2])
def test_hybrid_trainer_matches_oracle_loop(tau):
    import torch

    from paper_2111_05897_b200 import hps
    from paper_2111_05897_b200.hybrid import HybridTrainer

    D, F, nd, hidden, S = 8, 4, 3, (16, 8), 4
    salts = [W.mix64_int(7 + s) for s in range(S)]
    stream = _small_stream(8, F=F, D=D, nd=nd)
    table = hps.ShardSet(S, D, 4096, hps.ADAGRAD, salts=salts, device=0)
    tr = HybridTrainer(table, F, nd, hidden=hidden, dense_lr=0.1, embedding_lr=0.2,
                       staleness=tau, init_seed=5)
    dev = torch.device("cuda", 0)
    losses = []
    for ids, offs, x, y in stream:
        loss = tr.step(torch.from_numpy(ids.view(np.int64)).to(dev),
                       torch.from_numpy(offs.view(np.int32)).to(dev),
                       torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev))
        losses.append(loss)
    tr.flush()
    torch.cuda.synchronize()
    table.sync()
    got = np.array([float(v) for v in losses])
    want, params, orc = _oracle_loop(stream, salts, D, F, nd, hidden, tau, 0.1, 0.2, 5)
    np.testing.assert_allclose(got, want, rtol=TRAIN_RTOL)
    np.testing.assert_allclose(tr.tower.params.cpu().numpy(), params, rtol=TRAIN_RTOL,
                               atol=1e-6)
    uniq = np.unique(np.concatenate([s[0] for s in stream]))
    w, a, v, present = table.peek(uniq)
    wo, ao, vo, _ = orc.peek(uniq)
    assert present.all()
    np.testing.assert_array_equal(v, vo)  # versions: integer, exact
    np.testing.assert_allclose(w, wo, rtol=TRAIN_RTOL, atol=1e-6)
    np.testing.assert_allclose(a, ao, rtol=1e-3, atol=1e-9)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a GPU")
def test_hybrid_staleness_loss_curve():
    """Bounded staleness 4 vs sync on the C5 stream shape (small batch): both learn, and
    the late-training loss of the stale run stays within 3% of the sync run."""
    import torch

    from paper_2111_05897_b200 import hps
    from paper_2111_05897_b200.hybrid import HybridTrainer

    cfg = W.Config("c5s", 1024, 26, 2_000_000, 16, "adagrad", "mean")
    dev = torch.device("cuda", 0)
    data = []
    for s in range(60):
        b = W.make_batch(cfg, s)
        x, y = W.make_dense_inputs(cfg, b)
        data.append(tuple(torch.from_numpy(a).to(dev) for a in
                          (b.ids.view(np.int64), b.offsets.view(np.int32), x, y)))
    curves = {}
    for tau in (0, 4):
        table = hps.ShardSet(cfg.shards, cfg.dim, cfg.table_capacity(), hps.ADAGRAD,
                             salts=cfg.salts(), device=0)
        tr = HybridTrainer(table, cfg.features, W.C5_NON_ID, hidden=W.C5_HIDDEN,
                           dense_lr=0.5, embedding_lr=0.5, staleness=tau)
        ls = [tr.step(*d) for d in data]
        tr.flush()
        torch.cuda.synchronize()
        curves[tau] = np.array([float(v) for v in ls])
    for tau, c in curves.items():
        assert c[-10:].mean() < c[:5].mean(), f"tau={tau} did not learn: {c}"
    rel = abs(curves[4][-10:].mean() - curves[0][-10:].mean()) / curves[0][-10:].mean()
    assert rel < 0.03, (rel, curves)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_available(), reason="needs a GPU")
def test_hybrid_trainer_reports_divergence():
    """A non-finite dense input makes the loss and the dense gradient non-finite: the
    dense update of that step is skipped and flush() raises DivergenceError (the
    reference raises it in train_step, dense_nn.hpp:233,268, and aborts the run)."""
    import torch

    from paper_2111_05897_b200 import hps
    from paper_2111_05897_b200.hybrid import HybridTrainer

    D, F, nd, S = 8, 4, 3, 4
    salts = [W.mix64_int(7 + s) for s in range(S)]
    stream = _small_stream(3, F=F, D=D, nd=nd)
    table = hps.ShardSet(S, D, 4096, hps.ADAGRAD, salts=salts, device=0)
    tr = HybridTrainer(table, F, nd, hidden=(8,), staleness=1, init_seed=5)
    dev = torch.device("cuda", 0)
    for k, (ids, offs, x, y) in enumerate(stream):
        x = x.copy()
        if k == 1:
            x[0, 0] = np.nan
        tr.step(torch.from_numpy(ids.view(np.int64)).to(dev),
                torch.from_numpy(offs.view(np.int32)).to(dev),
                torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev))
    with pytest.raises(hps.DivergenceError):
        tr.flush()
    tr.check()  # reported once
