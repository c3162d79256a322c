"""TEST INFRASTRUCTURE: one multi-rank sharded-step parity case, run by every rank.

The global batch of step s has W*B samples; rank r serves samples r, r+W, ... -- the
reference's sample -> embedding-worker assignment (sample i -> EW i % E,
oracle/ref_driver.cpp; sid = (i % E) << 56 | i / E, data.hpp:392). The expected result
is the oracle table driven with the whole global batch and those sample keys (pinned
against the reference's multi-worker run in tests/test_oracle_pinning.py).
"""
from __future__ import annotations

import os
import sys
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def global_batch(step, W, B, F, space, seed=11, fixed_shape=False):
    rng = np.random.default_rng(seed * 1000 + step)
    crng = np.random.default_rng(seed) if fixed_shape else rng
    counts = crng.integers(0, 4, W * B * F)
    counts[crng.random(W * B * F) < 0.5] = 1
    offs = np.zeros(W * B * F + 1, np.int64)
    np.cumsum(counts, out=offs[1:])
    ids = rng.integers(0, space, int(offs[-1])).astype(np.uint64)
    if len(ids) > 3:
        ids[rng.integers(0, len(ids), 2)] = np.uint64(0xFFFFFFFFFFFFFFFF)  # the special id
    return ids, offs, counts


def local_part(ids, offs, W, B, F, r):
    """CSR of samples r, r+W, ... of the global batch."""
    lid, loff = [], [0]
    for b in range(r, W * B, W):
        for f in range(F):
            sg = b * F + f
            seg = ids[offs[sg]:offs[sg + 1]]
            lid.extend(seg.tolist())
            loff.append(loff[-1] + len(seg))
    return np.array(lid, np.uint64), np.array(loff, np.int64)


def _spawn_world(target, world, timeout, args_of, kw, attempts=3):
    """Runs target(*args_of(rank, port), **kw, q=q) in `world` spawned processes on a fresh
    rendezvous port. A rank that fails stops the wait (its peers would block in the
    rendezvous); a port another process took between the probe and the bind
    (EADDRINUSE) retries on a new port."""
    import multiprocessing as mp
    import queue
    import socket

    for attempt in range(attempts):
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        procs = [ctx.Process(target=target, args=args_of(r, port), kwargs=dict(kw, q=q))
                 for r in range(world)]
        for p in procs:
            p.start()
        results = []
        try:
            for _ in range(world):
                try:
                    r = q.get(timeout=timeout)
                except queue.Empty:
                    break
                results.append(r)
                if r[1] != "ok":
                    break
        finally:
            for p in procs:
                p.join(timeout=1 if len(results) < world else 30)
                if p.is_alive():
                    p.kill()
        if any("EADDRINUSE" in str(r[1]) for r in results) and attempt + 1 < attempts:
            continue
        if len(results) < world and all(r[1] == "ok" for r in results):
            raise TimeoutError(f"{world - len(results)} rank(s) reported nothing in {timeout} s")
        return results
    return results


class RefExpect:
    """The reference itself (oracle/_ref: E = world embedding workers over S PsShards, sync
    order) behind the Restatement calls run_rank uses; compress: PS pull replies and push
    frames carry compress_values blocks (the exchange's codec mode)."""

    def __init__(self, salts, D, opt, agg, F, world, compress):
        import oracle as O

        self.ref = O.Reference(salts, 1 << 14, D, opt, agg, F, workers=world,
                               compress=compress)
        self.D = D

    def pull_batch(self, B, F, ids, offsets, agg):
        pooled, rv, _ = self.ref.step(B, ids, offsets, pull=True, push=False)
        return pooled, rv

    def push_batch(self, B, F, ids, offsets, grads, lr, step, read_versions=None,
                   sample_keys=None, agg=None):
        self.ref.step(B, ids, offsets, grads, lr, step, True, pull=False, push=True)
        return True, None

    def peek(self, ids):
        st = self.ref.state()
        n = len(ids)
        w = np.zeros((n, self.D), np.float32)
        a = np.zeros((n, self.D), np.float32)
        v = np.zeros(n, np.uint64)
        p = np.zeros(n, bool)
        for k, i in enumerate(ids):
            if int(i) in st:
                w[k], a[k], v[k] = st[int(i)]
                p[k] = True
        return w, a, v, p


def run_rank(rank, world, backend, port, use_device, D=8, B=12, F=3, steps=3, agg="mean",
             opt="adagrad", space=60, transport="p2p", graph=False, nan_step=-1, codec=0.0,
             q=None):
    try:
        import torch
        import torch.distributed as dist

        import oracle as O
        from paper_2111_05897_b200 import hps
        from paper_2111_05897_b200.sharded import ShardedEmbeddingWorker

        if use_device:
            # ranks may share a GPU (gloo control plane + the p2p transport: CUDA IPC works
            # between processes on one device), so a 1-GPU box runs the multi-rank exchange
            torch.cuda.set_device(rank % torch.cuda.device_count())
        dist.init_process_group(backend, init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        S = 8
        salts = [O.mix64(7 + s) for s in range(S)]
        # the whole global batch, one table (codec: the reference itself with compression)
        exp = RefExpect(salts, D, opt, agg, F, world, True) if codec else \
            O.Restatement(salts, D, opt)
        if use_device:
            dev = torch.device("cuda", rank % torch.cuda.device_count())
            table = hps.ShardSet(S, D, 1 << 14, hps.ADAGRAD if opt == "adagrad" else hps.SGD,
                                 salts=salts)
            ew = ShardedEmbeddingWorker(table, hps.MEAN if agg == "mean" else hps.SUM,
                                        transport=transport, max_ids=world * B * F * 4,
                                        codec_kappa=codec)
            owner_peek = table.peek
        else:
            from sharded_oracle_ops import EpochOnly, OracleOps

            dev = torch.device("cpu")
            local = O.Restatement(salts, D, opt)
            ew = ShardedEmbeddingWorker(EpochOnly(local), hps.MEAN if agg == "mean" else hps.SUM,
                                        ops=OracleOps(local, world, S, D, agg))
            owner_peek = local.peek
        seen = set()
        cg = None  # graph mode: one step captured at s == 1, replayed on new inputs
        flags = hps.ASYNC | hps.DEVICE_STEP if graph else hps.ASYNC
        for s in range(steps):
            gids, goffs, _ = global_batch(s, world, B, F, space, fixed_shape=graph)
            rng = np.random.default_rng(500 + s)
            g_all = (rng.standard_normal((world * B, F, D)) * 0.3).astype(np.float32)
            if s == nan_step:  # one non-finite gradient of the first non-empty group
                g0 = int(np.argmax(np.diff(goffs) > 0))
                g_all[g0 // F, g0 % F, D // 2] = np.nan
            sk = np.array([((i % world) << 56) | (i // world) for i in range(world * B)],
                          np.uint64)
            pooled_exp, rv_exp = exp.pull_batch(world * B, F, gids, goffs.astype(np.uint64), agg)
            lid, loff = local_part(gids, goffs, world, B, F, rank)
            seen.update(int(x) for x in gids)
            n_ids = torch.from_numpy(lid.view(np.int64).copy())
            n_off = torch.from_numpy(loff.astype(np.int32))
            n_g = torch.from_numpy(np.ascontiguousarray(g_all[rank::world]))
            if graph and s >= 1:
                t_ids.copy_(n_ids)
                t_off.copy_(n_off)
                g_local.copy_(n_g)
                if cg is None:
                    torch.cuda.synchronize()
                    cg = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(cg, capture_error_mode="thread_local"):
                        ew.register_batch(t_ids, t_off, B, F)
                        ew.serve_pull(out_pooled=pooled)
                        ew.apply_backward(g_local, 0.05, 0, flags=flags)
                cg.replay()  # (capture itself does not run the kernels)
            else:
                t_ids, t_off, g_local = n_ids.to(dev), n_off.to(dev), n_g.to(dev)
                ew.register_batch(t_ids, t_off, B, F)
                pooled = ew.serve_pull()
            if not (graph and s >= 1):
                got = pooled.cpu().numpy()
            else:
                torch.cuda.synchronize()
                got = pooled.cpu().numpy()
            want = pooled_exp[rank::world]
            assert got.tobytes() == want.tobytes(), f"rank {rank} step {s}: pooled differs"
            if not (graph and s >= 1):
                ok = ew.apply_backward(g_local, 0.05, s + 1, flags=flags)
                assert ok
            if s == nan_step:
                # world 1: the (only) owner rejects the whole step -- nothing applied, the
                # DivergenceError surfaces from the next synchronising call
                assert world == 1 and use_device
                torch.cuda.synchronize()
                try:
                    table.sync()
                    raise AssertionError("non-finite contribution not reported")
                except hps.DivergenceError:
                    pass
                continue
            ok2, _ = exp.push_batch(world * B, F, gids, goffs.astype(np.uint64), g_all, 0.05,
                                    s + 1, read_versions=rv_exp, sample_keys=sk, agg=agg)
            assert ok2
        if use_device:
            torch.cuda.synchronize()
            table.sync()  # deferred (HPS_ASYNC) errors of the steps surface here
        mine = np.array(sorted(i for i in seen
                               if hps.route_shard(i, S) % world == rank), np.uint64)
        w, a, v, p = owner_peek(mine)
        we, ae, ve, pe = exp.peek(mine)
        assert p.all() and pe.all()
        assert w.tobytes() == we.tobytes(), f"rank {rank}: rows differ"
        assert a.tobytes() == ae.tobytes(), f"rank {rank}: optimizer state differs"
        assert (v == ve).all(), f"rank {rank}: versions differ"
        dist.barrier()
        dist.destroy_process_group()
        if q is not None:
            q.put((rank, "ok", len(mine)))
    except Exception:
        if q is not None:
            q.put((rank, traceback.format_exc(), 0))
        raise


def run_world(world, backend, use_device, timeout=240, **kw):
    return _spawn_world(run_rank, world, timeout, lambda r, port: (r, world, backend, port, use_device), kw)


def run_hybrid_rank(rank, world, port, tau=2, D=8, B=12, F=3, nd=2, steps=6, space=60, q=None):
    """The sharded hybrid step (HybridTrainer over tau + 1 exchanges): every rank records the
    embedding gradients its dense tower produced; the owners' rows must equal the oracle
    table driven with the global batches and those gradients in the staleness-tau order
    (pull(s) before push(s - tau)), and the dense parameters must agree across ranks."""
    try:
        import torch
        import torch.distributed as dist

        import oracle as O
        from paper_2111_05897_b200 import hps
        from paper_2111_05897_b200.hybrid import HybridTrainer
        from paper_2111_05897_b200.sharded import ShardedEmbeddingWorker

        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        S = 8
        salts = [O.mix64(7 + s) for s in range(S)]
        dev = torch.device("cuda", rank)
        table = hps.ShardSet(S, D, 1 << 14, hps.ADAGRAD, salts=salts)
        ews = [ShardedEmbeddingWorker(table, hps.MEAN, max_ids=world * B * F * 4)
               for _ in range(tau + 1)]
        tr = HybridTrainer(table, F, nd, hidden=(8,), dense_lr=0.1, embedding_lr=0.2,
                           staleness=tau, sharded_workers=ews, init_seed=3)
        batches, my_grads = [], []
        for s in range(steps):
            gids, goffs, _ = global_batch(s, world, B, F, space)
            lid, loff = local_part(gids, goffs, world, B, F, rank)
            rng = np.random.default_rng(900 + 10 * s + rank)
            x = (rng.random((B, nd)) * 2 - 1).astype(np.float32)
            y = (rng.random(B) > 0.5).astype(np.float32)
            tr.step(torch.from_numpy(lid.view(np.int64)).to(dev),
                    torch.from_numpy(loff.astype(np.int32)).to(dev),
                    torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev))
            tr.sync()
            torch.cuda.synchronize()
            my_grads.append(tr._buf(s % (tau + 1), B)["grads"].cpu().numpy().copy())
            batches.append((gids, goffs))
        tr.flush()
        torch.cuda.synchronize()
        table.sync()
        allg = [None] * world
        dist.all_gather_object(allg, my_grads)
        params = [None] * world
        dist.all_gather_object(params, tr.tower.params.cpu().numpy().tobytes())
        assert all(p == params[0] for p in params), "dense replicas diverged"
        # oracle: global batch, sample i = rank i % W's local sample i // W
        exp = O.Restatement(salts, D, "adagrad")
        sk = np.array([((i % world) << 56) | (i // world) for i in range(world * B)], np.uint64)
        pending = []
        for s, (gids, goffs) in enumerate(batches):
            _, rv = exp.pull_batch(world * B, F, gids, goffs.astype(np.uint64), "mean")
            g = np.zeros((world * B, F, D), np.float32)
            for r in range(world):
                g[r::world] = allg[r][s]
            pending.append((s, gids, goffs, g, rv))
            if len(pending) > tau:
                ps, pg, po, pgr, prv = pending.pop(0)
                ok, _ = exp.push_batch(world * B, F, pg, po.astype(np.uint64), pgr, 0.2, ps + 1,
                                       read_versions=prv, sample_keys=sk, agg="mean")
                assert ok
        for ps, pg, po, pgr, prv in pending:
            exp.push_batch(world * B, F, pg, po.astype(np.uint64), pgr, 0.2, ps + 1,
                           read_versions=prv, sample_keys=sk, agg="mean")
        seen = set(int(i) for gids, _ in batches for i in gids)
        mine = np.array(sorted(i for i in seen if hps.route_shard(i, S) % world == rank),
                        np.uint64)
        w, a, v, p = table.peek(mine)
        we, ae, ve, pe = exp.peek(mine)
        assert p.all() and pe.all()
        assert w.tobytes() == we.tobytes(), f"rank {rank}: rows differ"
        assert a.tobytes() == ae.tobytes(), f"rank {rank}: optimizer state differs"
        assert (v == ve).all(), f"rank {rank}: versions differ"
        dist.barrier()
        dist.destroy_process_group()
        if q is not None:
            q.put((rank, "ok", len(mine)))
    except Exception:
        if q is not None:
            q.put((rank, traceback.format_exc(), 0))
        raise


def run_hybrid_world(world, timeout=300, **kw):
    return _spawn_world(run_hybrid_rank, world, timeout, lambda r, port: (r, world, port), kw)


def run_pipelined_rank(rank, world, port, D=8, B=12, F=3, steps=5, space=60, q=None):
    """bench.py's pipelined sharded schedule: two workers (exchanges) alternate; batch s+1
    is prefetched (routed, pairs planned) on a second stream beside batch s's lookup,
    pull and backward. Pooled outputs and the owners' rows must equal the oracle driven
    with the global batches in plain sync order."""
    try:
        import torch
        import torch.distributed as dist

        import oracle as O
        from paper_2111_05897_b200 import hps
        from paper_2111_05897_b200.sharded import ShardedEmbeddingWorker

        ndev = torch.cuda.device_count()
        torch.cuda.set_device(rank % ndev)
        # two ranks on one GPU: gloo control plane (NCCL refuses duplicate devices)
        dist.init_process_group("nccl" if ndev >= world else "gloo",
                                init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        S = 8
        salts = [O.mix64(7 + s) for s in range(S)]
        exp = O.Restatement(salts, D, "adagrad")
        dev = torch.device("cuda", rank % ndev)
        table = hps.ShardSet(S, D, 1 << 14, hps.ADAGRAD, salts=salts)
        ews = [ShardedEmbeddingWorker(table, hps.MEAN, max_ids=world * B * F * 4)
               for _ in range(2)]
        data = []
        for s in range(steps):
            gids, goffs, _ = global_batch(s, world, B, F, space)
            lid, loff = local_part(gids, goffs, world, B, F, rank)
            rng = np.random.default_rng(500 + s)
            g_all = (rng.standard_normal((world * B, F, D)) * 0.3).astype(np.float32)
            data.append((gids, goffs, torch.from_numpy(lid.view(np.int64).copy()).to(dev),
                         torch.from_numpy(loff.astype(np.int32)).to(dev), g_all,
                         torch.from_numpy(np.ascontiguousarray(g_all[rank::world])).to(dev)))
        sk = np.array([((i % world) << 56) | (i // world) for i in range(world * B)], np.uint64)
        main = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        ews[0].prefetch(data[0][2], data[0][3], B, F)
        seen = set()
        for s in range(steps):
            side.wait_stream(main)
            if s + 1 < steps:
                with torch.cuda.stream(side):
                    ews[(s + 1) % 2].prefetch(data[s + 1][2], data[s + 1][3], B, F)
            w = ews[s % 2]
            w.register_prefetched()
            pooled = w.serve_pull()
            gids, goffs, _, _, g_all, g_local = data[s]
            got = pooled.cpu().numpy()
            pooled_exp, rv_exp = exp.pull_batch(world * B, F, gids, goffs.astype(np.uint64),
                                                "mean")
            assert got.tobytes() == pooled_exp[rank::world].tobytes(), f"step {s}: pooled"
            assert w.apply_backward(g_local, 0.05, s + 1)
            main.wait_stream(side)
            exp.push_batch(world * B, F, gids, goffs.astype(np.uint64), g_all, 0.05, s + 1,
                           read_versions=rv_exp, sample_keys=sk, agg="mean")
            seen.update(int(x) for x in gids)
        torch.cuda.synchronize()
        table.sync()
        mine = np.array(sorted(i for i in seen if hps.route_shard(i, S) % world == rank),
                        np.uint64)
        w_, a_, v_, p_ = table.peek(mine)
        we, ae, ve, pe = exp.peek(mine)
        assert p_.all() and pe.all()
        assert w_.tobytes() == we.tobytes(), f"rank {rank}: rows differ"
        assert a_.tobytes() == ae.tobytes(), f"rank {rank}: optimizer state differs"
        assert (v_ == ve).all(), f"rank {rank}: versions differ"
        dist.barrier()
        dist.destroy_process_group()
        if q is not None:
            q.put((rank, "ok", len(mine)))
    except Exception:
        if q is not None:
            q.put((rank, traceback.format_exc(), 0))
        raise


def run_pipelined_world(world, timeout=300, **kw):
    return _spawn_world(run_pipelined_rank, world, timeout, lambda r, port: (r, world, port), kw)
